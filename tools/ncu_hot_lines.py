#!/usr/bin/env python3
"""Hottest CUDA source lines of one kernel in an ncu report: executed
warp-level instructions and warp-stall samples per source line (files
compiled with -lineinfo, report captured with --import-source on).

    python tools/ncu_hot_lines.py report.ncu-rep kernel_regex [--top N] [--skip K]

kernel_regex is matched by ncu against the function name (no template
arguments: use --skip to pick the K-th matching launch).
"""

from __future__ import annotations

import csv
import io
import subprocess
import sys


def main() -> None:
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25
    skip = sys.argv[sys.argv.index("--skip") + 1] if "--skip" in sys.argv else "0"
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--launch-skip", skip,
                          "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    fname, data = "", []
    for r in csv.reader(io.StringIO(out)):
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif r and r[0].isdigit():
            try:  # Line No, Source, Address, Source, stall (all), stall (not issued), # Samples, Instructions Executed
                data.append((int(r[7]), int(r[6]), fname, r[0], r[1][:110]))
            except (ValueError, IndexError):
                pass
    tot = sum(d[0] for d in data) or 1
    ts = sum(d[1] for d in data) or 1
    print(f"instructions {tot}  stall samples {ts}")
    for d in sorted(data, reverse=True)[:top]:
        print(f"{d[0]:>11} {100 * d[0] / tot:5.1f}%  samples {100 * d[1] / ts:5.1f}%  {d[2]}:{d[3]}  {d[4]}")


if __name__ == "__main__":
    main()
