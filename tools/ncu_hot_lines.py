#!/usr/bin/env python3
"""Hottest CUDA source lines of one kernel in an ncu report (stall samples,
executed instructions, average active threads).

    python tools/ncu_hot_lines.py report.ncu-rep kernel_regex [--top N]
"""

from __future__ import annotations

import csv
import io
import subprocess
import sys


def num(s: str) -> float:
    try:
        return float(s)
    except ValueError:
        return 0.0


def main() -> None:
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 15
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    data, ix, cur, fname, width = [], None, None, "", 0
    for r in rows:
        if r and r[0] in ("File Name", "File Path"):
            fname = r[1].rsplit("/", 1)[-1]
        elif r and r[0] == "Line No":
            cur = {h: i for i, h in enumerate(r)} if "# Samples" in r else None
            ix = cur or ix
            width = len(r)
        elif cur is not None and len(r) == width:
            data.append([f"{fname}:{r[0]}"] + r[1:])
    tot = sum(num(r[ix["# Samples"]]) for r in data) or 1.0
    inst = sum(num(r[ix["Instructions Executed"]]) for r in data) or 1.0
    data.sort(key=lambda r: -num(r[ix["# Samples"]]))
    print(f"samples={tot:.0f} warp-instructions={inst:.0f}")
    for r in data[:top]:
        s = num(r[ix["# Samples"]])
        print(f"{r[0]:>5} {100 * s / tot:5.1f}%  inst={num(r[ix['Instructions Executed']]) / inst * 100:5.1f}%  "
              f"thr={r[ix['Avg. Threads Executed']]:>4}  {r[1].strip()[:100]}")


if __name__ == "__main__":
    main()
