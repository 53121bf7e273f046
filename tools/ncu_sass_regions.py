#!/usr/bin/env python3
"""Stall samples and executed instructions of one kernel, per window of SASS
instructions (from `ncu -i REP --page source --csv --print-source sass`).

    python tools/ncu_sass_regions.py REP.ncu-rep KERNEL_REGEX [--window 50] [--dump START END]
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import subprocess


def load(rep: str, kernel: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kernel}", "--page", "source", "--csv",
                          "--print-source", "sass"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(r for r in rows if "Address" in r and "Source" in r)
    ix = {k: i for i, k in enumerate(hdr)}
    res = []
    for r in rows:
        if len(r) != len(hdr) or r[ix["Address"]] == "Address":
            continue
        try:
            res.append({"addr": r[ix["Address"]], "src": r[ix["Source"]],
                        "samp": float(r[ix["Warp Stall Sampling (All Samples)"]] or 0),
                        "inst": float(r[ix["Instructions Executed"]] or 0)})
        except ValueError:
            continue
    return res


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("kernel")
    ap.add_argument("--window", type=int, default=50)
    ap.add_argument("--dump", nargs=2, type=int)
    a = ap.parse_args()
    data = load(a.rep, a.kernel)
    ts = sum(d["samp"] for d in data) or 1.0
    ti = sum(d["inst"] for d in data) or 1.0
    print(f"{len(data)} SASS lines, {ts:.0f} samples, {ti:.3e} warp-instructions")
    if a.dump:
        for k in range(*a.dump):
            d = data[k]
            print(f"{k:5d} {d['samp'] / ts * 100:6.2f}% {d['inst'] / ti * 100:6.3f}%  {d['src']}")
        return
    for k in range(0, len(data), a.window):
        ch = data[k:k + a.window]
        s = sum(d["samp"] for d in ch) / ts * 100
        i = sum(d["inst"] for d in ch) / ti * 100
        if s < 0.3 and i < 0.3:
            continue
        c = collections.Counter(d["src"].split()[0].split(".")[0] if d["src"].strip() else "" for d in ch)
        print(f"{k:5d} samples {s:5.1f}%  inst {i:5.1f}%  " + " ".join(f"{o}:{n}" for o, n in c.most_common(5)))


if __name__ == "__main__":
    main()
