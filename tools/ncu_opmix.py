#!/usr/bin/env python3
"""Dynamic SASS opcode mix of one kernel in an ncu report.
    python tools/ncu_opmix.py rep.ncu-rep kernel_regex [--top N]"""
import collections, csv, io, subprocess, sys


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
    h = rows[hi]
    ix = {k: i for i, k in enumerate(h)}
    seen, c = set(), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) != len(h) or r[0] in seen:
            continue
        seen.add(r[0])
        t = r[ix["Source"]].split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        c[op] += num(r[ix["Instructions Executed"]])
    tot = sum(c.values())
    print(f"total warp-instructions {tot:.4g}")
    print("  ".join(f"{k}:{v / tot * 100:.1f}%" for k, v in c.most_common(top)))


if __name__ == "__main__":
    main()
