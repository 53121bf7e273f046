#!/usr/bin/env python3
"""Per-opcode dynamic SASS counts of one kernel in an ncu report (thread- and
warp-level), per unit of work, and the fp64-pipe total bench.py uses as the EM
tail's work per fit (DFMA + DADD + DMUL + DSETP thread instructions / fits).

    python tools/ncu_thread_counts.py rep.ncu-rep kernel_regex UNITS [--top N]
"""
import collections
import csv
import io
import subprocess
import sys

FP64_PIPE = ("DFMA", "DADD", "DMUL", "DSETP")


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def counts(rep: str, kern: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--launch-count", "1",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
    h = rows[hi]
    ix = {k: i for i, k in enumerate(h)}
    seen, thr, warp = set(), collections.Counter(), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) != len(h) or r[0] in seen:
            continue
        seen.add(r[0])
        t = r[ix["Source"]].split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        thr[op] += num(r[ix["Thread Instructions Executed"]])
        warp[op] += num(r[ix["Instructions Executed"]])
    return thr, warp


def main():
    rep, kern, units = sys.argv[1], sys.argv[2], float(sys.argv[3])
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 26
    thr, warp = counts(rep, kern)
    print(f"{'opcode':8s} {'thread-instructions':>20s} {'per-unit':>9s} {'warp-instructions':>18s}")
    for op, v in thr.most_common(top):
        print(f"{op:8s} {v:20.0f} {v / units:9.2f} {warp[op]:18.0f}")
    fp64 = sum(thr[o] for o in FP64_PIPE) / units
    print(f"total thread-instructions per unit {sum(thr.values()) / units:.1f}; "
          f"fp64 pipe (DFMA+DADD+DMUL+DSETP) per unit {fp64:.1f}; "
          f"flops per unit (FMA = 2) {(2 * thr['DFMA'] + thr['DADD'] + thr['DMUL']) / units:.1f}")


if __name__ == "__main__":
    main()
