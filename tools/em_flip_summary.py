#!/usr/bin/env python3
"""Summarise tools/em_flip_study.py output: per schedule, seeds, coefficients,
fit-count flips against the all-fp64 schedule, median us/frame per stage,
restarts per 64-frame batch; then every flip with its replayed rel/tol history.
    python tools/em_flip_summary.py STUDY.jsonl [...]"""
import collections
import json
import statistics
import sys


def main():
    for path in sys.argv[1:]:
        recs = [json.loads(l) for l in open(path) if l.startswith("{")]
        runs = [r for r in recs if "flip" not in r]
        flips = [r for r in recs if "flip" in r]
        seeds = sorted({r["seed"] for r in runs})
        print(f"== {path}: seeds {seeds[0]}..{seeds[-1]} ({len(seeds)} x 64 textured 1080p frames, "
              f"{len(seeds) * 8294400} low-pass coefficients per schedule)")
        print(f"{'schedule':14s} {'flips':>5s} {'us/frame':>9s}  {'ll / lead / tail / px / fixup':32s} {'restarts':>9s}")
        agg = collections.defaultdict(list)
        for r in runs:
            agg[r["schedule"]].append(r)
        for k, rs in agg.items():
            st = [statistics.median(x["us"][i] for x in rs) for i in range(5)]
            print(f"{k:14s} {sum(x.get('flips', 0) for x in rs):5d} {statistics.median(x['total_us'] for x in rs):9.2f}  "
                  f"{' / '.join(f'{v:.2f}' for v in st):32s} {sum(x['restarts'] for x in rs) // len(rs):9d}")
        for f in flips:
            print(f"  flip: schedule {f['schedule']} seed {f['seed']} fits ref {f['fits_ref']} got {f['fits_test']} "
                  f"|x| {f['xnorm']:.1f} last rel/tol {f['rel_over_tol_last']}")


if __name__ == "__main__":
    main()
