#!/usr/bin/env python3
"""Regenerate profiles/ summaries from the latest ncu captures.
    python tools/refresh_profiles.py FULL.ncu-rep LAUNCHES.csv BENCH.log FRAMES_PER_PROFILED_LAUNCH [TAG]"""
import collections, csv, pathlib, shutil, subprocess, sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
P = ROOT / "profiles"


def launches(path: str) -> str:
    """Kernel shares of the two timed bench steps: the launch list is cut into
    steps at each zero_counters launch (step 1 = the warm-up launch; later
    groups -- gathered leg, e2e, schedule check -- are not the timed steps)."""
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    data = [r for r in rows[1:] if r[ix["Metric Name"]] == "gpu__time_duration.sum"]
    steps, cur = [], None
    for r in data:
        name = r[ix["Kernel Name"]].split("(")[0]
        if "zero_counters" in name:
            cur = []
            steps.append(cur)
        if cur is not None and "oxm::" in name:
            cur.append((name, float(r[ix["Metric Value"]])))
    timed = steps[1:3]
    agg = collections.defaultdict(list)
    for st in timed:
        for name, t in st:
            agg[name].append(t)
    tot = sum(sum(v) for v in agg.values())
    out = ["ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py --steps 2 --warmup 1 --no-cpu --no-dropin",
           "(cold-cache, serialised launches: compare SHARES; the two timed steps of the bench batch (1080p n=2), cut at",
           " zero_counters; warm-up, input staging, gathered leg, e2e and the schedule check excluded)",
           f"{'kernel':70s} {'n':>3} {'mean ns':>12} {'share':>7}"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append(f"{k[-70:]:70s} {len(v):3d} {sum(v) / len(v):12.1f} {100 * sum(v) / tot:6.1f}%")
    out.append(f"total per step: {tot / len(timed) / 1e3:.1f} us")
    return "\n".join(out) + "\n"


def main():
    rep, lcsv, bench, frames = sys.argv[1:5]
    tag = sys.argv[5] if len(sys.argv) > 5 else "r02"
    (P / f"{tag}_launches.txt").write_text(launches(lcsv))
    summ = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), rep], capture_output=True, text=True).stdout
    for k in ("em_lead", "em_persistent", "px_f32", "px_fallback", "ll_kernel"):
        summ += f"== opcode mix {k}\n" + subprocess.run(
            [sys.executable, str(ROOT / "tools" / "ncu_opmix.py"), rep, k, "--top", "16"], capture_output=True, text=True).stdout
    (P / f"{tag}_ncu_summary.txt").write_text(f"source: {rep} (tools/profile_hybrid.py, {frames} frames per launch)\n" + summ)
    subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_traffic.py"), rep, frames], check=True, capture_output=True)
    shutil.copy(bench, P / f"{tag}_bench.jsonl")
    print((P / f"{tag}_launches.txt").read_text())


if __name__ == "__main__":
    main()
