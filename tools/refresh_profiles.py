#!/usr/bin/env python3
"""Regenerate profiles/ summaries from the latest ncu captures.
    python tools/refresh_profiles.py FULL.ncu-rep LAUNCHES.csv BENCH.log FRAMES_PER_PROFILED_LAUNCH"""
import collections, csv, pathlib, shutil, subprocess, sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
P = ROOT / "profiles"


def launches(path: str) -> str:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    data = [r for r in rows[1:] if r[ix["Metric Name"]] == "gpu__time_duration.sum"]
    agg = collections.defaultdict(list)
    for r in data:
        agg[r[ix["Kernel Name"]].split("(")[0]].append(float(r[ix["Metric Value"]]))
    ours = {k: v for k, v in agg.items()
            if "oxm::" in k and not any(x in k for x in ("probe", "synth_kernel", "patch_mean", "pack_hwc3"))}
    tot = sum(sum(v) for v in ours.values())
    out = ["ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu",
           "(cold-cache, serialised launches: compare SHARES; batch = 64 frames 1080p n=2;",
           " untimed input staging (synth_kernel) and the roofline probes excluded)",
           f"{'kernel (hot path only)':70s} {'n':>3} {'mean ns':>12} {'share':>7}"]
    for k, v in sorted(ours.items(), key=lambda x: -sum(x[1])):
        out.append(f"{k[-70:]:70s} {len(v):3d} {sum(v) / len(v):12.1f} {100 * sum(v) / tot:6.1f}%")
    return "\n".join(out) + "\n"


def main():
    rep, lcsv, bench, frames = sys.argv[1:5]
    tag = "r01"
    (P / f"{tag}_launches.txt").write_text(launches(lcsv))
    summ = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), rep], capture_output=True, text=True).stdout
    for k in ("em_lead", "em_persistent", "em_exact", "px_f32", "px_fallback", "ll_kernel"):
        summ += f"== opcode mix {k}\n" + subprocess.run(
            [sys.executable, str(ROOT / "tools" / "ncu_opmix.py"), rep, k, "--top", "16"], capture_output=True, text=True).stdout
    (P / f"{tag}_ncu_summary.txt").write_text(f"source: {rep} (tools/profile_hybrid.py, {frames} frames per launch)\n" + summ)
    subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_traffic.py"), rep, frames], check=True, capture_output=True)
    shutil.copy(bench, P / f"{tag}_bench.jsonl")
    print((P / f"{tag}_launches.txt").read_text())


if __name__ == "__main__":
    main()
