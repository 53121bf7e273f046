#!/usr/bin/env python3
"""BASELINE config 4: a 1080p synthetic video of 4096 frames, frame-sharded
over the GPUs of one node, maps consumed on the device by the
patch-mean THb trace (timeseries.py:44-73, the pulse-analysis input).

The 102 GB of fp32 frames never exist at once: a pool of one chunk of
device-synthesised frames (4 seeded phantoms per rank, per-frame Philox
noise, oxm_synth_frames_f32) is cycled through the video, as SURVEY.md §8d
allows for config 4.  The timed region is the hybrid path plus the trace
reduction per chunk; input staging is excluded.  Each rank takes a contiguous block of frames
(parallel.shard_range); the step time is the max over ranks.

    python tools/cfg4_video.py [--frames 4096] [--chunk 64]
    torchrun --nproc-per-node N tools/cfg4_video.py      (one process per GPU)
"""
from __future__ import annotations

import argparse
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=4096)
    ap.add_argument("--chunk", type=int, default=64)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import bench
    import paper_1706_07263_b200 as ox
    from paper_1706_07263_b200.parallel import max_over_ranks, shard_range, world
    from paper_1706_07263_b200 import _native
    from paper_1706_07263_b200.device import ptr, stream_handle

    ws, rank, local = world()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if ws > 1 else 0)
    H, W, n = 1080, 1920, 2
    lo, hi = shard_range(args.frames, rank, ws)
    sens, basis = bench.operators()
    eng = ox.HybridMapEngine(sens, basis, ox.PipelineConfig(n_levels=n), device=dev)
    # one chunk of frames, cycled (bench.make_frames: 4 seeded phantoms, per-frame noise)
    pool = bench.make_frames(args.chunk, H, W, 0.3, rank, dev)
    out = eng.allocate(args.chunk, H, W)
    rect = (W // 2 - 32, H // 2 - 32, 64, 64)
    eng.launch(pool, out)  # warm
    torch.cuda.synchronize()
    # per-frame patch sums / counts stay on the device until the end (one sync)
    lib = _native.load()
    nloc = hi - lo
    sums = torch.empty(nloc, dtype=torch.float64, device=dev)
    counts = torch.empty(nloc, dtype=torch.int64, device=dev)
    outs = [out] + ([eng.allocate(args.chunk, H, W)] if nloc > args.chunk else [])
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k, c0 in enumerate(range(0, nloc, args.chunk)):
        nb = min(args.chunk, nloc - c0)
        res = outs[k % len(outs)]
        thb = res.thb[:nb]
        if nb < args.chunk:  # last partial chunk (uneven shards)
            res = eng.allocate(nb, H, W)
            thb = res.thb
        eng.launch(pool[:nb], res)
        st = lib.oxm_patch_mean_f32(ptr(thb), nb, H, W, *rect, ptr(sums[c0:c0 + nb]), ptr(counts[c0:c0 + nb]),
                                    stream_handle())
        _native.check(st, "patch_mean")
    b.record()
    b.synchronize()
    total_ms = a.elapsed_time(b)
    trace = (sums / counts.clamp_min(1)).cpu().numpy().tolist()
    eng.check_flags(out)
    t = max_over_ranks(total_ms * 1e-3, dev)
    if rank == 0:
        print(json.dumps({"config": "cfg4 1080p n=2, 4096-frame synthetic video, frame-sharded",
                          "frames": args.frames, "gpus": ws, "chunk": args.chunk, "seconds": t,
                          "frames_per_s": args.frames / t, "thb_patch_mean_first": trace[:4],
                          "note": "device-synthesised input excluded from the timed region; maps reduced to "
                                  "the patch-mean THb trace on the device"}))
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
