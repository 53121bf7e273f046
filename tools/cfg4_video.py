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
    ap.add_argument("--gather", action="store_true",
                    help="also stream every chunk's THb/SO2 maps to rank 0 (NCCL p2p) and time that run")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    import bench
    import paper_1706_07263_b200 as ox
    from paper_1706_07263_b200.parallel import gather_chunk_to_root, max_over_ranks, shard_range, world
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
    n_chunks = max(-(-(b - a) // args.chunk) for a, b in (shard_range(args.frames, r, ws) for r in range(ws)))

    def run(gather: bool) -> float:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if ws > 1:
            dist.barrier()
        a.record()
        for k in range(n_chunks):  # every rank takes part in every chunk's gather
            c0 = k * args.chunk
            nb = max(0, min(args.chunk, nloc - c0))
            res = outs[k % len(outs)]
            if 0 < nb < args.chunk:  # last partial chunk (uneven shards)
                res = eng.allocate(nb, H, W)
            if nb:
                eng.launch(pool[:nb], res)
                st = lib.oxm_patch_mean_f32(ptr(res.thb), nb, H, W, *rect, ptr(sums[c0:c0 + nb]),
                                            ptr(counts[c0:c0 + nb]), stream_handle())
                _native.check(st, "patch_mean")
            if gather:  # maps of chunk k of every rank to rank 0 over NVLink (NCCL p2p)
                gather_chunk_to_root(res.thb[:nb], args.frames, args.chunk, k)
                gather_chunk_to_root(res.so2[:nb], args.frames, args.chunk, k)
        b.record()
        b.synchronize()
        return max_over_ranks(a.elapsed_time(b) * 1e-3, dev)

    t = run(False)
    tg = run(True) if args.gather else None
    trace = (sums / counts.clamp_min(1)).cpu().numpy().tolist()
    eng.check_flags(out)
    if rank == 0:
        rec = {"config": "cfg4 1080p n=2, 4096-frame synthetic video, frame-sharded",
               "frames": args.frames, "gpus": ws, "chunk": args.chunk, "seconds": t,
               "frames_per_s": args.frames / t, "thb_patch_mean_first": trace[:4],
               "note": "device-synthesised input excluded from the timed region; maps reduced to "
                       "the patch-mean THb trace on the device"}
        if tg is not None:
            rec.update({"gathered_seconds": tg, "gathered_frames_per_s": args.frames / tg,
                        "gather": "every chunk's THb + SO2 maps to rank 0 (gather_chunk_to_root)"})
        print(json.dumps(rec))
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
