#!/usr/bin/env python3
"""Do co-resident batches on two streams beat back-to-back batches?

The EM lead-in is MUFU-bound, the EM tail fp64-pipe-bound and the per-pixel
stage MUFU-bound; if warps of different stages shared an SM, their pipes
could overlap.  Two engines (two workspaces) run alternate 32-frame batches
on two streams through oxm_hybrid_maps_f32_split (per-pixel stage on the same
stream), the persistent EM kernels leaving `reserve` CTA slots per SM free
for the other stream's kernels; stream B starts `offset` stages behind.
Reported: us per frame against the same batches back to back on one stream.

    python tools/costream_probe.py
"""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import torch

    import bench
    import paper_1706_07263_b200 as ox
    from paper_1706_07263_b200 import _native
    from paper_1706_07263_b200.device import ptr

    dev = torch.device("cuda", 0)
    sens, basis = bench.operators()
    B, H, W, n, NB = 32, 1080, 1920, 2, 8
    engs = [ox.HybridMapEngine(sens, basis, ox.PipelineConfig(n_levels=n), device=dev) for _ in range(2)]
    frames = [bench.make_frames(B, H, W, 0.3, r, dev) for r in range(2)]
    outs = [e.allocate(B, H, W) for e in engs]
    nbytes = engs[0].workspace_bytes(B, H, W)
    ws = [torch.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(2)]
    lib = _native.load()
    streams = [torch.cuda.Stream(device=dev) for _ in range(2)]

    def split(i, s, reserve):
        e, o = engs[i], outs[i]
        rc = lib.oxm_hybrid_maps_f32_split(e.ctx.handle, ptr(frames[i]), B, H, W, n, 1.0, ptr(ws[i]), nbytes,
                                           ptr(o.thb), ptr(o.so2), None, None, None, None, ptr(o.flags),
                                           s.cuda_stream, s.cuda_stream, int(reserve))
        _native.check(rc, "split")

    def timeit(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) * 1e3 / reps / (NB * B)

    cur = torch.cuda.current_stream()

    def sequential():
        for k in range(NB):
            engs[k % 2].launch(frames[k % 2], outs[k % 2])

    ref = [o.thb.clone() for o in outs]
    print(json.dumps({"mode": "sequential", "us_per_frame": timeit(sequential)}), flush=True)
    ref = [o.thb.clone() for o in outs]

    for reserve in (0, 1, 2):
        def two_streams():
            for s in streams:
                s.wait_stream(cur)
            for k in range(NB):
                split(k % 2, streams[k % 2], reserve)
            for s in streams:
                cur.wait_stream(s)

        us = timeit(two_streams)
        torch.cuda.synchronize()
        same = all(torch.equal(o.thb, r) for o, r in zip(outs, ref))
        print(json.dumps({"mode": "two streams", "reserve": reserve, "us_per_frame": us, "bitwise_same": same}),
              flush=True)


if __name__ == "__main__":
    main()
