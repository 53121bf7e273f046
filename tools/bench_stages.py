#!/usr/bin/env python3
"""Standalone K1 / K2 / K3 / K5 kernels at 1080p (the explicit-transform API
path: haar.forward / haar.inverse / tikhonov_unmix / fit_cube), timed with CUDA
events through the C ABI and scored by achieved HBM GB/s against the measured
copy bandwidth (MEASURED_PEAKS.json), as SURVEY.md §8(d) prescribes for these
stages.  Algorithmic bytes = every input element read once + every output
element written once.  Each launch works on a different one of 8 frames (or
row blocks), so the working set exceeds the 126 MB L2 and the bytes come from
HBM.

    python tools/bench_stages.py [--reps 20]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    import numpy as np
    import torch

    import bench
    from paper_1706_07263_b200 import _native
    from paper_1706_07263_b200.haar import level_dims
    from paper_1706_07263_b200.operators import context
    from paper_1706_07263_b200.pipeline import PipelineConfig, _hybrid_operators

    lib = _native.load()
    dev = torch.device("cuda", 0)
    def S():  # the current stream (a side stream while a CUDA graph is being captured)
        return torch.cuda.current_stream().cuda_stream
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6451.2
    sens, basis = bench.operators()
    H, W, n, C, L, K = 1080, 1920, 2, 3, 26, 8
    frames = bench.make_frames(K, H, W, 0.3, 0, dev).contiguous()
    dims = level_dims(H, W, n)
    nplanes = sum(4 * h * w for h, w in dims)

    def timed(fn, nbytes):
        for i in range(3):
            fn(i % K)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(args.reps):
            fn(i % K)
        b.record()
        b.synchronize()
        t = a.elapsed_time(b) * 1e-3 / args.reps
        rec = {"us": t * 1e6, "bytes": nbytes, "gbs": nbytes / t / 1e9, "frac_hbm": nbytes / t / 1e9 / peak}
        # the same K calls captured once in a CUDA graph and replayed: GPU time
        # without the host's per-call cost (argument checks, launch)
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for i in range(K):
                    fn(i)
            g.replay()
            torch.cuda.synchronize()
            reps = max(1, args.reps // K)
            a.record()
            for _ in range(reps):
                g.replay()
            b.record()
            b.synchronize()
            tg = a.elapsed_time(b) * 1e-3 / (reps * K)
            rec.update({"graph_us": tg * 1e6, "graph_frac_hbm": nbytes / tg / 1e9 / peak})
        except Exception as exc:  # noqa: BLE001 -- report, keep the direct numbers
            rec["graph_error"] = str(exc)[:120]
        torch.cuda.synchronize()
        return rec

    out = {}
    # K1: haar.forward, fp32, 3 channels, n = 2 (all four planes of every level)
    planes = torch.empty((K, nplanes * C), dtype=torch.float32, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    out["K1 haar_forward_f32 1080p n=2 C=3"] = timed(
        lambda i: lib.oxm_haar_forward_f32(frames[i].data_ptr(), H, W, C, n, planes[i].data_ptr(), flags.data_ptr(), S()),
        4 * (H * W * C + nplanes * C))
    # K1 at 4K (BASELINE config 5 frame size, 3 levels): the same kernel on a 4x larger plane
    H4, W4, n4 = 2160, 3840, 3
    dims4 = level_dims(H4, W4, n4)
    np4 = sum(4 * h * w for h, w in dims4)
    f4 = torch.rand((2, H4, W4, C), dtype=torch.float32, device=dev)
    pl4 = torch.empty((2, np4 * C), dtype=torch.float32, device=dev)
    out["K1 haar_forward_f32 4K n=3 C=3"] = timed(
        lambda i: lib.oxm_haar_forward_f32(f4[i % 2].data_ptr(), H4, W4, C, n4, pl4[i % 2].data_ptr(),
                                           flags.data_ptr(), S()),
        4 * (H4 * W4 * C + np4 * C))
    del f4, pl4
    planes64 = torch.empty((2, nplanes * C), dtype=torch.float64, device=dev)
    frames64 = frames[:2].double().contiguous()
    out["K1 haar_forward_f64 1080p n=2 C=3"] = timed(
        lambda i: lib.oxm_haar_forward_f64(frames64[i % 2].data_ptr(), H, W, C, n, planes64[i % 2].data_ptr(),
                                           flags.data_ptr(), S()),
        8 * (H * W * C + nplanes * C))
    del planes64, frames64
    # K2: haar.inverse of a 26-band pyramid (the reference's spectral-domain inverse, pipeline.py:207)
    shapes = []
    prev = (H, W)
    for h, w in dims:
        shapes.append((h, w, prev[0], prev[1]))
        prev = (h, w)
    shp = (ctypes.c_int64 * (4 * n))(*[v for t in shapes for v in t])
    hL, wL = dims[-1]
    ndir = sum(3 * h * w for h, w in dims)
    coarse = torch.rand((K, hL * wL * L), dtype=torch.float32, device=dev)
    dirs = torch.rand((K, ndir * L), dtype=torch.float32, device=dev) - 0.5
    cube = torch.empty((2, H * W * L), dtype=torch.float32, device=dev)
    out["K2 haar_inverse_f32 1080p n=2 C=26"] = timed(
        lambda i: lib.oxm_haar_inverse_f32(coarse[i].data_ptr(), dirs[i].data_ptr(), ctypes.addressof(shp), n, L,
                                           cube[i % 2].data_ptr(), S()),
        4 * (hL * wL * L + ndir * L + H * W * L))
    del dirs, coarse
    # K3: Tikhonov unmix of the directional coefficients (3 -> 26 per coefficient)
    ops = _hybrid_operators(sens, basis, PipelineConfig(n_levels=n))
    solve = np.ascontiguousarray(ops.solve, dtype=np.float64)
    nd = ndir
    rgb = torch.rand((K, nd * 3), dtype=torch.float32, device=dev)
    spec = torch.empty((2, nd * L), dtype=torch.float32, device=dev)
    out["K3 unmix_f32 1.944M dir coeffs -> 26"] = timed(
        lambda i: lib.oxm_unmix_f32(L, solve.ctypes.data, rgb[i].data_ptr(), nd, spec[i % 2].data_ptr(), S()),
        4 * nd * (3 + L))
    del rgb, spec
    # K5: fit_cube of a 1080p 26-band cube -> hbo, hb, offset
    ctx = context(ops, dev.index)
    hbo = torch.empty((3, H * W), dtype=torch.float32, device=dev)
    cube.uniform_(0.05, 0.9)
    out["K5 fit_f32 1080p cube 26 -> 3"] = timed(
        lambda i: lib.oxm_fit_f32(ctx.handle, cube[i % 2].data_ptr(), H * W, 1.0, hbo[0].data_ptr(), hbo[1].data_ptr(),
                                  hbo[2].data_ptr(), S()),
        4 * H * W * (L + 3))
    for k, v in out.items():
        print(json.dumps({"kernel": k, **{a: round(b, 4) if isinstance(b, float) else b for a, b in v.items()},
                          "peak_gbs": peak}))


if __name__ == "__main__":
    main()
