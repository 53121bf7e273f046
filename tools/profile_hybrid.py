#!/usr/bin/env python3
"""Minimal driver for ncu: a few launches of the fused hybrid path on a
1080p batch (same kernels and shapes as bench.py, fewer frames).

    python tools/profile_hybrid.py [--batch 4] [--launches 2] [--levels 2]
"""

from __future__ import annotations

import argparse
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main() -> None:
    p = argparse.ArgumentParser()
    p.add_argument("--batch", type=int, default=4)
    p.add_argument("--launches", type=int, default=2)
    p.add_argument("--levels", type=int, default=2)
    p.add_argument("--height", type=int, default=1080)
    p.add_argument("--width", type=int, default=1920)
    p.add_argument("--texture", type=float, default=0.3)
    a = p.parse_args()
    import torch

    import bench
    import paper_1706_07263_b200 as ox

    dev = torch.device("cuda", 0)
    sens, basis = bench.operators()
    eng = ox.HybridMapEngine(sens, basis, ox.PipelineConfig(n_levels=a.levels), device=dev)
    frames = bench.make_frames(a.batch, a.height, a.width, a.texture, 0, dev)
    out = eng.allocate(a.batch, a.height, a.width, fits=True)
    for _ in range(a.launches):
        eng.launch(frames, out)
    torch.cuda.synchronize()
    eng.check_flags(out)
    print("ok", float(out.thb.float().mean()), int(out.fits.sum()))


if __name__ == "__main__":
    main()
