#!/usr/bin/env python3
"""Error of the fp32 per-pixel path WITHOUT the fp64 fixup, binned by the
pixel's smallest reconstructed band (oracle cube), to choose fallback_below.
    python tools/fallback_study.py"""
from __future__ import annotations

import pathlib
import sys

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main() -> None:
    import torch

    import paper_1706_07263_b200 as ox
    from oracle import oximap_oracle as O
    from paper_1706_07263_b200 import fixtures, synth

    sens, basis = fixtures.default_sensitivity(), fixtures.default_basis()
    edges = [0, 1e-6, 1e-4, 1e-3, 2e-3, 5e-3, 1e-2, 2e-2, 5e-2, 1e9]
    cases = [(576, 720, 1, 0.3, s) for s in (0, 1)] + [(1080, 1920, 2, 0.3, 3), (256, 256, 1, 0.3, 6)]
    agg = {}
    for H, W, n, td, seed in cases:
        rgb = synth.phantom_rgb_f32(H, W, seed, sens, basis, texture_density=td)
        ref = O.estimate_frame(rgb, sens.c, basis.xi, n_levels=n, threads=O.default_threads())
        mb = ref["cube"].min(axis=-1)
        # fallback effectively off: threshold at epsilon (the floor the ABI allows)
        eng = ox.HybridMapEngine(sens, basis, ox.PipelineConfig(n_levels=n), fallback_below=1e-6)
        out = eng.run(torch.from_numpy(rgb[None].astype(np.float32)).cuda())
        thb, so2 = out.thb[0].double().cpu().numpy(), out.so2[0].double().cpu().numpy()
        rel = np.abs(thb - ref["thb"]) / np.maximum(np.abs(ref["thb"]), 1e-12)
        ab = np.abs(so2 - ref["so2"])
        for lo, hi in zip(edges[:-1], edges[1:]):
            m = (mb >= lo) & (mb < hi)
            if m.any():
                a = agg.setdefault((lo, hi), [0, 0.0, 0.0])
                a[0] += int(m.sum())
                a[1] = max(a[1], float(np.nanmax(rel[m])))
                a[2] = max(a[2], float(np.nanmax(ab[m])))
    print(f"{'min band in':>22} {'pixels':>9} {'THb max rel':>12} {'SO2 max abs':>12}")
    for (lo, hi), (c, r, a) in sorted(agg.items()):
        print(f"[{lo:8.0e}, {hi:8.0e}) {c:9d} {r:12.3e} {a:12.3e}")


if __name__ == "__main__":
    main()
