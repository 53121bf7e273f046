#!/usr/bin/env python3
"""Randomised parity sweep of the hybrid path against the oracle (GPU box).

Random frame sizes (odd and even, 8..320 px a side), level counts (1..4, as
the frame allows), batch sizes (1..4), texture densities and exposures; each
case runs the fp32 map engine (default EM precision schedule) and the fp64
drop-in estimate_frame, and compares every frame with the oracle
(oracle/oximap_oracle.py, pinned bit-for-bit to the reference):
  * engine: EM fit counts bit-exact, THb <= 1e-4 rel, SO2 <= 1e-5 abs, SO2 NaN
    pattern identical (the north-star tolerances);
  * estimate_frame: cube <= 1e-9 abs, concentrations <= 1e-8 of the map's
    largest magnitude (values reach several hundred g/l in textured frames).
One JSON line per case, then a summary line.

    python tools/parity_fuzz.py [CASES] [SEED] [MAX_SIDE]
"""
from __future__ import annotations

import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def run(cases: int, seed: int, emit=print, max_side: int = 320) -> dict:
    """Run the sweep; emit(json line) per case; returns the summary."""
    import numpy as np
    import torch

    import paper_1706_07263_b200 as ox
    from oracle import oximap_oracle as O
    from paper_1706_07263_b200 import fixtures, synth

    rng = np.random.default_rng(seed)
    dev = torch.device("cuda", 0)
    sens, basis = fixtures.default_sensitivity(), fixtures.default_basis()
    engines = {}
    worst = {"thb_rel": 0.0, "so2_abs": 0.0, "cube_abs": 0.0, "x_abs": 0.0}
    fails = 0
    for case in range(cases):
        H, W = int(rng.integers(8, max_side + 1)), int(rng.integers(8, max_side + 1))
        nmax = max(1, min(4, int(np.floor(np.log2(min(H, W))))))
        n = int(rng.integers(1, nmax + 1))
        B = int(rng.integers(1, 5))
        tex = float(rng.choice([0.0, 0.3, 0.6]))
        gain = float(rng.choice([0.5, 1.0, 1.5]))
        frames = np.stack([synth.phantom_rgb_f32(H, W, int(rng.integers(0, 1 << 30)), sens, basis,
                                                 texture_density=tex) for _ in range(B)])
        frames = (frames * gain).astype(np.float32).astype(np.float64)  # fp32-exact inputs on both sides
        if n not in engines:
            engines[n] = ox.HybridMapEngine(sens, basis, ox.PipelineConfig(n_levels=n), device=dev)
        out = engines[n].run(torch.from_numpy(frames.astype(np.float32)).to(dev), fits=True)
        torch.cuda.synchronize()
        rec = {"case": case, "H": H, "W": W, "n": n, "B": B, "texture": tex, "gain": gain}
        ok = True
        flips = 0
        for b in range(B):
            ref = O.estimate_frame(frames[b], sens.c, basis.xi, n_levels=n)
            thb, so2 = out.thb[b].double().cpu().numpy(), out.so2[b].double().cpu().numpy()
            flips += int(np.sum(out.fits[b].cpu().numpy() != ref["fits"]))
            nz = ref["thb"] != 0
            trel = float(np.max(np.abs(thb - ref["thb"])[nz] / np.abs(ref["thb"])[nz])) if nz.any() else 0.0
            okm = ~np.isnan(ref["so2"])
            sabs = float(np.max(np.abs(so2[okm] - ref["so2"][okm]))) if okm.any() else 0.0
            nan_eq = bool(np.array_equal(np.isnan(so2), np.isnan(ref["so2"])))
            worst["thb_rel"] = max(worst["thb_rel"], trel)
            worst["so2_abs"] = max(worst["so2_abs"], sabs)
            ok &= trel <= 1e-4 and sabs <= 1e-5 and nan_eq
            if b == 0:  # fp64 drop-in on the first frame
                cube, cmap = ox.estimate_frame(ox.RgbImage(frames[b]), sens, basis, ox.PipelineConfig(n_levels=n))
                cabs = float(np.max(np.abs(cube.data - ref["cube"])))
                xabs = float(np.max(np.abs(cmap.stacked() - ref["x"])))
                xrel = xabs / max(float(np.max(np.abs(ref["x"]))), 1.0)
                worst["cube_abs"] = max(worst["cube_abs"], cabs)
                worst["x_abs"] = max(worst["x_abs"], xabs)
                worst["x_rel_of_max"] = max(worst.get("x_rel_of_max", 0.0), xrel)
                ok &= cabs <= 1e-9 and xrel <= 1e-8
                rec.update({"cube_abs": cabs, "x_abs": xabs, "x_rel_of_max": xrel})
        ok &= flips == 0
        rec.update({"fit_count_flips": flips, "max_thb_rel": trel, "max_so2_abs": sabs, "pass": bool(ok)})
        fails += not ok
        emit(json.dumps(rec))
    summary = {"summary": True, "cases": cases, "failed": fails, "worst": worst}
    emit(json.dumps(summary))
    return summary


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 2024
    max_side = int(sys.argv[3]) if len(sys.argv) > 3 else 320
    run(cases, seed, emit=lambda line: print(line, flush=True), max_side=max_side)


if __name__ == "__main__":
    main()
