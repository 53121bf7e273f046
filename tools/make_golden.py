#!/usr/bin/env python3
"""Generate tests/golden/*.npz by running the REFERENCE implementation.

Run in the build container only (it imports /root/reference/pkg/src, which
does not exist on the GPU box):   python tools/make_golden.py
The fixtures pin the CPU oracle (oracle/oximap_oracle.py) bit-for-bit and
give the GPU parity tests reference outputs without the reference present.
All RGB inputs are rounded to float32-representable values first (SURVEY.md
§8c tolerance protocol) so the fp32 GPU path sees the same numbers.
"""

from __future__ import annotations

import pathlib
import sys

import numpy as np

REF = pathlib.Path("/root/reference/pkg/src")
OUT = pathlib.Path(__file__).resolve().parents[1] / "tests" / "golden"


def main() -> None:
    sys.path.insert(0, str(REF))
    from oximap import fixtures, haar, pipeline, synth
    from oximap.bayes import BayesConfig, LowPassBlock, estimate_lowpass, fit_concentration
    from oximap.core import RgbImage, SpectralCube, WavelengthGrid
    from oximap.unmix import TikhonovOperator, tikhonov_unmix

    OUT.mkdir(parents=True, exist_ok=True)
    sens, basis = fixtures.default_sensitivity(), fixtures.default_basis()
    op = TikhonovOperator.from_relative(sens, 1e-3)

    # ---- operators (26-band default grid + a 55-band grid)
    g55 = WavelengthGrid(440.0, 5.0, 55)
    np.savez_compressed(
        OUT / "operators.npz",
        c=sens.c, xi=basis.xi, solve=op.solve, gamma=op.gamma,
        c55=fixtures.default_sensitivity(g55).c, xi55=fixtures.default_basis(g55).xi,
    )

    rng = np.random.default_rng(20240817)

    # ---- Haar: forward planes + inverse for assorted shapes / levels / channels
    haar_cases = {}
    shapes = [((2, 2), 1), ((3, 5), 1), ((6, 8), 1), ((4, 4), 2), ((40, 40), 3), ((33, 21), 3),
              ((1, 1), 2), ((9, 15, 3), 2), ((64, 64, 3), 1), ((32, 48, 3), 3), ((17, 29, 26), 2),
              ((50, 70, 3), 5)]
    for i, (shape, n) in enumerate(shapes):
        img = rng.normal(size=shape)
        pyr = haar.forward(img, n)
        haar_cases[f"img{i}"] = img
        haar_cases[f"n{i}"] = np.array(n)
        for k, lv in enumerate(pyr.levels):
            for name in ("lp", "dh", "dv", "dd"):
                haar_cases[f"c{i}_l{k}_{name}"] = getattr(lv, name)
            haar_cases[f"c{i}_l{k}_orig"] = np.array(lv.orig_shape)
        haar_cases[f"inv{i}"] = haar.inverse(pyr)
    np.savez_compressed(OUT / "haar.npz", count=len(shapes), **haar_cases)

    # ---- Tikhonov unmix
    rgb = rng.uniform(-1.0, 2.0, size=(257, 3))
    np.savez_compressed(OUT / "unmix.npz", rgb=rgb, out=tikhonov_unmix(rgb, op))

    # ---- EM on low-pass data of phantom frames + random pixels
    em = {}
    for j, (H, W, n, td, seed) in enumerate([(64, 96, 1, 0.3, 11), (96, 64, 2, 0.0, 12)]):
        spec = synth.tissue_phantom_spec(H, W, seed=seed, texture_density=td)
        _, _, rgbf = synth.generate_phantom(spec, sens, basis)
        lp = haar.forward(rgbf.data.astype(np.float32).astype(np.float64), n).residual_lp
        spectra, cmap = estimate_lowpass(LowPassBlock(lp, 2.0**n), sens, basis, BayesConfig(), op)
        em[f"lp{j}"], em[f"scale{j}"] = lp, np.array(2.0**n)
        em[f"spectra{j}"], em[f"x{j}"] = spectra, cmap.stacked()
    x0 = np.column_stack([rng.uniform(5, 60, 100), rng.uniform(5, 60, 100), rng.uniform(-0.2, 0.2, 100)])
    y = np.exp(-(x0 @ basis.xi.T)) @ sens.c.T
    spectra, cmap = estimate_lowpass(LowPassBlock(y.reshape(1, 100, 3), 1.0), sens, basis, BayesConfig(), op)
    em["lp2"], em["scale2"], em["spectra2"], em["x2"] = y.reshape(1, 100, 3), np.array(1.0), spectra, cmap.stacked()
    # non-default knobs: beta, max_iters, rel_tol, epsilon
    cfg = BayesConfig(beta=0.5, max_iters=7, rel_tol=1e-6, epsilon=1e-4)
    spectra, cmap = estimate_lowpass(LowPassBlock(y.reshape(10, 10, 3), 1.0), sens, basis, cfg, op)
    em["lp3"], em["scale3"], em["spectra3"], em["x3"] = y.reshape(10, 10, 3), np.array(1.0), spectra, cmap.stacked()
    em["cfg3"] = np.array([cfg.beta, cfg.max_iters, cfg.rel_tol, cfg.epsilon])
    np.savez_compressed(OUT / "em.npz", count=4, **em)

    # ---- fit_concentration
    sp = rng.uniform(1e-8, 1.2, size=(300, 26))
    np.savez_compressed(OUT / "fit.npz", spectra=sp, x=fit_concentration(sp, basis))

    # ---- full frames (estimate_frame), all RGB modes
    frames = {}
    cases = [
        ("hybrid", 32, 48, 1, 0.3, 1, True),
        ("hybrid", 37, 23, 2, 0.3, 2, True),
        ("hybrid", 45, 70, 3, 0.3, 3, True),
        ("hybrid", 64, 64, 2, 0.0, 4, True),
        ("hybrid", 9, 15, 1, 0.0, 5, True),
        ("hybrid", 256, 256, 1, 0.3, 6, False),  # BASELINE config 1
        ("tikhonov_only", 24, 20, 2, 0.3, 7, True),
        ("bayes_only", 12, 10, 1, 0.3, 8, True),
    ]
    for i, (mode, H, W, n, td, seed, keep_cube) in enumerate(cases):
        spec = synth.tissue_phantom_spec(H, W, seed=seed, texture_density=td)
        _, _, rgbf = synth.generate_phantom(spec, sens, basis)
        data = rgbf.data.astype(np.float32).astype(np.float64)
        stats = {}
        cube, cmap = pipeline.estimate_frame(
            RgbImage(data), sens, basis, pipeline.PipelineConfig(mode=mode, n_levels=n), stats=stats
        )
        frames[f"rgb{i}"] = data
        frames[f"meta{i}"] = np.array([H, W, n, stats["bayes_coefficients"], stats["tikhonov_coefficients"]])
        frames[f"mode{i}"] = np.array(mode)
        frames[f"x{i}"] = cmap.stacked()
        frames[f"thb{i}"], frames[f"so2{i}"] = cmap.thb, cmap.sat_o2
        if keep_cube:
            frames[f"cube{i}"] = cube.data
    np.savez_compressed(OUT / "frames.npz", count=len(cases), **frames)
    for p in sorted(OUT.glob("*.npz")):
        print(f"{p.name}: {p.stat().st_size / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
