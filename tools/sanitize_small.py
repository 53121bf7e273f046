#!/usr/bin/env python3
"""Small run over every kernel family, for compute-sanitizer memcheck/racecheck."""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    import __graft_entry__
    import paper_1706_07263_b200 as ox
    from paper_1706_07263_b200 import fixtures, synth

    __graft_entry__.smoke()
    sens, basis = fixtures.default_sensitivity(), fixtures.default_basis()
    rng = np.random.default_rng(0)
    for shape, n in [((37, 23, 3), 2), ((9, 15), 5), ((64, 48, 26), 4)]:
        img = rng.normal(size=shape)
        assert np.max(np.abs(ox.inverse(ox.forward(img, n)) - img)) < 1e-12
    # TMA paths: K1 tiles in/out (3-channel planes with 16-byte rows, fp32 and fp64,
    # partial tiles), K5 bulk-copied slabs (>= 128 pixels), the TMA low-pass kernel
    from paper_1706_07263_b200.haar import pyramid_device

    for dt in (torch.float32, torch.float64):
        pyramid_device(torch.from_numpy(rng.uniform(0, 1, (70, 100, 3))).to("cuda", dt), 2)
        pyramid_device(torch.from_numpy(rng.uniform(0, 1, (37, 36, 3))).to("cuda", dt), 3)
    ox.fit_concentration(rng.uniform(0.1, 1, (300, 26)), basis)
    import os

    os.environ["OXM_LL_TMA"] = "1"
    for n in (1, 2):
        e = ox.HybridMapEngine(sens, basis, ox.PipelineConfig(n_levels=n))
        e.run(torch.from_numpy(synth.phantom_rgb_f32(46, 68, 3, sens, basis)[None].astype(np.float32)).cuda())
    os.environ["OXM_LL_TMA"] = "0"
    op = ox.TikhonovOperator.from_relative(sens, 1e-3)
    ox.tikhonov_unmix(rng.uniform(0, 1, (100, 3)), op)
    ox.estimate_lowpass(ox.LowPassBlock(rng.uniform(0.1, 1, (5, 7, 3)), 2.0), sens, basis, ox.BayesConfig(), op)
    ox.expectation_step(rng.uniform(0.1, 1, (4, 3)), rng.uniform(0.1, 1, (4, 26)), sens, ox.BayesConfig())
    ox.fit_concentration(rng.uniform(0.1, 1, (10, 26)), basis)
    ox.expected_spectrum(rng.uniform(0, 5, (10, 3)), basis)
    for mode in ("hybrid", "tikhonov_only", "bayes_only"):
        ox.estimate_frame(ox.RgbImage(synth.phantom_rgb_f32(33, 41, 1, sens, basis)), sens, basis,
                          ox.PipelineConfig(mode=mode, n_levels=2))
    rgb = synth.phantom_rgb_f32(70, 97, 2, sens, basis)
    for n in (1, 2, 3, 4):
        eng = ox.HybridMapEngine(sens, basis, ox.PipelineConfig(n_levels=n))
        eng.run(torch.from_numpy(rgb[None].astype(np.float32)).cuda(), planes=True, fits=True)
        counts = np.clip(np.round(rgb / (rgb.max() / 65535)), 0, 65535).astype(np.uint16)
        eng.run(torch.from_numpy(counts[None]).cuda(), scale=float(rgb.max() / 65535), big_endian=False)
    torch.cuda.synchronize()
    print("sanitize run ok")


if __name__ == "__main__":
    main()
