"""GPU parity of the individual kernels (K1-K5) through the drop-in API and
the C ABI, against golden reference vectors and the CPU oracle.  Known-answer
tests follow the reference's own tests (pkg/tests/test_haar.py,
test_unmix.py, test_bayes.py)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_1706_07263_b200 as ox
from oracle import oximap_oracle as O

pytestmark = pytest.mark.gpu


# ---------------------------------------------------------------- K1 / K2 Haar
def test_haar_forward_inverse_fp64_bitwise(cuda, golden):
    g = golden("haar")
    for i in range(int(g["count"])):
        img, n = g[f"img{i}"], int(g[f"n{i}"])
        pyr = ox.forward(img, n)
        for k, lv in enumerate(pyr.levels):
            for name in ("lp", "dh", "dv", "dd"):
                assert np.array_equal(getattr(lv, name), g[f"c{i}_l{k}_{name}"]), (i, k, name)
            assert tuple(lv.orig_shape) == tuple(g[f"c{i}_l{k}_orig"])
        assert np.array_equal(ox.inverse(pyr), g[f"inv{i}"]), i


def test_haar_fp32_within_1e6_of_plane_max(cuda, rng):
    from paper_1706_07263_b200.haar import inverse_device, pyramid_device

    for shape, n in [((1080, 1920, 3), 2), ((576, 720, 3), 1), ((333, 257, 3), 3), ((64, 48, 26), 4)]:
        img = rng.uniform(0.0, 8.0, size=shape).astype(np.float32)
        ref = O.haar_forward(img.astype(np.float64), n)
        levels = pyramid_device(torch.from_numpy(img).to(cuda), n)
        for (quad, oshape), lv in zip(levels, ref):
            assert tuple(oshape) == tuple(lv["orig_shape"])
            for p, name in zip(quad, ("lp", "dh", "dv", "dd")):
                got = p.double().cpu().numpy()
                want = lv[name]
                assert np.max(np.abs(got - want)) <= 1e-6 * max(np.max(np.abs(want)), 1e-30), (shape, name)
        # fp32 inverse of the fp32 pyramid reconstructs the image
        dirs = torch.cat([q.reshape(-1) for (quad, _) in levels for q in quad[1:]])
        shapes = [(q[0].shape[0], q[0].shape[1], o[0], o[1]) for (q, o) in levels]
        rec = inverse_device(levels[-1][0][0], dirs, shapes, shape[2]).cpu().numpy()
        assert np.max(np.abs(rec - img)) <= 1e-5 * np.max(np.abs(img))


def test_haar_tma_tiles_fp64_bitwise(cuda, rng):
    """RGB planes whose rows are 16-byte multiples take the TMA-tiled K1
    (haar_fwd_tma_kernel): bit-identical to the oracle (= the reference) in
    fp64, including edge tiles with per-level replication (odd heights, a
    width that is not a tile multiple) and the chained second pass (n = 5);
    non-finite samples anywhere in a tile -- interior, right / bottom edge --
    raise like haar.py:133-134."""
    for shape, n in [((1083, 1922, 3), 3), ((270, 482, 3), 2), ((99, 130, 3), 1), ((150, 202, 3), 5)]:
        img = rng.normal(size=shape)
        pyr = ox.forward(img, n)
        ref = O.haar_forward(img, n)
        for lv, rl in zip(pyr.levels, ref):
            for name in ("lp", "dh", "dv", "dd"):
                assert np.array_equal(getattr(lv, name), rl[name]), (shape, n, name)
    for (r, c) in [(40, 37), (269, 483), (0, 0), (133, 300)]:
        bad = rng.normal(size=(270, 484, 3))
        bad[r, c, 1] = np.nan if r % 2 else np.inf
        from paper_1706_07263_b200.haar import pyramid_device

        with pytest.raises(ox.ArgumentError):
            pyramid_device(torch.from_numpy(bad).to(cuda), 2)
        with pytest.raises(ox.ArgumentError):
            pyramid_device(torch.from_numpy(bad.astype(np.float32)).to(cuda), 2)
    huge = np.full((64, 64, 3), 3.0e38, dtype=np.float32)  # finite, but an fp32 window sum overflows
    from paper_1706_07263_b200.haar import pyramid_device

    pyramid_device(torch.from_numpy(huge).to(cuda), 2)  # must not raise


def test_haar_kats(cuda, rng):
    lv = ox.forward(np.full((2, 2), 3.5), 1).levels[0]
    assert lv.lp.shape == (1, 1) and lv.lp[0, 0] == 7.0
    assert lv.dh[0, 0] == lv.dv[0, 0] == lv.dd[0, 0] == 0.0
    # window == matrix product (test_haar.py:36-49)
    x = rng.normal(size=(6, 8))
    lvl = ox.forward(x, 1).levels[0]
    h = ox.haar_matrix()
    for wy in range(3):
        for wx in range(4):
            win = np.array([x[2 * wy, 2 * wx], x[2 * wy, 2 * wx + 1], x[2 * wy + 1, 2 * wx], x[2 * wy + 1, 2 * wx + 1]])
            got = [lvl.lp[wy, wx], lvl.dh[wy, wx], lvl.dv[wy, wx], lvl.dd[wy, wx]]
            assert np.allclose(got, win @ h, atol=1e-14)
    # Parseval per level, linearity, positivity
    x = rng.normal(size=(32, 48, 3))
    plane = x
    for lev in ox.forward(x, 3).levels:
        e_out = sum(np.sum(p**2) for p in (lev.lp, lev.dh, lev.dv, lev.dd))
        assert e_out == pytest.approx(np.sum(plane**2), rel=1e-10)
        plane = lev.lp
    pos = ox.forward(rng.uniform(0.0, 4.0, size=(33, 21)), 3)
    assert all(np.all(lev.lp >= 0) for lev in pos.levels)
    # one pixel, two levels
    pyr = ox.forward(np.array([[2.0]]), 2)
    assert pyr.residual_lp.shape == (1, 1) and np.allclose(ox.inverse(pyr), [[2.0]])


def test_haar_errors(cuda):
    bad = np.ones((4, 4))
    bad[1, 1] = np.inf
    with pytest.raises(ox.ArgumentError):
        ox.forward(bad, 1)
    with pytest.raises(ox.ArgumentError):
        ox.forward(np.ones((4, 4)), 0)
    with pytest.raises(ox.ArgumentError):
        ox.forward(np.ones((0, 4)), 1)
    pyr = ox.forward(np.random.default_rng(0).normal(size=(8, 8)), 1)
    lv = pyr.levels[0]
    with pytest.raises(ox.DataError):
        ox.inverse(ox.HaarPyramid(levels=(ox.HaarLevel(lp=lv.lp, dh=lv.dh[:2], dv=lv.dv, dd=lv.dd, orig_shape=lv.orig_shape),)))


def test_haar_inverse_assembled_pyramid(cuda, rng):
    # finer levels without lp, as the hybrid path assembles them (pipeline.py:203-206)
    x = rng.normal(size=(37, 23, 5))
    pyr = ox.forward(x, 3)
    bare = tuple(ox.HaarLevel(lp=None if k < 2 else lv.lp, dh=lv.dh, dv=lv.dv, dd=lv.dd, orig_shape=lv.orig_shape)
                 for k, lv in enumerate(pyr.levels))
    rec = ox.inverse(ox.HaarPyramid(levels=bare))
    assert np.max(np.abs(rec - x)) <= 1e-12


# ---------------------------------------------------------------- K3 unmix
def test_tikhonov_unmix(cuda, golden, sensitivity):
    g = golden("unmix")
    op = ox.TikhonovOperator.from_relative(sensitivity, 1e-3)
    got = ox.tikhonov_unmix(g["rgb"], op)
    assert np.max(np.abs(got - g["out"])) <= 1e-14 * np.max(np.abs(g["out"]))
    assert ox.tikhonov_unmix(np.zeros(3), op).shape == (26,)
    assert np.array_equal(ox.tikhonov_unmix(np.zeros(3), op), np.zeros(26))


def test_unmix_dense_oracles(cuda, rng):
    from paper_1706_07263_b200 import CameraSensitivity, WavelengthGrid

    for L in (4, 8, 16, 26, 40):
        sens = CameraSensitivity(WavelengthGrid(450.0, 5.0, L), rng.uniform(0.05, 1.0, size=(3, L)))
        y = rng.normal(size=3)
        assert np.max(np.abs(ox.lsq_unmix(y, sens) - np.linalg.pinv(sens.c) @ y)) <= 1e-9
        gamma = 10 ** rng.uniform(-6, -1)
        a = np.vstack([sens.c, np.sqrt(gamma) * np.eye(L)])
        b = np.concatenate([y, np.zeros(L)])
        oracle = np.linalg.lstsq(a, b, rcond=None)[0]
        assert np.max(np.abs(ox.tikhonov_unmix(y, ox.TikhonovOperator.build(sens, gamma)) - oracle)) <= 1e-9


def test_unmix_commutes_with_transform(cuda, rng, sensitivity):
    frame = rng.uniform(0.05, 1.0, size=(24, 20, 3))
    op = ox.TikhonovOperator.from_relative(sensitivity, 1e-3)
    spec = ox.forward(ox.tikhonov_unmix(frame, op), 2)
    pyr = ox.forward(frame, 2)
    for ls, lr in zip(spec.levels, pyr.levels):
        for name in ("lp", "dh", "dv", "dd"):
            assert np.max(np.abs(getattr(ls, name) - ox.tikhonov_unmix(getattr(lr, name), op))) <= 1e-10
    out = ox.unmix_pyramid_directional(pyr, op)
    assert out.residual_lp is pyr.residual_lp
    assert out.levels[0].dh.shape == pyr.levels[0].dh.shape[:2] + (26,)


def test_unmix_fp32(cuda, rng, sensitivity):
    from paper_1706_07263_b200.unmix import apply_matrix_device

    op = ox.TikhonovOperator.from_relative(sensitivity, 1e-3)
    rgb = rng.uniform(-1, 3, size=(100_003, 3)).astype(np.float32)
    got = apply_matrix_device(torch.from_numpy(rgb).to(cuda), op.solve).cpu().numpy()
    want = rgb.astype(np.float64) @ op.solve.T
    assert np.max(np.abs(got - want)) <= 1e-6 * np.max(np.abs(want))


# ---------------------------------------------------------------- K4 EM
def _oracle_fits(lp, scale, cfg_kw=None):
    g = np.load(__import__("pathlib").Path(__file__).parent / "golden" / "operators.npz")
    return O.estimate_lowpass(lp, scale, g["c"], g["xi"], g["solve"], **(cfg_kw or {}))


def test_em_matches_reference(cuda, golden, sensitivity, basis):
    g = golden("em")
    op = ox.TikhonovOperator.from_relative(sensitivity, 1e-3)
    for j in range(int(g["count"])):
        cfg, kw = ox.BayesConfig(), {}
        if f"cfg{j}" in g:
            beta, iters, tol, eps = g[f"cfg{j}"]
            cfg = ox.BayesConfig(beta=beta, max_iters=int(iters), rel_tol=tol, epsilon=eps)
            kw = dict(beta=beta, max_iters=int(iters), rel_tol=tol, eps=eps)
        block = ox.LowPassBlock(g[f"lp{j}"], float(g[f"scale{j}"]))
        spectra, cmap, fits = ox.estimate_lowpass_fits(block, sensitivity, basis, cfg, op)
        ref_s, ref_x = g[f"spectra{j}"], g[f"x{j}"]
        assert np.max(np.abs(spectra - ref_s) / np.maximum(np.abs(ref_s), 1e-3)) <= 1e-9, j
        assert np.max(np.abs(cmap.stacked() - ref_x)) <= 1e-8, j
        # discrete decision: fit counts bit-exact vs the pinned oracle
        _, _, ofits = _oracle_fits(g[f"lp{j}"], float(g[f"scale{j}"]), kw)
        assert np.array_equal(fits, ofits), (j, np.sum(fits != ofits))


def test_em_kats(cuda, sensitivity, basis, rng):
    op = ox.TikhonovOperator.from_relative(sensitivity, 1e-3)
    cfg = ox.BayesConfig()
    # constant phantom within 1 % (test_bayes.py:128-135)
    x0 = np.array([40.0, 40.0, 0.0])
    y = sensitivity.c @ np.exp(-(basis.xi @ x0))
    _, cmap = ox.estimate_lowpass(ox.LowPassBlock(np.tile(y, (3, 4, 1)), 1.0), sensitivity, basis, cfg, op)
    assert np.max(np.abs(cmap.hbo - 40.0)) / 40.0 <= 0.01
    # scale division (test_bayes.py:150-163)
    x0 = np.array([30.0, 20.0, 0.05])
    y = sensitivity.c @ np.exp(-(basis.xi @ x0))
    _, d = ox.estimate_lowpass(ox.LowPassBlock(y.reshape(1, 1, 3), 1.0), sensitivity, basis, cfg, op)
    _, s = ox.estimate_lowpass(ox.LowPassBlock((8.0 * y).reshape(1, 1, 3), 8.0), sensitivity, basis, cfg, op)
    assert np.allclose(s.stacked(), d.stacked(), atol=1e-12)
    # fixpoint start stays put (test_bayes.py:165-177), init_spectra path
    x0 = np.array([25.0, 35.0, -0.1])
    spec = np.exp(-(basis.xi @ x0))
    _, c2 = ox.estimate_lowpass(ox.LowPassBlock((sensitivity.c @ spec).reshape(1, 1, 3), 1.0), sensitivity, basis,
                                cfg, op, init_spectra=spec.reshape(1, 1, -1))
    assert np.linalg.norm(c2.stacked()[0, 0] - x0) / np.linalg.norm(x0) <= cfg.rel_tol
    # zero data stays finite (test_bayes.py:219-223)
    sp, c3 = ox.estimate_lowpass(ox.LowPassBlock(np.zeros((2, 2, 3)), 1.0), sensitivity, basis, cfg, op)
    assert np.all(np.isfinite(sp)) and np.all(np.isfinite(c3.stacked()))
    # max_iters=1: only the start fit
    sp1, c4, f4 = ox.estimate_lowpass_fits(ox.LowPassBlock(np.tile(y, (2, 2, 1)), 1.0), sensitivity, basis,
                                           ox.BayesConfig(max_iters=1), op)
    assert np.all(f4 == 1)
    assert np.allclose(sp1[0, 0], np.clip(op.solve @ y, 1e-6, None), rtol=1e-14)


def test_em_generic_band_count(cuda, rng):
    from paper_1706_07263_b200 import CameraSensitivity, ChromophoreBasis, WavelengthGrid

    for L in (6, 41):
        grid = WavelengthGrid(500.0, 20.0 if L == 6 else 5.0, L)
        xi = np.column_stack([np.linspace(0.02, 0.06, L), np.linspace(0.05, 0.015, L), np.ones(L)])
        sens = CameraSensitivity(grid, rng.uniform(0.05, 1.0, size=(3, L)))
        bas = ChromophoreBasis(grid, xi)
        op = ox.TikhonovOperator.from_relative(sens, 1e-3)
        x0 = np.column_stack([rng.uniform(5, 30, 64), rng.uniform(5, 30, 64), rng.uniform(-0.2, 0.2, 64)])
        y = np.exp(-(x0 @ xi.T)) @ sens.c.T
        spectra, cmap, fits = ox.estimate_lowpass_fits(ox.LowPassBlock(y.reshape(8, 8, 3), 1.0), sens, bas,
                                                       ox.BayesConfig(), op)
        ref_s, ref_x, ref_f = O.estimate_lowpass(y.reshape(8, 8, 3), 1.0, sens.c, xi, op.solve)
        assert np.array_equal(fits, ref_f), L
        assert np.max(np.abs(spectra - ref_s)) <= 1e-8 * np.max(np.abs(ref_s)), L
        assert np.max(np.abs(cmap.stacked() - ref_x)) <= 1e-7, L


def test_em_ragged_counts(cuda, sensitivity, basis, rng):
    """Coefficient counts around the persistent kernel's warp / chunk / grid
    boundaries (static first chunk per warp, 32-coefficient dynamic chunks,
    per-lane prefetch of the next coefficient): every coefficient is processed
    exactly once and matches the oracle."""
    op = ox.TikhonovOperator.from_relative(sensitivity, 1e-3)
    for n in (1, 31, 32, 33, 95, 129, 1000, 4099, 20000):
        x0 = np.column_stack([rng.uniform(5, 60, n), rng.uniform(5, 60, n), rng.uniform(-0.2, 0.2, n)])
        y = np.exp(-(x0 @ basis.xi.T)) @ sensitivity.c.T * rng.uniform(0.8, 1.2, (n, 1))
        blk = y.reshape(1, n, 3)
        spectra, cmap, fits = ox.estimate_lowpass_fits(ox.LowPassBlock(blk, 1.0), sensitivity, basis,
                                                       ox.BayesConfig(), op)
        ref_s, ref_x, ref_f = O.estimate_lowpass(blk, 1.0, sensitivity.c, basis.xi, op.solve)
        assert np.array_equal(fits, ref_f), n
        assert np.max(np.abs(spectra - ref_s) / np.maximum(np.abs(ref_s), 1e-3)) <= 1e-9, n
        assert np.max(np.abs(cmap.stacked() - ref_x)) <= 1e-8, n


def test_expectation_step_dense_oracle(cuda, rng, sensitivity):
    from paper_1706_07263_b200 import CameraSensitivity, WavelengthGrid

    cfg = ox.BayesConfig()
    e = rng.uniform(0.2, 1.0, 26)
    assert np.max(np.abs(ox.expectation_step(sensitivity.c @ e, e, sensitivity, cfg) - e)) <= 1e-8
    sens = CameraSensitivity(WavelengthGrid(450.0, 5.0, 6), rng.uniform(0.05, 1.0, size=(3, 6)))
    d2 = ox.second_difference(6)
    y, e = rng.uniform(0.1, 1.0, 3), rng.uniform(0.1, 1.0, 6)
    a = np.vstack([sens.c, d2])
    b = np.concatenate([y, d2 @ e])
    oracle = np.linalg.lstsq(a, b, rcond=None)[0]
    assert np.max(np.abs(ox.expectation_step(y, e, sens, ox.BayesConfig(beta=1.0)) - oracle)) <= 1e-9
    out = ox.expectation_step(rng.uniform(0.1, 1, (4, 7, 3)), rng.uniform(0.1, 1, (4, 7, 26)), sensitivity, cfg)
    assert out.shape == (4, 7, 26)


# ---------------------------------------------------------------- K5 fit
def test_fit_concentration(cuda, golden, basis, rng):
    g = golden("fit")
    got = ox.fit_concentration(g["spectra"], basis)
    assert np.max(np.abs(got - g["x"])) <= 1e-10 * np.max(np.abs(g["x"]))
    for _ in range(5):
        x = rng.uniform(-5, 5, 3)
        assert np.max(np.abs(ox.fit_concentration(ox.expected_spectrum(x, basis), basis) - x)) <= 1e-10
    assert np.max(np.abs(ox.fit_concentration(np.ones(26), basis))) <= 1e-12
    assert np.allclose(ox.expected_spectrum(np.zeros(3), basis), 1.0)
    plane = rng.uniform(0.1, 1.0, size=(4, 5, 26))
    assert ox.fit_concentration(plane, basis).shape == (4, 5, 3)


def test_fit_fp32_kernel(cuda, rng, basis):
    from paper_1706_07263_b200.bayes import fit_device
    from paper_1706_07263_b200.operators import make_operator_set

    x0 = np.column_stack([rng.uniform(5, 60, 4096), rng.uniform(5, 60, 4096), rng.uniform(-0.2, 0.2, 4096)])
    cube = np.exp(-(x0 @ basis.xi.T)).astype(np.float32)
    ops = make_operator_set(n_bands=26, xi=basis.xi)
    got = fit_device(torch.from_numpy(cube).to(cuda), ops).cpu().numpy()
    want = O.fit_cube(cube.astype(np.float64)[None], basis.xi)[0]
    assert np.max(np.abs(got[:, :2] - want[:, :2])) <= 1e-4 * np.max(np.abs(want[:, :2]))


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["exp", "log"])
def test_table_transcendentals_ulp(which):
    """The EM's table-driven exp/log (oxm_math.cuh) against a high-precision
    reference over the EM's argument range: exp of the pre-scaled argument
    zs (e = exp(zs ln2/256)) within 1.1 ulp; log within 1.5 ulp of max(|log x|, 1)
    absolute (the fit sums x = -F log s accumulate absolute errors)."""
    import ctypes
    from decimal import Decimal, getcontext

    from paper_1706_07263_b200 import _native

    getcontext().prec = 40
    rng = np.random.default_rng(7)
    if which == "exp":  # zs = -xi x * 256/ln2 for spectra in [eps, ~1], plus margin
        x = np.concatenate([rng.uniform(-15000.0, 2000.0, 20000), np.linspace(-3.0, 3.0, 2001)])
        c = Decimal(2).ln() / 256
        ref = np.array([float((Decimal(float(v)) * c).exp()) for v in x])
        ref_hp = [(Decimal(float(v)) * c).exp() for v in x]
    else:  # clamped spectra s >= eps: [1e-6, 10], log-uniform, plus values near 1
        x = np.concatenate([np.exp(rng.uniform(np.log(1e-6), np.log(10.0), 20000)), 1.0 + np.linspace(-1e-3, 1e-3, 2001)])
        ref_hp = [Decimal(float(v)).ln() for v in x]
        ref = np.array([float(v) for v in ref_hp])
    dev = torch.device("cuda", 0)
    xin = torch.from_numpy(x).to(dev)
    out = torch.empty_like(xin)
    st = _native.load().oxm_selftest_math(ctypes.c_void_p(xin.data_ptr()), x.size, 0 if which == "exp" else 1,
                                          ctypes.c_void_p(out.data_ptr()), None)
    _native.check(st, "selftest_math")
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    err = np.array([float(abs(Decimal(float(g)) - h)) for g, h in zip(got, ref_hp)])
    if which == "exp":
        ulps = err / np.spacing(np.abs(ref))
        assert ulps.max() <= 1.1, (ulps.max(), x[np.argmax(ulps)])
    else:
        ulps = err / np.spacing(np.maximum(np.abs(ref), 1.0))
        assert ulps.max() <= 1.5, (ulps.max(), x[np.argmax(ulps)])
