"""The CPU oracle must reproduce the reference's own outputs bit for bit
(golden vectors from tools/make_golden.py).  This pins the oracle before any
GPU result is compared against it."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oximap_oracle as O


def test_operators(golden):
    g = golden("operators")
    gamma, solve = O.ridge_solve(g["c"], 1e-3)
    assert gamma == g["gamma"]
    assert np.array_equal(solve, g["solve"])


def test_haar_forward_inverse_bitwise(golden):
    g = golden("haar")
    for i in range(int(g["count"])):
        img, n = g[f"img{i}"], int(g[f"n{i}"])
        levels = O.haar_forward(img, n)
        for k, lv in enumerate(levels):
            for name in ("lp", "dh", "dv", "dd"):
                assert np.array_equal(lv[name], g[f"c{i}_l{k}_{name}"]), (i, k, name)
            assert tuple(lv["orig_shape"]) == tuple(g[f"c{i}_l{k}_orig"])
        assert np.array_equal(O.haar_inverse(levels, levels[-1]["lp"]), g[f"inv{i}"])


def test_unmix(golden):
    g, ops = golden("unmix"), golden("operators")
    assert np.array_equal(O.unmix(g["rgb"], ops["solve"]), g["out"])


def test_em_bitwise(golden):
    g, ops = golden("em"), golden("operators")
    for j in range(int(g["count"])):
        kw = {}
        if f"cfg{j}" in g:
            beta, iters, tol, eps = g[f"cfg{j}"]
            kw = dict(beta=beta, max_iters=int(iters), rel_tol=tol, eps=eps)
        spectra, x, fits = O.estimate_lowpass(g[f"lp{j}"], float(g[f"scale{j}"]), ops["c"], ops["xi"], ops["solve"], **kw)
        assert np.array_equal(spectra, g[f"spectra{j}"]), j
        assert np.array_equal(x, g[f"x{j}"]), j
        assert fits.min() >= 1 and fits.max() <= kw.get("max_iters", 20)


def test_fit(golden):
    g, ops = golden("fit"), golden("operators")
    x = O.fit_cube(g["spectra"].reshape(1, -1, 26), ops["xi"]).reshape(-1, 3)
    assert np.array_equal(x, g["x"])


@pytest.mark.parametrize("i", range(8))
def test_estimate_frame_bitwise(golden, i):
    g, ops = golden("frames"), golden("operators")
    H, W, n, nb, nt = (int(v) for v in g[f"meta{i}"])
    mode = str(g[f"mode{i}"])
    out = O.estimate_frame(g[f"rgb{i}"], ops["c"], ops["xi"], mode=mode, n_levels=n)
    assert np.array_equal(out["x"], g[f"x{i}"])
    assert np.array_equal(out["thb"], g[f"thb{i}"])
    assert np.array_equal(out["so2"], g[f"so2{i}"], equal_nan=True)
    if f"cube{i}" in g:
        assert np.array_equal(out["cube"], g[f"cube{i}"])
    assert out["stats"] == {"bayes_coefficients": nb, "tikhonov_coefficients": nt}


def test_threaded_oracle_matches(golden):
    g, ops = golden("frames"), golden("operators")
    one = O.estimate_frame(g["rgb5"], ops["c"], ops["xi"], n_levels=1, threads=1)
    four = O.estimate_frame(g["rgb5"], ops["c"], ops["xi"], n_levels=1, threads=4)
    assert np.array_equal(one["fits"], four["fits"])
    # slab-wise BLAS/LAPACK calls re-associate: ~1e-11 relative jitter, no decision flips
    assert np.allclose(one["x"], four["x"], rtol=1e-10, atol=1e-9)
