"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A NumPy/SciPy restatement of the reference hybrid path
(/root/reference/pkg/src/oximap, pure Python), used solely as the checker by
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs.  Nothing in the product package imports it.

Parity is PINNED: tests/test_oracle_golden.py checks every function here
against golden vectors produced by running the reference itself
(tools/make_golden.py -> tests/golden/*.npz): Haar planes, Tikhonov unmix,
EM spectra/concentrations, fit_cube and full estimate_frame outputs must be
bit-identical (same NumPy/SciPy calls in the same order), which in turn pins
the per-coefficient fit counts this oracle records and the reference does
not expose (bayes.py:199-205).

Third-party arithmetic (not vendored in the reference, pinned only by
pyproject.toml:10-15 lower bounds): NumPy >= 1.24 (`@` -> OpenBLAS dgemm,
np.log/np.exp), SciPy >= 1.10 (cho_factor/cho_solve -> LAPACK dpotrf/dpotrs).
Golden vectors were generated with numpy 2.3.5 / scipy 1.18.1.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import scipy.linalg

# ---------------------------------------------------------------- Haar
# haar.py:80-150


def _edge_pad_even(p: np.ndarray) -> np.ndarray:
    """haar.py:80-85: replicate the last row / column of odd planes."""
    h, w = p.shape[:2]
    if h % 2 == 0 and w % 2 == 0:
        return p
    widths = [(0, h % 2), (0, w % 2)] + [(0, 0)] * (p.ndim - 2)
    return np.pad(p, widths, mode="edge")


def haar_forward(image: np.ndarray, n_levels: int) -> list[dict]:
    """haar.py:88-101, 120-142.  Levels finest first, each a dict with
    lp, dh, dv, dd, orig_shape."""
    plane = np.asarray(image, dtype=np.float64)
    out = []
    for _ in range(n_levels):
        shape = plane.shape[:2]
        q = _edge_pad_even(plane)
        a, b, c, d = q[0::2, 0::2], q[0::2, 1::2], q[1::2, 0::2], q[1::2, 1::2]
        lvl = {
            "lp": 0.5 * (a + b + c + d),
            "dh": 0.5 * (a + b - c - d),
            "dv": 0.5 * (a - b - c + d),
            "dd": 0.5 * (a - b + c - d),
            "orig_shape": shape,
        }
        out.append(lvl)
        plane = lvl["lp"]
    return out


def haar_inverse(levels: list[dict], residual_lp: np.ndarray) -> np.ndarray:
    """haar.py:104-117, 145-150 (no shape validation: oracle inputs are
    well formed)."""
    rec = residual_lp
    for lvl in reversed(levels):
        h2, w2 = rec.shape[:2]
        full = np.empty((2 * h2, 2 * w2) + rec.shape[2:])
        dh, dv, dd = lvl["dh"], lvl["dv"], lvl["dd"]
        full[0::2, 0::2] = 0.5 * (rec + dh + dv + dd)
        full[0::2, 1::2] = 0.5 * (rec + dh - dv - dd)
        full[1::2, 0::2] = 0.5 * (rec - dh - dv + dd)
        full[1::2, 1::2] = 0.5 * (rec - dh + dv - dd)
        oh, ow = lvl["orig_shape"]
        rec = full[:oh, :ow]
    return rec


# ---------------------------------------------------------------- operators
# unmix.py:53-82, bayes.py:84-135


def ridge_solve(c: np.ndarray, rel_gamma: float) -> tuple[float, np.ndarray]:
    """unmix.py:67-74 + 53-65: gamma = rel * tr(C^T C) / L;
    solve = C^T (C C^T + gamma I)^-1, returned L x 3."""
    gamma = rel_gamma * (np.trace(c.T @ c) / c.shape[1])
    return gamma, np.linalg.solve(c @ c.T + gamma * np.eye(3), c).T


def unmix(rgb: np.ndarray, solve: np.ndarray) -> np.ndarray:
    """unmix.py:77-82."""
    return np.asarray(rgb, dtype=np.float64) @ solve.T


def d2_operator(count: int) -> np.ndarray:
    """bayes.py:84-93."""
    d2 = np.zeros((count - 2, count))
    k = np.arange(count - 2)
    d2[k, k], d2[k, k + 1], d2[k, k + 2] = 1.0, -2.0, 1.0
    return d2


class EmOperators:
    """bayes.py:96-135: fit matrix and Cholesky of N = C^T C + beta D2^T D2."""

    def __init__(self, c: np.ndarray, xi: np.ndarray, beta: float, eps: float):
        self.c = c
        self.xi = xi
        self.eps = eps
        self.fit_mat = np.linalg.solve(xi.T @ xi, xi.T)
        d2 = d2_operator(c.shape[1])
        self.prior = beta * (d2.T @ d2)
        normal = c.T @ c + self.prior
        self.cond = np.linalg.cond(normal)
        self.cho = scipy.linalg.cho_factor(normal)

    def fit(self, spectra: np.ndarray) -> np.ndarray:
        return -(np.log(np.clip(spectra, self.eps, None)) @ self.fit_mat.T)

    def expected(self, x: np.ndarray) -> np.ndarray:
        return np.exp(-(x @ self.xi.T))

    def prior_update(self, y: np.ndarray, e: np.ndarray) -> np.ndarray:
        rhs = y @ self.c + e @ self.prior
        flat = rhs.reshape(-1, rhs.shape[-1])
        return scipy.linalg.cho_solve(self.cho, flat.T).T.reshape(e.shape)


# ---------------------------------------------------------------- EM
# bayes.py:185-272


def em_iterate(y, spectra0, ops: EmOperators, max_iters: int, rel_tol: float):
    """bayes.py:185-207 with the per-coefficient fit count recorded:
    every coefficient gets fit #1, then one more per loop pass it takes
    part in; it leaves the active set after the pass where rel < rel_tol."""
    spectra = spectra0
    x = ops.fit(spectra)
    fits = np.ones(y.shape[0], dtype=np.int32)
    active = np.arange(y.shape[0])
    for _ in range(max_iters - 1):
        e = ops.expected(x[active])
        new_spec = np.clip(ops.prior_update(y[active], e), ops.eps, None)
        new_x = ops.fit(new_spec)
        prev = x[active]
        rel = np.linalg.norm(new_x - prev, axis=-1) / np.maximum(np.linalg.norm(prev, axis=-1), 1e-8)
        spectra[active] = new_spec
        x[active] = new_x
        fits[active] += 1
        active = active[rel >= rel_tol]
        if active.size == 0:
            break
    return spectra, x, fits


def estimate_lowpass(rgb_lp, scale, c, xi, solve, *, beta=0.1, max_iters=20, rel_tol=1e-4, eps=1e-6,
                     threads=1, init_spectra=None):
    """bayes.py:210-272.  Returns spectra (h, w, L), x (h, w, 3), fits (h, w)."""
    rgb_lp = np.asarray(rgb_lp, dtype=np.float64)
    h, w = rgb_lp.shape[:2]
    n, L = h * w, c.shape[1]
    y = (rgb_lp / scale).reshape(n, 3)
    ops = EmOperators(c, xi, beta, eps)
    s0 = unmix(y, solve) if init_spectra is None else np.asarray(init_spectra, dtype=np.float64).reshape(n, L).copy()
    s0 = np.clip(s0, eps, None)
    if threads <= 1 or n < 2 * threads:
        spectra, x, fits = em_iterate(y, s0, ops, max_iters, rel_tol)
    else:
        spectra, x = np.empty_like(s0), np.empty((n, 3))
        fits = np.empty(n, dtype=np.int32)
        bounds = np.linspace(0, n, threads + 1, dtype=int)

        def run(lo_hi):
            lo, hi = lo_hi
            s, xx, ff = em_iterate(y[lo:hi], s0[lo:hi], ops, max_iters, rel_tol)
            spectra[lo:hi], x[lo:hi], fits[lo:hi] = s, xx, ff

        with ThreadPoolExecutor(max_workers=threads) as pool:
            list(pool.map(run, [(a, b) for a, b in zip(bounds[:-1], bounds[1:]) if b > a]))
    return spectra.reshape(h, w, L), x.reshape(h, w, 3), fits.reshape(h, w)


# ---------------------------------------------------------------- fit + maps
# pipeline.py:66-94, core.py:197-209


def fit_cube(cube: np.ndarray, xi: np.ndarray, eps: float = 1e-6, cal: float = 1.0, threads: int = 1) -> np.ndarray:
    """pipeline.py:66-94 -> (H, W, 3) = (hbo, hb, offset)."""
    h, w, L = cube.shape
    flat = cube.reshape(-1, L)
    fit_mat = np.linalg.solve(xi.T @ xi, xi.T)

    def fit(s):
        return -(np.log(np.clip(s, eps, None)) @ fit_mat.T)

    if threads <= 1 or h < 2 * threads:
        x = fit(flat)
    else:
        x = np.empty((flat.shape[0], 3))
        bounds = np.linspace(0, flat.shape[0], threads + 1, dtype=int)

        def run(lo_hi):
            lo, hi = lo_hi
            x[lo:hi] = fit(flat[lo:hi])

        with ThreadPoolExecutor(max_workers=threads) as pool:
            list(pool.map(run, zip(bounds[:-1], bounds[1:])))
    x = x * np.array([cal, cal, 1.0])
    return x.reshape(h, w, 3)


def thb_so2(hbo: np.ndarray, hb: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """core.py:197-209."""
    thb = np.clip(hbo, 0.0, None) + np.clip(hb, 0.0, None)
    so2 = np.full_like(thb, np.nan)
    np.divide(np.clip(hbo, 0.0, None), thb, out=so2, where=thb > 0)
    return thb, so2


# ---------------------------------------------------------------- frame
# pipeline.py:117-217


def estimate_frame(rgb: np.ndarray, c: np.ndarray, xi: np.ndarray, *, mode: str = "hybrid", n_levels: int = 1,
                   rel_gamma: float = 1e-3, beta: float = 0.1, max_iters: int = 20, rel_tol: float = 1e-4,
                   eps: float = 1e-6, cal: float = 1.0, threads: int = 1, want_cube: bool = True) -> dict:
    """Reference estimate_frame for an RGB frame.  Returns a dict with cube
    (H, W, L) | None, x (H, W, 3), thb, so2, fits (low-pass plane) | None,
    stats."""
    rgb = np.asarray(rgb, dtype=np.float64)
    H, W = rgb.shape[:2]
    _, solve = ridge_solve(c, rel_gamma)
    if mode == "bayes_only":
        spectra, _, fits = estimate_lowpass(rgb, 1.0, c, xi, solve, beta=beta, max_iters=max_iters,
                                            rel_tol=rel_tol, eps=eps, threads=threads)
        cube, stats = spectra, {"bayes_coefficients": H * W, "tikhonov_coefficients": 0}
    else:
        pyr = haar_forward(rgb, n_levels)
        dirs = [{k: (unmix(lv[k], solve) if k in ("dh", "dv", "dd") else lv[k]) for k in lv} for lv in pyr]
        residual = pyr[-1]["lp"]
        n_lp = residual.shape[0] * residual.shape[1]
        n_dir = 3 * sum(lv["dh"].shape[0] * lv["dh"].shape[1] for lv in pyr)
        scale = 2.0 ** n_levels
        if mode == "hybrid":
            spectra_lp, _, fits = estimate_lowpass(residual, scale, c, xi, solve, beta=beta, max_iters=max_iters,
                                                   rel_tol=rel_tol, eps=eps, threads=threads)
            coarse = spectra_lp * scale
            stats = {"bayes_coefficients": n_lp, "tikhonov_coefficients": n_dir}
        elif mode == "tikhonov_only":
            coarse, fits = unmix(residual, solve), None
            stats = {"bayes_coefficients": 0, "tikhonov_coefficients": n_lp + n_dir}
        else:
            raise ValueError(mode)
        cube = haar_inverse(dirs, coarse)
    x = fit_cube(cube, xi, eps, cal, threads)
    thb, so2 = thb_so2(x[..., 0], x[..., 1])
    return {"cube": cube if want_cube else None, "x": x, "thb": thb, "so2": so2, "fits": fits, "stats": stats}


def default_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
