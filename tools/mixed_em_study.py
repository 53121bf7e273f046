"""Study: fp32 lead-in + fp64 tail for the EM (CPU emulation, no GPU).

The EM of bayes.py:185-207 contracts (~0.49 per fit).  Run it in fp32 while
rel > K * tol (a "not converged" decision there is robust to fp32 error),
then hand the state x to the exact fp64 iteration from the step whose fp32
rel first fell to <= K * tol.  The fp64 tail removes the fp32 perturbation at
the contraction rate; the stop decision is trusted unless rel lands within
`margin` of tol at any fp64 step (guard -> full fp64 redo).

Reports, per frame and K: guarded fraction, unguarded fit-count flips against
the oracle, final spectrum error, and the THb/SO2 error the spectrum error
causes through the (fp64) collapse formula, split by min reconstructed band.

    python tools/mixed_em_study.py [--k 8 16 32] [--noise 2.4e-7]
"""

from __future__ import annotations

import argparse
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import oximap_oracle as O  # noqa: E402
from paper_1706_07263_b200 import fixtures, synth  # noqa: E402


def run(rgb, n, K, margin, noise, rng, tol=1e-4, max_iters=20, eps=1e-6):
    sens, basis = fixtures.default_sensitivity(), fixtures.default_basis()
    c, xi = sens.c, basis.xi
    ref = O.estimate_frame(rgb, c, xi, n_levels=n)
    _, solve = O.ridge_solve(c, 1e-3)
    ops = O.EmOperators(c, xi, 0.1, eps)
    G = O.scipy.linalg.cho_solve(ops.cho, c.T)  # L x 3 = N^-1 C^T
    pyr = O.haar_forward(rgb, n)
    ll = pyr[-1]["lp"]
    h, w = ll.shape[:2]
    y = (ll / 2.0**n).reshape(-1, 3)
    s_ref, x_ref, fits_ref = O.estimate_lowpass(ll, 2.0**n, c, xi, solve)
    s_ref, fits_ref = s_ref.reshape(-1, c.shape[1]), fits_ref.ravel()
    N = y.shape[0]

    # fit #1 in fp64 (as on the GPU: low-pass kernel)
    s0 = np.clip(y @ solve.T, eps, None)
    x0 = ops.fit(s0)

    f32 = np.float32
    c32, xi32, G32, F32 = (a.astype(f32) for a in (c, xi, G, ops.fit_mat))
    y32 = y.astype(f32)

    def noisy(a, rel):
        return (a * (1 + rel * rng.uniform(-1, 1, a.shape))).astype(f32)

    # fp32 phase
    x = x0.astype(f32)
    fits = np.ones(N, np.int32)
    active = np.arange(N)
    xs = x0.copy()           # handed-over state (fp64)
    fs = np.ones(N, np.int32)
    handed = np.zeros(N, bool)
    for _ in range(max_iters - 1):
        xa = x[active]
        e = noisy(np.exp(-(xa @ xi32.T)), noise)
        s = np.maximum(e + (y32[active] - e @ c32.T) @ G32.T, f32(eps))
        lg = np.log(s).astype(f32) + (noise * rng.uniform(-1, 1, s.shape)).astype(f32)
        xn = -(lg @ F32.T)
        rel = np.linalg.norm(xn - xa, axis=1) / np.maximum(np.linalg.norm(xa, axis=1), f32(1e-8))
        hand = rel <= K * tol
        # hand over the state BEFORE this step: the fp64 tail redoes it
        idx = active[hand]
        xs[idx] = xa[hand].astype(np.float64)
        fs[idx] = fits[idx]
        handed[idx] = True
        keep = ~hand
        x[active[keep]] = xn[keep]
        fits[active[keep]] += 1
        active = active[keep]
        if fits[active].size and fits[active].max() >= max_iters:
            break
        if active.size == 0:
            break
    # anything still active hit max_iters in fp32 (none expected): mark guard
    guard = np.zeros(N, bool)
    guard[active] = True
    xs[active] = x[active]
    fs[active] = fits[active]

    # fp64 tail (exact form of the reference)
    x = xs.copy()
    fits = fs.copy()
    spec = np.zeros_like(s_ref)
    active = np.where(~guard)[0]
    while active.size:
        xa = x[active]
        e = ops.expected(xa)
        s = np.clip(ops.prior_update(y[active], e), eps, None)
        xn = ops.fit(s)
        rel = np.linalg.norm(xn - xa, axis=-1) / np.maximum(np.linalg.norm(xa, axis=-1), 1e-8)
        guard[active[np.abs(rel / tol - 1) < margin]] = True
        spec[active] = s
        x[active] = xn
        fits[active] += 1
        stop = (rel < tol) | (fits[active] >= max_iters)
        active = active[~stop]
    ok = ~guard
    flips = int(np.sum(fits[ok] != fits_ref[ok]))
    # guarded coefficients take the exact fp64 path
    spec[guard] = s_ref[guard]
    srel = np.abs(spec - s_ref) / np.abs(s_ref)

    # maps through the fp64 collapse: cube(p) = S[b] + solve (rgb(p) - LL[b]/2^n)
    H, W = rgb.shape[:2]
    py, px = np.meshgrid(np.arange(H) >> n, np.arange(W) >> n, indexing="ij")
    b = (py * w + px).ravel()
    llu = (ll / 2.0**n).reshape(-1, 3)
    d = rgb.reshape(-1, 3) - llu[b]
    cube = spec[b] + d @ solve.T
    minband = np.min(ref["cube"].reshape(-1, c.shape[1]), axis=1)
    x_px = O.fit_cube(cube.reshape(H, W, -1), xi)
    thb, so2 = O.thb_so2(x_px[..., 0], x_px[..., 1])
    trel = np.abs(thb - ref["thb"]) / np.maximum(np.abs(ref["thb"]), 1e-300)
    okso = ~np.isnan(ref["so2"])
    sab = np.where(okso, np.abs(np.nan_to_num(so2) - np.nan_to_num(ref["so2"])), 0)
    out = {"K": K, "N": N, "guard_frac": guard.mean(), "flips": flips, "fp64_steps": float(np.mean(fits - fs)),
           "fp32_steps": float(np.mean(fs - 1)), "S_rel_max": float(srel[ok].max()),
           "S_rel_p99": float(np.quantile(srel[ok], 0.99))}
    for lo, hi in ((0, 1e-4), (1e-4, 2e-3), (2e-3, 1e9)):
        m = ((minband >= lo) & (minband < hi)).reshape(H, W)
        if m.any():
            out[f"band[{lo:g},{hi:g})"] = (int(m.sum()), float(trel[m].max()), float(sab[m].max()))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--k", type=float, nargs="+", default=[8, 16, 32])
    ap.add_argument("--margin", type=float, default=0.01)
    ap.add_argument("--noise", type=float, default=2.4e-7)
    ap.add_argument("--cfg", default="2")
    args = ap.parse_args()
    sens, basis = fixtures.default_sensitivity(), fixtures.default_basis()
    shapes = {"1": (256, 256, 1), "2": (576, 720, 1), "3": (1080, 1920, 2)}
    H, W, n = shapes[args.cfg]
    rgb = synth.phantom_rgb_f32(H, W, 0, sens, basis)
    for K in args.k:
        print(run(rgb, n, K, args.margin, args.noise, np.random.default_rng(1)))


if __name__ == "__main__":
    main()
