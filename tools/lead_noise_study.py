"""Study: which fp32 error source of the EM lead-in dominates the hand-over
perturbation (CPU emulation, no GPU; test infrastructure, not product code).

The fp32 lead-in (oxm_em.cuh, em_lead_kernel) hands its state x to the fp64
tail once rel <= K tol.  Its error delta = |x_lead - x_fp64| / |x_fp64| at
that step decides how small K may be (EM tail).  This emulates
the lead-in's step (bayes.py:185-207 in the e + G (y - C e) form) in fp64 with
each fp32 error source switched on alone, then all together:

    y      data rounded to fp32
    state  x rounded to fp32 after every fit
    ex2    2^t with a uniform relative error of +-2^-22 (ex2.approx model)
    lg2    log2 s with a uniform absolute error of +-2^-22 (lg2.approx model)
    sums   the 26-term sums (C e, G r, F log s) and their operands in fp32,
           split into consts (C, G, F rounded to fp32 only), csum (C e and
           e + G r in fp32), fitsum (F log s in fp32) and ssum (C e and
           y - C e exact, only e + G r in fp32)

and reports delta at the step where the fp64 rel first falls to <= K tol.

    python tools/lead_noise_study.py [--size 256] [--k 16 4] [--seed 1]
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

SOURCES = ("y", "state", "ex2", "lg2", "sums")
SPLIT = ("consts", "csum", "fitsum", "ssum")  # parts of "sums" (see the module docstring)


def f32(v):
    return np.asarray(v, dtype=np.float32).astype(np.float64)


def trajectory(y, x1, ops, G, steps, on, rng, tol):
    """x after fits 1..steps+1 and the fp64-convention rel of each step."""
    log2e, ln2 = 1.0 / np.log(2.0), np.log(2.0)
    xi, C, F = ops.xi, ops.c, ops.fit_mat
    if "consts" in on:
        C, G, F = f32(C), f32(G), f32(F)
    if "y" in on:
        y = f32(y)
    x = f32(x1) if on else x1.copy()
    xs, rels = [x], []
    for _ in range(steps):
        t = -(x @ xi.T) * log2e
        e = 2.0 ** t
        if "ex2" in on:
            e = f32(e * (1.0 + rng.uniform(-2.0**-22, 2.0**-22, e.shape)))
        if "sums" in on or "csum" in on:
            e32, C32, G32 = e.astype(np.float32), C.astype(np.float32), G.astype(np.float32)
            r = (y.astype(np.float32) - e32 @ C32.T).astype(np.float32)
            s = (e32 + r @ G32.T).astype(np.float64)
        elif "ssum" in on:  # residual y - C e exact (fp64), e + G r in fp32
            r = y - e @ C.T
            s = (e.astype(np.float32) + r.astype(np.float32) @ G.astype(np.float32).T).astype(np.float64)
        else:
            s = e + (y - e @ C.T) @ G.T
        s = np.maximum(s, ops.eps)
        lg = np.log2(s)
        if "lg2" in on:
            lg = f32(lg + rng.uniform(-2.0**-22, 2.0**-22, lg.shape))
        Fl = F * ln2
        if "sums" in on or "fitsum" in on:
            xn = -(lg.astype(np.float32) @ Fl.astype(np.float32).T).astype(np.float64)
        else:
            xn = -(lg @ Fl.T)
        if "state" in on:
            xn = f32(xn)
        rels.append(np.linalg.norm(xn - x, axis=1) / np.maximum(np.linalg.norm(x, axis=1), 1e-8))
        x = xn
        xs.append(x)
    return np.stack(xs), np.stack(rels)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=256)
    ap.add_argument("--k", type=float, nargs="+", default=[16.0, 4.0])
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--texture", type=float, default=0.3)
    a = ap.parse_args()
    tol, n = 1e-4, 2
    sens, basis = fixtures.default_sensitivity(), fixtures.default_basis()
    rgb = synth.phantom_rgb_f32(a.size, a.size, a.seed, sens, basis, texture_density=a.texture).astype(np.float64)
    ops = O.EmOperators(sens.c, basis.xi, 0.1, 1e-6)
    G = O.scipy.linalg.cho_solve(ops.cho, sens.c.T)  # L x 3
    _, solve = O.ridge_solve(sens.c, 1e-3)
    y = O.haar_forward(rgb, n)[-1]["lp"].reshape(-1, 3) / 2.0**n
    x1 = ops.fit(np.maximum(y @ solve.T, ops.eps))
    steps = 19
    rng = np.random.default_rng(0)
    xs64, rel64 = trajectory(y, x1, ops, G, steps, (), rng, tol)
    print(f"{y.shape[0]} low-pass coefficients ({a.size}^2, n = {n}, texture {a.texture}, seed {a.seed})")
    for K in a.k:
        # hand-over step: first step whose fp64 rel <= K tol (the state before it is handed over)
        below = rel64 <= K * tol
        hit = below.any(axis=0)
        k_h = np.where(hit, below.argmax(axis=0), -1)
        sel = np.nonzero(hit)[0]
        print(f"K = {K:g}: {sel.size} coefficients reach rel <= K tol; delta at hand-over "
              "(|x_lead - x_fp64| / |x_fp64|): median / 99.9% / max")
        no_resid = ("y", "state", "ex2", "lg2", "consts", "fitsum", "ssum")  # all but the fp32 residual
        no_resid_y = tuple(s for s in no_resid if s != "y")  # ... and y kept in fp64 (e.g. a hi/lo pair)
        for on in [(s,) for s in SOURCES + SPLIT] + [SOURCES, no_resid, no_resid_y]:
            xs, _ = trajectory(y, x1, ops, G, steps, on, np.random.default_rng(1), tol)
            xh, xr = xs[k_h[sel], sel], xs64[k_h[sel], sel]
            d = np.linalg.norm(xh - xr, axis=1) / np.linalg.norm(xr, axis=1)
            name = {SOURCES: "all (the lead-in today)", no_resid: "all, fp64 residual",
                    no_resid_y: "all, fp64 residual + y"}.get(on, "+".join(on))
            print(f"   {name:24s} {np.median(d):.2e}  {np.quantile(d, 0.999):.2e}  {d.max():.2e}")


if __name__ == "__main__":
    main()
