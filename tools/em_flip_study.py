#!/usr/bin/env python3
"""Fit-count flip study of the EM precision schedule (GPU box).

For each seed set r (bench.make_frames(batch, 1080, 1920, 0.3, r): 4 textured
phantoms, per-frame noise), every schedule's per-coefficient fit counts are
compared with the all-fp64 schedule's (which equal the oracle's: the GPU
tests pin that).  For every mismatch ("flip") the coefficient is replayed in
fp64 on the host with the oracle's operators (bayes.py:185-207) to record its
|x|, fit count and the rel / tol values of its last decisions -- which is what
decides whether a schedule knob (hand-over ratio K, guard bands) protects it.

    python tools/em_flip_study.py SEEDS FIRST_SEED [schedule ...]
schedule = "K[:first_guard[:halvings]]" (e.g. 16, 4, 4:0.1:64; round-2 runs used an
extra x_floor field, since removed: "4:0:0.1:64"); one JSON line per (seed,
schedule) with flips, restarts and per-stage us/frame, then one per flip.
"""
from __future__ import annotations

import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def replay(y, c, xi, solve):
    """fp64 EM of one coefficient exactly as oracle.em_iterate, returning the
    rel value of every iteration and the final x."""
    import numpy as np

    from oracle import oximap_oracle as O

    ops = O.EmOperators(c, xi, 0.1, 1e-6)
    s = np.clip(O.unmix(y[None], solve), 1e-6, None)
    x = ops.fit(s)
    rels = []
    for _ in range(19):
        e = ops.expected(x)
        s = np.clip(ops.prior_update(y[None], e), 1e-6, None)
        nx = ops.fit(s)
        rels.append(float(np.linalg.norm(nx - x) / max(np.linalg.norm(x), 1e-8)))
        x = nx
        if rels[-1] < 1e-4:
            break
    return rels, x[0]


def main():
    import numpy as np
    import torch

    import bench
    import paper_1706_07263_b200 as ox
    from oracle import oximap_oracle as O

    n_seeds, first = int(sys.argv[1]), int(sys.argv[2])
    specs = sys.argv[3:] or ["16", "8", "4", "4:60", "8:60"]
    B, H, W, n = 64, 1080, 1920, 2
    dev = torch.device("cuda", 0)
    sens, basis = bench.operators()
    _, solve = O.ridge_solve(sens.c, 1e-3)
    engines = {"0": ox.HybridMapEngine(sens, basis, ox.PipelineConfig(n_levels=n), device=dev, em_lead=None)}
    for sp in specs:
        p = [float(v) for v in sp.split(":")]
        lead = (p[0], 0.01, 2e-3) + tuple(p[1:3])  # K[:first_guard[:halvings]]
        engines[sp] = ox.HybridMapEngine(sens, basis, ox.PipelineConfig(n_levels=n), device=dev, em_lead=lead)
    outs = {k: e.allocate(B, H, W, fits=True) for k, e in engines.items()}
    hL, wL = -(-H // 4), -(-W // 4)
    for r in range(first, first + n_seeds):
        frames = bench.make_frames(B, H, W, 0.3, r, dev)
        ref = None
        for k, eng in engines.items():
            out = outs[k]
            eng.launch(frames, out)
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
            eng.launch(frames, out, stage_events=evs)
            torch.cuda.synchronize()
            eng.check_flags(out)
            st = [evs[i].elapsed_time(evs[i + 1]) / B * 1e3 for i in range(5)]
            cnt = eng.em_counters(B, H, W)
            rec = {"seed": r, "schedule": k, "us": [round(v, 2) for v in st], "total_us": round(sum(st), 2),
                   "restarts": cnt["restarts"], "tail_fits": cnt["tail_fits"], "lead_fits": cnt["lead_fits"]}
            if k == "0":
                ref = out.fits.clone()
                print(json.dumps(rec), flush=True)
                continue
            diff = (out.fits != ref).nonzero().cpu().numpy()
            rec["flips"] = int(len(diff))
            print(json.dumps(rec), flush=True)
            for f, by, bx in diff:
                blk = frames[f, 4 * by:4 * by + 4, 4 * bx:4 * bx + 4].double().cpu().numpy()
                if blk.shape[:2] != (4, 4):
                    continue
                y = O.haar_forward(blk, 2)[-1]["lp"][0, 0] / 4.0
                rels, x = replay(y, sens.c, basis.xi, solve)
                print(json.dumps({"flip": True, "seed": r, "schedule": k, "frame": int(f), "by": int(by), "bx": int(bx),
                                  "fits_ref": int(ref[f, by, bx]), "fits_test": int(out.fits[f, by, bx]),
                                  "x": [round(float(v), 4) for v in x], "xnorm": float(np.linalg.norm(x)),
                                  "rel_over_tol_last": [round(v / 1e-4, 5) for v in rels[-4:]]}), flush=True)
        del frames
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
