#!/usr/bin/env python3
"""Safety margin of the EM precision schedule, measured (GPU box).

The fp64 tail's stop decisions see the fp32 lead-in's hand-over noise as a
relative perturbation of rel = |dx| / |x|.  This tool measures that
perturbation directly: the all-fp64 schedule and the schedule under test run
the same batch with oxm_ctx_set_em_debug_log on, which records rel of every
fit of every low-pass coefficient (and, for the schedule, which tail step j
after the hand-over made it; restarted coefficients are re-recorded as exact).
For each tail step j (3 = the third or a later one) the script reports the distribution of
|rel_tail / rel_exact - 1| over all decisions, next to the guard band the
schedule applies at that step (max(guard, guard1 2^(-(j-1) h))).

    python tools/em_margin_study.py SEEDS FIRST_SEED K [guard1 halvings]
"""
from __future__ import annotations

import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import torch

    import bench
    import paper_1706_07263_b200 as ox
    from paper_1706_07263_b200 import _native
    from paper_1706_07263_b200.device import ptr

    n_seeds, first, K = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
    g1 = float(sys.argv[4]) if len(sys.argv) > 4 else 0.1
    h = int(sys.argv[5]) if len(sys.argv) > 5 else 2
    B, H, W, n = 64, 1080, 1920, 2
    dev = torch.device("cuda", 0)
    lib = _native.load()
    sens, basis = bench.operators()
    ref = ox.HybridMapEngine(sens, basis, ox.PipelineConfig(n_levels=n), device=dev, em_lead=None)
    sch = ox.HybridMapEngine(sens, basis, ox.PipelineConfig(n_levels=n), device=dev,
                             em_lead=(K, 0.01, 2e-3, g1, h))
    nll = B * (-(-H // 4)) * (-(-W // 4))
    bufs = {}
    for name, eng in (("ref", ref), ("sch", sch)):
        rel = torch.zeros(nll * 24, dtype=torch.float32, device=dev)
        step = torch.zeros(nll * 24, dtype=torch.uint8, device=dev)
        _native.check(lib.oxm_ctx_set_em_debug_log(eng.ctx.handle, ptr(rel), ptr(step)), "debug_log")
        bufs[name] = (rel, step)
    outs = {"ref": ref.allocate(B, H, W, fits=True), "sch": sch.allocate(B, H, W, fits=True)}
    tol = 1e-4
    edges = [1e-6, 1e-5, 1e-4, 1e-3, 2.5e-3, 5e-3, 1e-2, 2.5e-2, 5e-2, 1e-1]
    agg = {}
    for r in range(first, first + n_seeds):
        frames = bench.make_frames(B, H, W, 0.3, r, dev)
        for name, eng in (("ref", ref), ("sch", sch)):
            bufs[name][0].zero_()
            bufs[name][1].zero_()
            eng.launch(frames, outs[name])
        torch.cuda.synchronize()
        er, _ = bufs["ref"]
        tr, tj = bufs["sch"]
        flips = int((outs["ref"].fits != outs["sch"].fits).sum())
        ok = (tj > 0) & (er > 0) & (tr > 0)
        ratio = (tr[ok].double() / er[ok].double() - 1.0).abs()
        js = tj[ok].long()
        near = (er[ok] > 0.5 * tol) & (er[ok] < 2 * tol)
        for j in range(1, 9):
            m = js == j
            if not bool(m.any()):
                continue
            v = ratio[m]
            vn = ratio[m & near]
            a = agg.setdefault(j, {"decisions": 0, "near_tol": 0, "max": 0.0, "max_near_tol": 0.0,
                                   "hist": [0] * (len(edges) + 1)})
            a["decisions"] += int(v.numel())
            a["near_tol"] += int(vn.numel())
            a["max"] = max(a["max"], float(v.max()))
            if vn.numel():
                a["max_near_tol"] = max(a["max_near_tol"], float(vn.max()))
            idx = torch.bucketize(v, torch.tensor(edges, dtype=v.dtype, device=dev))
            a["hist"] = [x + int(c) for x, c in zip(a["hist"], torch.bincount(idx, minlength=len(edges) + 1).tolist())]
        print(json.dumps({"seed": r, "flips": flips}), flush=True)
        del frames
        torch.cuda.empty_cache()
    for j, a in sorted(agg.items()):
        guard = max(0.01, g1 * 2.0 ** (-(j - 1) * h))
        print(json.dumps({"K": K, "tail_step": j, "guard": guard, **a, "hist_edges": edges,
                          "margin_max": guard / a["max"] if a["max"] else None}), flush=True)


if __name__ == "__main__":
    main()
