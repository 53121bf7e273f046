#!/usr/bin/env python3
"""Build EM tuning variants (CPU side) or time them (GPU side).

    python tools/em_variants.py build          # here: nvcc each variant into build/variants/<name>/
    python tools/em_variants.py time [B]       # on the box: per-variant stage times on a 1080p batch
"""
from __future__ import annotations

import json
import os
import pathlib
import subprocess
import sys

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
VARIANTS = {  # name -> extra -D defines (EM kernel knobs)
    "base": (),
    "c64": ("OXM_EM_CHUNK=64",),
}


def lib(name: str) -> pathlib.Path:
    return ROOT / "build" / "variants" / name / "liboximap_b200.so"


def build() -> None:
    from paper_1706_07263_b200 import _build

    for name, defs in VARIANTS.items():
        _build.build(force=True, defines=defs, out=lib(name))
        print(name, "built")


def time_one(batch: int) -> dict:
    import torch

    import bench
    import paper_1706_07263_b200 as ox

    dev = torch.device("cuda", 0)
    sens, basis = bench.operators()
    eng = ox.HybridMapEngine(sens, basis, ox.PipelineConfig(n_levels=2), device=dev)
    frames = bench.make_frames(batch, 1080, 1920, 0.3, 0, dev)
    out = eng.allocate(batch, 1080, 1920, fits=True)
    for _ in range(2):
        eng.launch(frames, out)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(5)]
    for e in evs:
        eng.launch(frames, out, stage_events=e)
    torch.cuda.synchronize()
    st = [sum(e[i].elapsed_time(e[i + 1]) for e in evs) / len(evs) / batch * 1e3 for i in range(5)]
    return {"ll_us": st[0], "em_lead_us": st[1], "em_us": st[2], "px_us": st[3], "fixup_us": st[4], "fits": int(out.fits.sum()), **eng.em_counters(batch, 1080, 1920),
            "thb": float(out.thb.double().sum())}


def main() -> None:
    if sys.argv[1] == "build":
        build()
        return
    if sys.argv[1] == "one":
        print(json.dumps(time_one(int(sys.argv[2]))))
        return
    batch = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    for name in VARIANTS:
        env = dict(os.environ, OXM_LIB_PATH=str(lib(name)))
        r = subprocess.run([sys.executable, __file__, "one", str(batch)], env=env, capture_output=True, text=True)
        print(name, r.stdout.strip() or r.stderr[-500:], flush=True)


if __name__ == "__main__":
    main()
