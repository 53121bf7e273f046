#!/usr/bin/env python3
"""Large-batch check (GPU box): one launch over B 1080p frames (default 512:
66 M low-pass coefficients, 1.06 G pixels) audited against the all-fp64 EM
schedule (HybridMapEngine.audit) and timed.   python tools/large_batch_check.py [B]"""
import json
import pathlib
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import torch

    import bench
    import paper_1706_07263_b200 as ox

    B = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    dev = torch.device("cuda", 0)
    sens, basis = bench.operators()
    eng = ox.HybridMapEngine(sens, basis, ox.PipelineConfig(n_levels=2), device=dev)
    frames = bench.make_frames(B, 1080, 1920, 0.3, 7, dev)
    out = eng.allocate(B, 1080, 1920, fits=True)
    eng.launch(frames, out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    eng.launch(frames, out)
    b.record()
    b.synchronize()
    eng.check_flags(out)
    t = a.elapsed_time(b) * 1e-3
    rep = eng.audit(frames, out)
    print(json.dumps({"frames": B, "seconds": t, "fps": B / t, "em": eng.em_counters(B, 1080, 1920), "audit": rep,
                      "peak_mem_gb": torch.cuda.max_memory_allocated(dev) / 1e9}), flush=True)


if __name__ == "__main__":
    main()
