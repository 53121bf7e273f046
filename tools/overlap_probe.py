#!/usr/bin/env python3
"""Plain launch vs sub-batch overlapped launch (per-frame time)."""
import json, pathlib, sys
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import torch
    import bench
    import paper_1706_07263_b200 as ox

    dev = torch.device("cuda", 0)
    sens, basis = bench.operators()
    B = 32
    eng = ox.HybridMapEngine(sens, basis, ox.PipelineConfig(n_levels=2), device=dev)
    frames = bench.make_frames(B, 1080, 1920, 0.3, 0, dev)
    ref = eng.allocate(B, 1080, 1920)
    eng.launch(frames, ref)
    torch.cuda.synchronize()

    def timeit(fn, reps=5):
        for _ in range(2):
            fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) * 1e3 / reps / B

    print(json.dumps({"plain_us_per_frame": timeit(lambda: eng.launch(frames, ref))}))
    for parts in (2, 4, 8):
        for reserve in (0, 1, 2):
            out = eng.allocate(B, 1080, 1920)
            st = {}
            us = timeit(lambda: eng.launch_overlapped(frames, out, parts=parts, em_reserve=reserve, _state=st))
            torch.cuda.synchronize()
            same = bool(torch.equal(out.thb, ref.thb))
            print(json.dumps({"parts": parts, "reserve": reserve, "us_per_frame": us, "bitwise_same": same}), flush=True)


if __name__ == "__main__":
    main()
