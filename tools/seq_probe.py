#!/usr/bin/env python3
"""Drop-in API throughput probe (GPU box): estimate_sequence frames/s over 16
host fp64 1080p frames and estimate_frame latency (median of 3 after a warm
call), under the current OXM_COPY_THREADS.   python tools/seq_probe.py"""
import json
import os
import pathlib
import statistics
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    import bench
    import paper_1706_07263_b200 as ox
    from paper_1706_07263_b200.pipeline import _copy_threads

    sens, basis = bench.operators()
    fr = bench.make_frames(16, 1080, 1920, 0.3, 0, torch.device("cuda", 0)).cpu().numpy().astype(np.float64)
    imgs = [ox.RgbImage(f) for f in fr]
    cfg = ox.PipelineConfig(n_levels=2)
    for _ in ox.estimate_sequence(imgs[:4], sens, basis, cfg):
        pass
    t = time.perf_counter()
    n = sum(1 for _ in ox.estimate_sequence(imgs, sens, basis, cfg))
    seq = n / (time.perf_counter() - t)
    ox.estimate_frame(imgs[0], sens, basis, cfg)  # warm (pinned staging for the cube)
    lat = []
    for k in range(3):
        t = time.perf_counter()
        ox.estimate_frame(imgs[k], sens, basis, cfg)
        lat.append(time.perf_counter() - t)
    print(json.dumps({"copy_threads": _copy_threads(), "estimate_sequence_fps": seq,
                      "estimate_frame_ms": 1e3 * statistics.median(lat), "cpus": os.cpu_count()}), flush=True)


if __name__ == "__main__":
    main()
