#!/usr/bin/env python3
"""Throughput at the BASELINE.json frame configurations (device-resident batches).
    python tools/sweep_configs.py"""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

CONFIGS = [  # (name, H, W, n, frames per launch)
    ("cfg1 256x256 n=1", 256, 256, 1, 256),
    ("cfg2 576x720 n=1 (stereo pairs)", 576, 720, 1, 64),
    ("cfg3 1080x1920 n=2", 1080, 1920, 2, 32),
    ("cfg3 1080x1920 n=2 (bench batch)", 1080, 1920, 2, 64),
    ("cfg5 2160x3840 n=3", 2160, 3840, 3, 8),
    ("cfg5 2160x3840 n=3 (batches of 32)", 2160, 3840, 3, 32),
]


def main():
    import torch

    import bench
    import paper_1706_07263_b200 as ox

    dev = torch.device("cuda", 0)
    sens, basis = bench.operators()
    for name, H, W, n, B in CONFIGS:
        eng = ox.HybridMapEngine(sens, basis, ox.PipelineConfig(n_levels=n), device=dev)
        frames = bench.make_frames(B, H, W, 0.3, 0, dev)
        out = eng.allocate(B, H, W)
        for _ in range(3):
            eng.launch(frames, out)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            eng.launch(frames, out)
        b.record()
        b.synchronize()
        eng.check_flags(out)
        fps = 5 * B / (a.elapsed_time(b) * 1e-3)
        print(json.dumps({"config": name, "frames_per_launch": B, "fps": round(fps, 1),
                          "us_per_frame": round(1e6 / fps, 1), "mpix_per_s": round(fps * H * W / 1e6, 1)}), flush=True)
        del frames, out, eng
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
