#!/usr/bin/env python3
"""Pinned host <-> device copy bandwidth on this box: each direction alone and
both together, with 1 or 2 streams per direction (GB/s, best of 3)."""
import json
import time

import torch


def run(n_h2d, n_d2h, nbytes=512 * 2**20, reps=4):
    dev = torch.device("cuda", 0)
    hs = [torch.empty(nbytes, dtype=torch.uint8).pin_memory() for _ in range(max(n_h2d, n_d2h))]
    ds = [torch.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(max(n_h2d, n_d2h))]
    streams = [torch.cuda.Stream() for _ in range(n_h2d + n_d2h)]
    best = 0.0
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            for i in range(n_h2d):
                with torch.cuda.stream(streams[i]):
                    ds[i].copy_(hs[i], non_blocking=True)
            for i in range(n_d2h):
                with torch.cuda.stream(streams[n_h2d + i]):
                    hs[i].copy_(ds[i], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        best = max(best, reps * nbytes / dt / 1e9)
    return best  # GB/s per stream-direction pair... per stream


def main():
    for h2d, d2h in ((1, 0), (2, 0), (0, 1), (0, 2), (1, 1), (2, 2)):
        per_stream = run(h2d, d2h)
        print(json.dumps({"h2d_streams": h2d, "d2h_streams": d2h, "GBps_per_stream": round(per_stream, 2),
                          "GBps_h2d_total": round(per_stream * h2d, 2), "GBps_d2h_total": round(per_stream * d2h, 2)}))


if __name__ == "__main__":
    main()
