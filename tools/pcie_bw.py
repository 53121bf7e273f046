#!/usr/bin/env python3
"""Pinned host<->device copy bandwidth on this box: H2D, D2H, and both at once."""
import torch, time

dev = torch.device("cuda", 0)
n = 512 * 2**20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_a = torch.empty(n, dtype=torch.uint8, device=dev)
d_b = torch.empty(n, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in [("h2d", lambda: d_a.copy_(h_in, non_blocking=True)),
                 ("d2h", lambda: h_out.copy_(d_b, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    print(name, f"{5 * n / (time.perf_counter() - t) / 1e9:.1f} GB/s")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t
print(f"concurrent: {5 * n / dt / 1e9:.1f} GB/s each direction")
