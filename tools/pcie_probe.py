#!/usr/bin/env python
"""PCIe floor for the e2e number: 1 GiB pinned H2D, D2H, and both at once on
two streams (GB/s, best of 3)."""
import time
import torch

import os
n = 1 << int(os.environ.get("PROBE_EXP", "27"))
h_in = torch.empty(n, dtype=torch.int64, pin_memory=True)
h_out = torch.empty(n, dtype=torch.int64, pin_memory=True)
d_a = torch.empty(n, dtype=torch.int64, device="cuda")
d_b = torch.empty(n, dtype=torch.int64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn):
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best
gb = 8 * n / 1e9
t = timed(lambda: d_a.copy_(h_in, non_blocking=True))
print(f"H2D: {1e3 * t:.2f} ms = {gb / t:.1f} GB/s")
t = timed(lambda: h_out.copy_(d_b, non_blocking=True))
print(f"D2H: {1e3 * t:.2f} ms = {gb / t:.1f} GB/s")
def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
t = timed(both)
print(f"H2D + D2H concurrently : {1e3 * t:.2f} ms = {2 * gb / t:.1f} GB/s total")
