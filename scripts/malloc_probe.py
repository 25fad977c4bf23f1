"""Latency of fresh cudaMalloc calls (torch.cuda.caching_allocator_alloc
with the cache emptied) over a few seconds: are there stalls of tens of
ms on this box?  Usage: python scripts/malloc_probe.py [seconds]"""
import sys
import time

import torch

dur = float(sys.argv[1]) if len(sys.argv) > 1 else 5.0
torch.cuda.init()
x = torch.empty(1, device="cuda")
lat = []
t_end = time.perf_counter() + dur
while time.perf_counter() < t_end:
    torch.cuda.empty_cache()
    t = time.perf_counter()
    a = torch.empty(3 << 20, dtype=torch.float64, device="cuda")      # 24 MB: a fresh segment
    lat.append(time.perf_counter() - t)
    del a
    time.sleep(0.005)
lat.sort()
n = len(lat)
print("fresh 24 MB allocations: %d, median %.3f ms, p99 %.3f ms, max %.3f ms, >10 ms: %d" % (
    n, 1e3 * lat[n // 2], 1e3 * lat[int(0.99 * n)], 1e3 * lat[-1], sum(v > 0.01 for v in lat)))
