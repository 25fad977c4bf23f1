"""Where the end-to-end product time goes (h2.mvm with numpy in / out):
host staging copy, pinned output allocation, graph re-binding, the graph
with host-resident x / y, and the device-resident graph.  Usage:
python scripts/e2e_parts.py level eps"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_08429_b200 import cli, geometry, h2  # noqa: E402

L, eps = int(sys.argv[1]), float(sys.argv[2])
mesh = geometry.build_sphere_mesh(L)
hm, _, _ = cli.build_h2_operator(mesh, cli.default_config(eps=eps))
p = h2.plan(hm)
n = mesh.nt
x = np.random.default_rng(0).standard_normal(n)
K = 200


def timeit(fn, k=K):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k * 1e6


print("L%d n=%d" % (L, n))
print("h2.mvm (public API)                 %7.1f us" % timeit(lambda: h2.mvm(hm, x)))
print("plan.apply_host                     %7.1f us" % timeit(lambda: p.apply_host(x)))
pin_x = torch.empty(n, dtype=torch.float64, pin_memory=True)
pin_y = torch.empty(n, dtype=torch.float64, pin_memory=True)
print("numpy -> pinned copy                %7.1f us" % timeit(lambda: pin_x.numpy().__setitem__(slice(None), x)))
print("pinned -> numpy copy                %7.1f us" % timeit(lambda: pin_y.numpy().copy()))
print("torch.empty pinned (cached)         %7.1f us" % timeit(lambda: torch.empty(n, dtype=torch.float64,
                                                                                   pin_memory=True)))
dx = torch.randn(n, dtype=torch.float64, device="cuda")
dy = torch.empty_like(dx)
p.bind(pin_x, pin_y)


def graph_host_fixed():
    p.graph.replay()
    torch.cuda.current_stream().synchronize()


print("graph, pinned x/y bound, + sync     %7.1f us" % timeit(graph_host_fixed))
ys = [torch.empty(n, dtype=torch.float64, pin_memory=True) for _ in range(2)]
it = [0]


def graph_rebind():
    it[0] ^= 1
    p.bind(pin_x, ys[it[0]])
    p.graph.replay()
    torch.cuda.current_stream().synchronize()


print("graph, y re-bound every call, +sync %7.1f us" % timeit(graph_rebind))
p.bind(dx, dy)


def graph_dev():
    p.graph.replay()
    torch.cuda.current_stream().synchronize()


print("graph, device x/y, + sync           %7.1f us" % timeit(graph_dev))


def graph_dev_nosync():
    p.graph.replay()


print("graph, device x/y, back to back     %7.1f us" % timeit(graph_dev_nosync))


def dma_path():
    dx.copy_(pin_x, non_blocking=True)
    p.graph.replay()
    pin_y.copy_(dy, non_blocking=True)
    torch.cuda.current_stream().synchronize()


p.bind(dx, dy)
print("DMA in, graph (device x/y), DMA out  %7.1f us" % timeit(dma_path))


def ctx_only():
    with torch.cuda.device(p.dev):
        pass


print("torch.cuda.device context           %7.1f us" % timeit(ctx_only))
import threading
lk = threading.Lock()


def lock_only():
    with lk:
        pass


print("lock                                %7.1f us" % timeit(lock_only))
