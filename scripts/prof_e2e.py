"""Where the end-to-end h2.mvm time goes at C2 (host timers around each
step of the zero-copy path: numpy -> pinned, re-point + replay, sync,
pinned -> numpy)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1810_08429_b200 import cli, geometry, h2
L = int(sys.argv[1]) if len(sys.argv) > 1 else 6
mesh = geometry.build_sphere_mesh(L)
hm, _, _ = cli.build_h2_operator(mesh, cli.default_config(eps=1e-6))
x = np.random.default_rng(0).standard_normal(mesh.nt)
for _ in range(20):
    h2.mvm(hm, x)
p = h2.plan(hm)
N = 200
t = np.zeros(6)
for _ in range(N):
    a = time.perf_counter()
    xx = h2._check_dim(x, mesh.nt)
    b = time.perf_counter()
    p.pin_x.numpy()[:] = xx
    c = time.perf_counter()
    p.bind(p.pin_x, p.pin_y)
    p.graph.replay()
    d = time.perf_counter()
    torch.cuda.current_stream().synchronize()
    e = time.perf_counter()
    y = p.pin_y.numpy().copy()
    f = time.perf_counter()
    t += np.array([b - a, c - b, d - c, e - d, f - e, f - a])
t = t / N * 1e6
print("check %.1f  pin-in %.1f  bind+replay-enq %.1f  gpu+sync %.1f  copy-out %.1f  total %.1f us" % tuple(t))
a = time.perf_counter()
for _ in range(N):
    h2.mvm(hm, x)
print("h2.mvm %.1f us" % ((time.perf_counter() - a) / N * 1e6))
xd = torch.from_numpy(x).cuda(); yd = torch.empty_like(xd)
for _ in range(5):
    p.run(xd, yd)
torch.cuda.synchronize()
a = time.perf_counter()
for _ in range(N):
    p.run(xd, yd)
    torch.cuda.current_stream().synchronize()
print("device run + sync %.1f us" % ((time.perf_counter() - a) / N * 1e6))
