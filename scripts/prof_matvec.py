"""Per-phase matvec timing (events around every launch) + graph replay."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1810_08429_b200 import cli, geometry, h2, _native
from paper_1810_08429_b200.device import ptr, stream_handle
L = int(sys.argv[1]) if len(sys.argv) > 1 else 6
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
mesh = geometry.build_sphere_mesh(L)
hm, tree, bt = cli.build_h2_operator(mesh, cli.default_config(level=L, eps=eps))
p = h2.plan(hm)
n = mesh.nt
x = torch.randn(n, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
for _ in range(5): p.run(x, y)
torch.cuda.synchronize()
# per-launch timing
acc = {}
for rep in range(20):
    evs = []
    st = stream_handle()
    _native.call("gc_gather", ptr(x), ptr(p.perm_in), p.n_in, ptr(p.xt), st)
    p.yhat.zero_()
    for Lc in p.launches:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _native.call("gc_segmv", Lc.nseg, ptr(Lc.seg), ptr(Lc.blk), ptr(Lc.A0), ptr(Lc.A1), ptr(Lc.in0), ptr(Lc.in1), ptr(Lc.out), Lc.acc, Lc.maxT, st)
        b.record(); evs.append((Lc, a, b))
    torch.cuda.synchronize()
    if rep >= 5:
        for i, (Lc, a, b) in enumerate(evs):
            acc.setdefault((i, Lc.name, Lc.nseg), []).append(a.elapsed_time(b))
tot = 0
for k, v in acc.items():
    print("%2d %-10s nseg %6d  %.1f us" % (k[0], k[1], k[2], 1e3 * np.median(v))); tot += np.median(v)
print("sum of kernels %.1f us" % (1e3 * tot))
rep = h2.storage_report(hm); print(rep)
# eager end-to-end
for mode in ("eager",):
    torch.cuda.synchronize(); a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50): p.run(x, y)
    b.record(); torch.cuda.synchronize()
    print(mode, "%.1f us/mvm" % (a.elapsed_time(b) / 50 * 1e3))
# graph
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    p.run(x, y)
torch.cuda.current_stream().wait_stream(s)
with torch.cuda.graph(g):
    p.run(x, y)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50): g.replay()
b.record(); torch.cuda.synchronize()
print("graph %.1f us/mvm" % (a.elapsed_time(b) / 50 * 1e3))
