"""Per-phase matvec timing for the panel plan (events around every phase
launch, all on one stream) + graph replay."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1810_08429_b200 import cli, geometry, h2
from paper_1810_08429_b200.device import stream_handle
L = int(sys.argv[1]) if len(sys.argv) > 1 else 6
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
mesh = geometry.build_sphere_mesh(L)
hm, tree, bt = cli.build_h2_operator(mesh, cli.default_config(level=L, eps=eps))
p = h2.plan(hm)
x = torch.randn(mesh.nt, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
for _ in range(5): p.run(x, y)
torch.cuda.synchronize()
phases = p.phases
acc = {}
for rep in range(15):
    evs = []
    for i, P in enumerate(phases):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); p._launch(P, stream_handle()); b.record(); evs.append((i, P, a, b))
    torch.cuda.synchronize()
    if rep >= 5:
        for i, P, a, b in evs:
            acc.setdefault(i, []).append(a.elapsed_time(b))
tot = 0
for i, P in enumerate(phases):
    t = np.median(acc[i]); tot += t
    print("%2d %-10s h%-2d items %6d red %5d  %7.1f us  %6.1f MB  %6.0f GB/s" % (i, P.name, P.height, P.nitems, P.nred, 1e3 * t, P.bytes / 1e6, P.bytes / (t * 1e-3) / 1e9))
print("sum of phases %.1f us" % (1e3 * tot))
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50): p.run(x, y)
b.record(); torch.cuda.synchronize()
print("graph %.1f us/mvm  -> %.0f GB/s" % (a.elapsed_time(b) / 50 * 1e3, (h2.storage_report(hm)["total"] + 16 * mesh.nt) / (a.elapsed_time(b) / 50 * 1e-3) / 1e9))
