import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1810_08429_b200 import cli, geometry, h2
L = int(sys.argv[1]) if len(sys.argv) > 1 else 6
mesh = geometry.build_sphere_mesh(L)
hm, tree, bt = cli.build_h2_operator(mesh, cli.default_config(eps=1e-6))
t0 = time.time(); p = h2.PersistentPlan(hm); print("plan build %.3fs" % (time.time() - t0), p.counts, "items", p.nitems, "max_rows", p.max_rows)
x = torch.randn(mesh.nt, dtype=torch.float64, device="cuda")
ref = h2.PanelPlan(hm); yr = torch.empty_like(x); ref.run(x, yr)
y = torch.empty_like(x)
p.run(x, y); torch.cuda.synchronize()
print("max abs diff vs PanelPlan", float((y - yr).abs().max()), "rel", float((y - yr).norm() / yr.norm()))
nbytes = h2.storage_report(hm)["total"] + 16 * mesh.nt
for grid in (0, 296, 444):
    p.grid = grid
    for _ in range(3): p.run(x, y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50): p.run(x, y)
    b.record(); torch.cuda.synchronize()
    us = a.elapsed_time(b) / 50 * 1e3
    print("grid %d: %.1f us/mvm -> %.0f GB/s" % (grid, us, nbytes / (us * 1e-6) / 1e9))
p.grid = 0
g = p.capture()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50): p.run(x, y)
b.record(); torch.cuda.synchronize()
us = a.elapsed_time(b) / 50 * 1e3
print("graph: %.1f us/mvm -> %.0f GB/s" % (us, nbytes / (us * 1e-6) / 1e9))
# item timeline
p.timing = torch.zeros(3 * p.nitems + 1, dtype=torch.int64, device="cuda")
p.graph = None
for _ in range(3): p.run(x, y)
torch.cuda.synchronize()
tm = p.timing.cpu().numpy()
t0 = tm[3 * p.nitems]
tm = (tm[:3 * p.nitems].reshape(-1, 3) - t0) / 1e3
it = p.items.cpu().numpy()
k = 0
agg = {}
for name, cnt in p.segments:
    seg = tm[k:k + cnt]
    k += cnt
    if not cnt: continue
    a = agg.setdefault(name, [])
    a.append(seg)
for name, segs in agg.items():
    seg = np.concatenate(segs)
    print("%-8s n=%5d  run %7.1f..%7.1f  done max %7.1f  mean run %.2f us  mean wait %.2f" % (
        name, len(seg), seg[:, 1].min(), seg[:, 1].max(), seg[:, 2].max(), (seg[:, 2] - seg[:, 1]).mean(), (seg[:, 1] - seg[:, 0]).mean()))
