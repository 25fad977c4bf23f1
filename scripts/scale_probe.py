"""Assembly + matvec at a given level (timings per phase)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1810_08429_b200 import cli, geometry, h2
L = int(sys.argv[1]); eps = float(sys.argv[2]); geo = sys.argv[3] if len(sys.argv) > 3 else "sphere"
t0 = time.time()
mesh = geometry.build_sphere_mesh(L) if geo == "sphere" else geometry.build_cube_mesh(L)
print("mesh %.2fs nt=%d" % (time.time() - t0, mesh.nt), flush=True)
for rep in range(2):
    tm = {}
    t0 = time.time()
    hm, tree, bt = cli.build_h2_operator(mesh, cli.default_config(eps=eps), timings=tm)
    torch.cuda.synchronize()
    print("assembly %.3fs" % (time.time() - t0), {k: round(v, 3) for k, v in tm.items()}, flush=True)
    print("  row basis", {k: round(v, 3) for k, v in hm.row_basis.store.timing.items()}, "build_h2", {k: round(v, 3) for k, v in hm.dev.timing.items()}, flush=True)
rep = h2.storage_report(hm)
print("storage MB", {k: round(v / 1e6, 1) for k, v in rep.items()}, "blocks", len(hm.coupling), len(hm.nearfield), flush=True)
t0 = time.time(); p = h2.PanelPlan(hm); torch.cuda.synchronize(); t1 = time.time()
p.capture(); torch.cuda.synchronize(); t2 = time.time()
print("plan %.2fs  capture %.2fs" % (t1 - t0, t2 - t1), flush=True)
x = torch.randn(mesh.nt, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
for _ in range(3): p.run(x, y)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): p.run(x, y)
b.record(); torch.cuda.synchronize()
us = a.elapsed_time(b) / 10 * 1e3
print("matvec %.1f us -> %.0f GB/s" % (us, (rep["total"] + 16 * mesh.nt) / (us * 1e-6) / 1e9), flush=True)
print("mem GB", torch.cuda.max_memory_allocated() / 1e9)
