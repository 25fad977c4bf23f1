import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1810_08429_b200 import cli, geometry, h2
L = int(sys.argv[1]) if len(sys.argv) > 1 else 6
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
mesh = geometry.build_sphere_mesh(L)
hm, tree, bt = cli.build_h2_operator(mesh, cli.default_config(eps=eps))
nbytes = h2.storage_report(hm)["total"] + 16 * mesh.nt
x = torch.randn(mesh.nt, dtype=torch.float64, device="cuda")
ref = h2.PanelPlan(hm); yr = torch.empty_like(x)
for cls in (h2.PanelPlan, h2.LaunchPlan):
    p = cls(hm); y = torch.empty_like(x)
    p.run(x, y); ref.run(x, yr); torch.cuda.synchronize()
    print(cls.__name__, "kernels", p.num_kernels, "rel diff", float((y - yr).norm() / yr.norm()))
    p.capture()
    for _ in range(3): p.run(x, y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50): p.run(x, y)
    b.record(); torch.cuda.synchronize()
    us = a.elapsed_time(b) / 50 * 1e3
    print("  graph %.1f us/mvm -> %.0f GB/s" % (us, nbytes / (us * 1e-6) / 1e9))
    if cls is h2.LaunchPlan:
        for name in ("fwd", "cpl", "reduce", "bwd", "final"):
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ts = []
            for _ in range(10):
                p._body(ev, name); torch.cuda.synchronize(); ts.append(ev[0].elapsed_time(ev[1]))
            print("  eager phase %-6s first-range %.1f us" % (name, 1e3 * np.median(ts)))
