import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1810_08429_b200 import cli, geometry, h2
L = int(sys.argv[1]) if len(sys.argv) > 1 else 6
mesh = geometry.build_sphere_mesh(L)
hm, tree, bt = cli.build_h2_operator(mesh, cli.default_config(eps=1e-6))
p = h2.PersistentPlan(hm)
print("stage sizes", p.stage_sizes)
x = torch.randn(mesh.nt, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
p.timing = torch.zeros(2 * len(p.stage_sizes) + 4, dtype=torch.int64, device="cuda")
for grid in (0, 148, 296, 444, 592):
    p.grid = grid
    for _ in range(3): p.run(x, y)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        p.run(x, y); torch.cuda.synchronize(); ts.append(p.timing.cpu().numpy().copy())
    t = np.median(np.array(ts), axis=0)
    t = t - t[0]
    n = len(p.stage_sizes)
    work = [t[2 + 2 * s] - t[1 + 2 * s] for s in range(n)]
    bar = [t[3 + 2 * s] - t[2 + 2 * s] for s in range(n - 1)]
    print("grid", grid, "total %.1f us" % (t[2 * n] / 1e3), "stage0 %.1f" % (t[1] / 1e3))
    print("  work us ", " ".join("%.1f" % (w / 1e3) for w in work))
    print("  barrier ", " ".join("%.1f" % (b / 1e3) for b in bar))
