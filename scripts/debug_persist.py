import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1810_08429_b200 import cli, geometry, h2
mesh = geometry.build_sphere_mesh(5)
hm, tree, bt = cli.build_h2_operator(mesh, cli.default_config(eps=1e-6))
p = h2.PersistentPlan(hm)
it = p.items.cpu().numpy()
k = 0
for name, cnt in p.segments:
    w7 = it[k, 7]; w1 = w7 & 0xffffffff; w2 = (w7 >> 32) & 0xffffffff
    w6 = it[k, 6]
    print("%-7s n=%5d  wait1 ctr %3d tgt %6d | wait2 ctr %3d tgt %6d | sig %3d %3d" % (name, cnt, w1 >> 24, w1 & 0xffffff, w2 >> 24, w2 & 0xffffff, (w6 >> 32) & 0xff, (w6 >> 40) & 0xff))
    k += cnt
x = torch.randn(mesh.nt, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
p.run(x, y); torch.cuda.synchronize()
s = p.sync.cpu().numpy()
print("counters", {i: int(s[1 + i]) for i in range(0, 90) if s[1 + i]})
