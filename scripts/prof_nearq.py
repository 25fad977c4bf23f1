"""Near-field quadrature time at C2 (block kernel + singular flush), the
descriptor pre-uploaded; median of 7."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1810_08429_b200 import cli, geometry
from paper_1810_08429_b200.assembly import device_block_assembly
from paper_1810_08429_b200.device import DeviceMesh, DeviceRules, SingularQueue, to_dev
mesh = geometry.build_sphere_mesh(6)
hm, tree, bt = cli.build_h2_operator(mesh, cli.default_config(eps=1e-6))
d = hm.dev
dm, rules, q = DeviceMesh.get(mesh, 3, d.device), DeviceRules.get(5, d.device), SingularQueue.get(mesh, d.device)
ndesc = np.stack([tree.flat.start[d.n_rows], d.n_nr, tree.flat.start[d.n_cols], d.n_nc, d.n_off], 1)
dd = to_dev(ndesc.astype(np.int64), d.device)
out = torch.empty_like(d.near)
ts = []
for _ in range(8):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    device_block_assembly(dm, rules, q, d.perm_r, d.perm_c, ndesc, out, d_desc=dd)
    b.record(); b.synchronize()
    ts.append(a.elapsed_time(b))
print("nearq %.3f ms" % np.median(ts[1:]), "bitwise", torch.equal(out, d.near))
