"""Short profiling target (C2): one assembly, then NVTX-ranged kernels:
'coupling' = the coupling panel product, 'nearq' = near-field quadrature,
'mvm' = 3 graph-replayed matvecs, 'tiers' = the tier transforms once each.  Used under ncu; prints nothing heavy."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1810_08429_b200 import cli, geometry, h2
from paper_1810_08429_b200.assembly import device_block_assembly
from paper_1810_08429_b200.device import DeviceMesh, DeviceRules, SingularQueue, stream_handle
L = int(os.environ.get("PROF_LEVEL", "6"))
mesh = geometry.build_sphere_mesh(L)
hm, tree, bt = cli.build_h2_operator(mesh, cli.default_config(eps=1e-6))
p = h2.plan(hm, graph=False) if False else h2.PanelPlan(hm)
x = torch.randn(mesh.nt, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
p.run(x, y); torch.cuda.synchronize()
torch.cuda.nvtx.range_push("mvm")
for _ in range(3):
    p.run(x, y)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
coup = max((P for P in p.phases if P.name == "coupling"), key=lambda P: P.bytes)
torch.cuda.nvtx.range_push("coupling")
for _ in range(3):
    p._launch(coup, stream_handle())
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
torch.cuda.nvtx.range_push("tiers")          # the tier transforms, each once, as chain launches
for P in p._fwd + [b for b, _ in p._bwd] + [b for b, _ in p._leafparts]:
    p._launch(P, stream_handle(), True, 0)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
d = hm.dev
dm, rules, q = DeviceMesh.get(mesh, 3, d.device), DeviceRules.get(5, d.device), SingularQueue.get(mesh, d.device)
ndesc = np.stack([tree.flat.start[d.n_rows], d.n_nr, tree.flat.start[d.n_cols], d.n_nc, d.n_off], 1)
scratch = torch.empty_like(d.near)
torch.cuda.nvtx.range_push("nearq")
device_block_assembly(dm, rules, q, d.perm_r, d.perm_c, ndesc, scratch)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("prof target done", mesh.nt)
