"""ncu target: the dominant launch of the product (the largest coupling
launch) alone, after a write flush of L2, inside an NVTX range "dominant"
(ncu --nvtx --nvtx-include "dominant/"), plus the whole product once in an
NVTX range "product".  Usage: python scripts/prof_dominant.py LEVEL EPS"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_08429_b200 import cli, geometry, h2  # noqa: E402
from paper_1810_08429_b200.device import stream_handle  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 6
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
hm, _, _ = cli.build_h2_operator(geometry.build_sphere_mesh(L), cli.default_config(eps=eps))
p = h2.plan(hm)
x = torch.randn(hm.shape[1], dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    p.run(x, y)
torch.cuda.synchronize()
big = max((P for P in p.phases if P.name == "coupling"), key=lambda P: P.bytes)
flush = torch.empty(32 << 20, dtype=torch.float64, device="cuda")
for _ in range(2):
    flush.zero_()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("dominant")
    p._launch(big, stream_handle())
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
torch.cuda.nvtx.range_push("product")
p.run(x, y)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("done", big.name, big.height, big.nitems, big.bytes, "ring" if big.ring else "panelmv")
