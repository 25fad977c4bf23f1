"""One C2-style assembly (after a warm-up on another mesh object) inside
an NVTX range "assembly" - an ncu / launch-list target.
Usage: python scripts/assembly_once.py LEVEL EPS"""
import gc
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_08429_b200 import cli, geometry, h2  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 6
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
cfg = cli.default_config(eps=eps)
hm, _, _ = cli.build_h2_operator(geometry.build_sphere_mesh(level), cfg)
h2.plan(hm)
del hm
gc.collect()
torch.cuda.synchronize()
mesh = geometry.build_sphere_mesh(level)
torch.cuda.nvtx.range_push("assembly")
hm, _, _ = cli.build_h2_operator(mesh, cfg)
h2.plan(hm)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
