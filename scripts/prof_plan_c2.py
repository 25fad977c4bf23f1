"""cProfile of h2.plan alone (fresh operator after a warm-up build): the
matvec plan's host cost by function.  Usage: python scripts/prof_plan_c2.py LEVEL EPS"""
import cProfile
import io
import os
import pstats
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_08429_b200 import cli, geometry, h2  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 6
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
cfg = cli.default_config(eps=eps)
hm, _, _ = cli.build_h2_operator(geometry.build_sphere_mesh(L), cfg)
h2.plan(hm)
hm, _, _ = cli.build_h2_operator(geometry.build_sphere_mesh(L), cfg)
hm.settle()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
p = h2.plan(hm)
torch.cuda.synchronize()
pr.disable()
print("plan timing:", {k: round(v, 4) for k, v in p.timing.items()})
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(35)
print(s.getvalue()[:9000])
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(45)
print(s.getvalue()[:9000])
