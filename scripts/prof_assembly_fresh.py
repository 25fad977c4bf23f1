"""Assembly time split on a FRESH mesh object (no per-mesh caches: chart
pack, vertex stars, device uploads), after a warm-up build on another mesh
object: cProfile of the host side plus the phase timings.
Usage: python scripts/prof_assembly_fresh.py LEVEL EPS"""
import cProfile
import io
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_08429_b200 import cli, geometry, h2  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 6
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
cfg = cli.default_config(eps=eps)
hm, _, _ = cli.build_h2_operator(geometry.build_sphere_mesh(level), cfg)
h2.plan(hm)
torch.cuda.synchronize()
del hm
for rep in range(2):
    mesh = geometry.build_sphere_mesh(level)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    tm = {}
    hm, _, _ = cli.build_h2_operator(mesh, cfg, timings=tm)
    t1 = time.perf_counter()
    h2.plan(hm)
    torch.cuda.synchronize()
    pr.disable()
    t2 = time.perf_counter()
    print("level %d: operator %.4f s + plan %.4f s = %.4f s   %s" % (
        level, t1 - t0, t2 - t1, t2 - t0, {k: round(v, 4) for k, v in tm.items()}))
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(45)
print(s.getvalue()[:9000])
