"""The first assembly in a process (cold: fresh device and pinned-host
allocations, lazy module loading) against a second one, phase by phase.
Usage: python scripts/cold_build.py LEVEL EPS"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_08429_b200 import cli, geometry, h2  # noqa: E402

L, eps = int(sys.argv[1]), float(sys.argv[2])
cfg = cli.default_config(eps=eps)
torch.cuda.init()
torch.empty(1, device="cuda")
for tag in ("cold", "warm"):
    mesh = geometry.build_sphere_mesh(L)
    torch.cuda.synchronize()
    tm = {}
    t0 = time.perf_counter()
    hm, _, _ = cli.build_h2_operator(mesh, cfg, timings=tm)
    t1 = time.perf_counter()
    p = h2.plan(hm)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print("%s: %.3f s = operator %.3f + plan %.3f  %s  plan %s  reserved %.1f GB" % (
        tag, t2 - t0, t1 - t0, t2 - t1, {k: round(v, 3) for k, v in tm.items()},
        {k: round(v, 3) for k, v in p.timing.items()}, torch.cuda.memory_reserved() / 1e9), flush=True)
    del hm, p
    import gc
    gc.collect()
    torch.cuda.synchronize()
