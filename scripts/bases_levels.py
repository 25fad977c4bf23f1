"""Device time of the per-level launches of the nested bases (green box
rules, factor, ACA, bookkeeping), CUDA events around each native call.
Usage: python scripts/bases_levels.py LEVEL EPS"""
import os
import sys
from collections import defaultdict

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_08429_b200 import _native, cli, geometry, h2  # noqa: E402

L, eps = int(sys.argv[1]), float(sys.argv[2])
cfg = cli.default_config(eps=eps)
hm, _, _ = cli.build_h2_operator(geometry.build_sphere_mesh(L), cfg)
h2.plan(hm)
torch.cuda.synchronize()
rec = []
orig = _native.call


def timed(name, *args):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    r = orig(name, *args)
    b.record()
    extra = ""
    if name == "gc_aca":
        extra = "nn=%d max_rows=%d" % (args[0], args[10])
    rec.append((name, a, b, extra))
    return r


_native.call = timed
hm, _, _ = cli.build_h2_operator(geometry.build_sphere_mesh(L), cfg)
torch.cuda.synchronize()
tot = defaultdict(float)
for name, a, b, extra in rec:
    t = a.elapsed_time(b)
    tot[name] += t
    if name in ("gc_aca", "gc_green_factor"):
        print("%-20s %8.3f ms %s" % (name, t, extra))
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print("total %-24s %8.3f ms" % (k, v))
