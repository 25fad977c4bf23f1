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
from paper_1810_08429_b200 import _native, cli, geometry, h2  # noqa: E402

_calls = {}
_orig_call = _native.call


def _timed_call(name, *args):
    t = time.perf_counter()
    try:
        return _orig_call(name, *args)
    finally:
        c = _calls.setdefault(name, [0, 0.0])
        c[0] += 1
        c[1] += time.perf_counter() - t


_native.call = _timed_call

level = int(sys.argv[1]) if len(sys.argv) > 1 else 6
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
cfg = cli.default_config(eps=eps)
hm, _, _ = cli.build_h2_operator(geometry.build_sphere_mesh(level), cfg)
h2.plan(hm)
torch.cuda.synchronize()
del hm
import gc
gc.collect()                     # as bench.py: the warm-up operator's blocks return to the allocator
torch.cuda.synchronize()
for rep in range(1):
    _calls.clear()
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
    print("plan timing:", {k: round(v, 4) for k, v in h2.plan(hm).timing.items()})
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(40)
print(s.getvalue()[:8000])
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(30)
print(s.getvalue()[:7000])
s = io.StringIO()
st = pstats.Stats(pr, stream=s)
st.sort_stats("tottime").print_callers("argsort|_native.py:138|method 'cpu'|method 'to' of|stack|tolist")
print(s.getvalue()[:12000])
callees = os.environ.get("PROF_CALLEES")
if callees:
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("cumulative").print_callees(callees)
    print(s.getvalue()[:20000])
print("native calls (count, s):")
for k, (n, t) in sorted(_calls.items(), key=lambda kv: -kv[1][1])[:20]:
    print("  %-28s %5d %8.4f" % (k, n, t))
