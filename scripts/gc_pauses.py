"""Python GC pauses during the timed assembly (bench.py's sequence: a
warm-up build, gc.collect, then fresh-mesh builds), per generation.
Usage: python scripts/gc_pauses.py LEVEL EPS [reps]"""
import gc
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_08429_b200 import cli, geometry, h2  # noqa: E402

L, eps = int(sys.argv[1]), float(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
cfg = cli.default_config(eps=eps)
pauses, t_start = [], [0.0]


def cb(phase, info):
    if phase == "start":
        t_start[0] = time.perf_counter()
    else:
        pauses.append((info["generation"], time.perf_counter() - t_start[0]))


hm, _, _ = cli.build_h2_operator(geometry.build_sphere_mesh(L), cfg)
h2.plan(hm)
del hm
gc.collect()
torch.cuda.synchronize()
print("tracked objects after warm-up:", len(gc.get_objects()))
gc.callbacks.append(cb)
from paper_1810_08429_b200 import clustering  # noqa: E402
_bt = clustering._build_block_tree_device
seg = {}


def _bt_wrapped(*a, **k):
    s0 = torch.cuda.memory_stats().get("segment.all.allocated", 0)
    t = time.perf_counter()
    r = _bt(*a, **k)
    seg["bt"] = (torch.cuda.memory_stats().get("segment.all.allocated", 0) - s0, time.perf_counter() - t)
    return r


clustering._build_block_tree_device = _bt_wrapped
for r in range(reps):
    s_before = torch.cuda.memory_stats().get("segment.all.allocated", 0)
    mesh = geometry.build_sphere_mesh(L)
    pauses.clear()
    tm = {}
    t0 = time.perf_counter()
    hm, _, _ = cli.build_h2_operator(mesh, cfg, timings=tm)
    h2.plan(hm)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    g2 = [p for g, p in pauses if g == 2]
    print("   new cudaMalloc segments: build %d, block tree %d (%.4f s)" % (
        torch.cuda.memory_stats().get("segment.all.allocated", 0) - s_before, *seg.get("bt", (0, 0))))
    print("rep %d: %.4f s  block_tree %.4f  gc pauses: %d (gen2 %d, %.2f ms total, gen2 %.2f ms)" % (
        r, t, tm.get("block_tree_s", 0), len(pauses), len(g2), 1e3 * sum(p for _, p in pauses), 1e3 * sum(g2)))
    del hm
    gc.collect()
    torch.cuda.synchronize()
