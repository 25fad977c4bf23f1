"""Product time of one library build (GC_LIB) at a few sphere levels:
graph replay (CUDA events, 3 x 50 replays, best of 3) and the largest
coupling launch alone after a 256 MB write flush.  Usage:
GC_LIB=... python scripts/kvar.py tag level:eps [level:eps ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_08429_b200 import cli, geometry, h2  # noqa: E402
from paper_1810_08429_b200.device import stream_handle  # noqa: E402

tag = sys.argv[1]
for spec in sys.argv[2:]:
    L, eps = spec.split(":")
    L, eps = int(L), float(eps)
    mesh = geometry.build_sphere_mesh(L)
    hm, _, _ = cli.build_h2_operator(mesh, cli.default_config(eps=eps))
    nbytes = h2.storage_report(hm)["total"] + 16 * mesh.nt
    p = h2.plan(hm)
    x = torch.randn(mesh.nt, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(5):
        p.run(x, y)
    torch.cuda.synchronize()
    reps = 50 if L <= 7 else 10
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            p.run(x, y)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / reps * 1e3)
    big = max((P for P in p.phases if P.name == "coupling"), key=lambda P: P.bytes)
    flush = torch.empty(32 << 20, dtype=torch.float64, device="cuda")
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
    for e0, e1 in ev:
        flush.zero_()
        e0.record()
        p._launch(big, stream_handle())
        e1.record()
    torch.cuda.synchronize()
    tb = np.median([e0.elapsed_time(e1) for e0, e1 in ev]) * 1e3
    bb = big.bytes + 8 * big.in_elems + 8 * big.out_elems
    tiers = []
    for P in p.phases:
        if not getattr(P, "pair", False):
            continue
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
        for e0, e1 in ev:
            flush.zero_()
            e0.record()
            p._launch(P, stream_handle())
            e1.record()
        torch.cuda.synchronize()
        tiers.append("%s%d %.1f" % (P.name[0], P.height, np.median([e0.elapsed_time(e1) for e0, e1 in ev]) * 1e3))
    print("%-10s L%d eps %g  product %8.1f us  %6.0f GB/s   big %7.1f us %6.0f GB/s (ring %d)" % (
        tag, L, eps, min(ts), nbytes / min(ts) / 1e3, tb, bb / tb / 1e3, int(bool(big.ring))), " | pair phases alone (us):", ", ".join(tiers), flush=True)
    del p, hm
    torch.cuda.empty_cache()
