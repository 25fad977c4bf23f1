"""Micro-timings of the transform chain: grid barrier cost, and each chain
level run through the co-resident chain kernel vs the one-CTA-per-item
kernel, every measurement a CUDA graph of R back-to-back copies."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1810_08429_b200 import _native, cli, geometry, h2
from paper_1810_08429_b200.device import ptr, stream_handle, to_dev

L = int(sys.argv[1]) if len(sys.argv) > 1 else 6
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
mesh = geometry.build_sphere_mesh(L)
hm, tree, bt = cli.build_h2_operator(mesh, cli.default_config(level=L, eps=eps))
p = h2.plan(hm)
R = 20


def per_call(fn, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(R):
            fn()
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / R * 1e3


def seg(phases):
    def addr(t):
        return ptr(t).value or 0
    desc = np.array([[addr(P.items), P.nitems, addr(P.xidx), addr(P.A0), addr(P.A1), addr(P.in0),
                      addr(P.in1), addr(P.out), addr(P.scratch), addr(P.red), addr(P.arrivals), 0]
                     for P in phases], dtype=np.uint64)
    d = to_dev(desc.view(np.int64), p.dev)
    return d


empty = []
for P in p._fwd[:1]:
    E = h2._Phase()
    for k in P.__slots__:
        setattr(E, k, getattr(P, k))
    E.nitems = 0
    empty = [E] * 9
d_empty = seg(empty)
print("grid %d CTAs" % p._chain_grid)
for n in (1, 2, 5, 9):
    t = per_call(lambda: _native.call("gc_panel_chain", n, ptr(d_empty), p._chain_grid, ptr(p._barrier),
                                      stream_handle()))
    print("chain kernel, %d empty phases: %6.2f us" % (n, t))
print("level              items    MB   chain-kernel  cta-kernel(PDL)  cta-kernel")
for P in p._fwd + [b for b, _ in p._bwd]:
    d = seg([P])
    t1 = per_call(lambda: _native.call("gc_panel_chain", 1, ptr(d), p._chain_grid, ptr(p._barrier),
                                       stream_handle()))
    t2 = per_call(lambda: p._launch(P, stream_handle(), True))
    t3 = per_call(lambda: p._launch(P, stream_handle(), False))
    print("%-9s h%-2d %7d %6.1f   %8.2f us   %8.2f us   %8.2f us" % (P.name, P.height, P.nitems, P.bytes / 1e6,
                                                                  t1, t2, t3))
