"""Bulk-phase kernel variants of the product (PanelPlan(bulk="auto"|"plain"|"ring")):
whole-product graph time and the largest coupling bucket launched alone
(L2 flushed), CUDA events.  Usage: python scripts/bulk_variants.py [level eps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_08429_b200 import cli, geometry, h2  # noqa: E402
from paper_1810_08429_b200.device import stream_handle  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 6
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
mesh = geometry.build_sphere_mesh(L)
hm, _, _ = cli.build_h2_operator(mesh, cli.default_config(eps=eps))
nbytes = h2.storage_report(hm)["total"] + 16 * mesh.nt
x = torch.randn(mesh.nt, dtype=torch.float64, device="cuda")
flush = torch.empty(32 << 20, dtype=torch.float64, device="cuda")
ref = None
for bulk in ("auto", "plain", "ring"):
    p = h2.PanelPlan(hm, bulk=bulk)
    p.capture()
    y = torch.empty_like(x)
    for _ in range(5):
        p.run(x, y)
    torch.cuda.synchronize()
    if ref is None:
        ref = y.clone()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        p.run(x, y)
    b.record()
    torch.cuda.synchronize()
    t = a.elapsed_time(b) / 50 * 1e-3
    big = max((P for P in p.phases if P.name == "coupling"), key=lambda P: P.bytes)
    ts, tr = [], []
    for _ in range(8):
        # read-only sweep: evicts L2 without dirty lines to write back
        flush.sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        p._launch(big, stream_handle())
        e1.record()
        torch.cuda.synchronize()
        tr.append(e0.elapsed_time(e1) * 1e-3)
    for _ in range(8):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        p._launch(big, stream_handle())
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    tb = float(np.mean(ts[1:]))
    tbr = float(np.mean(tr[1:]))
    bb = big.bytes + 8 * big.in_elems + 8 * big.out_elems
    print("   read-sweep flush: largest bucket %6.1f us %5.0f GB/s" % (tbr * 1e6, bb / tbr / 1e9))
    print("%-6s product %6.1f us %5.0f GB/s | largest bucket %4d items %6.1f us %5.0f GB/s | diff %.1e"
          % (bulk, t * 1e6, nbytes / t / 1e9, big.nitems, tb * 1e6, bb / tb / 1e9,
             ((y - ref).norm() / ref.norm()).item()), flush=True)
