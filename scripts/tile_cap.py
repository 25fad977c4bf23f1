"""Product time vs the shared-memory tile of the paired tier panels
(PanelPlan(tile_cap=c): k_panel_tile stages each panel's matrix by one TMA
copy; 0 = k_panel_pair).  Results must be bitwise equal to cap 0.
Usage: CAPS=0,1664,... python scripts/tile_cap.py level:eps ..."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_08429_b200 import cli, geometry, h2  # noqa: E402
from paper_1810_08429_b200.device import stream_handle  # noqa: E402

caps = [int(f) for f in os.environ.get("CAPS", "0,1664,2112,2800,4096,8194").split(",")]
for spec in sys.argv[1:]:
    L, eps = spec.split(":")
    L, eps = int(L), float(eps)
    mesh = geometry.build_sphere_mesh(L)
    hm, _, _ = cli.build_h2_operator(mesh, cli.default_config(eps=eps))
    nbytes = h2.storage_report(hm)["total"] + 16 * mesh.nt
    x = torch.randn(mesh.nt, dtype=torch.float64, device="cuda")
    ref = None
    res = {c: [] for c in caps}
    plans = {}
    for c in caps:
        p = h2.PanelPlan(hm, tile_cap=c)
        p.capture()
        plans[c] = p
    reps = 50 if L <= 7 else 10
    flush = torch.empty(32 << 20, dtype=torch.float64, device="cuda")
    alone = {}
    for rnd in range(3):
        for c in caps:
            p = plans[c]
            y = torch.empty_like(x)
            for _ in range(3):
                p.run(x, y)
            torch.cuda.synchronize()
            if ref is None:
                ref = y.clone()
            assert torch.equal(y, ref), (c, float((y - ref).norm() / ref.norm()))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                p.run(x, y)
            b.record()
            torch.cuda.synchronize()
            res[c].append(a.elapsed_time(b) / reps * 1e3)
            if rnd == 0:
                tl = []
                for P in p.phases:
                    if not P.pair:
                        continue
                    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                          for _ in range(10)]
                    for e0, e1 in ev:
                        flush.zero_()
                        e0.record()
                        p._launch(P, stream_handle())
                        e1.record()
                    torch.cuda.synchronize()
                    tl.append("%s%d %.1f (tile %d)" % (P.name[0], P.height,
                                                       np.median([e0.elapsed_time(e1) for e0, e1 in ev]) * 1e3, P.tile))
                alone[c] = ", ".join(tl)
    for c in caps:
        t = min(res[c])
        print("L%d eps %g tile_cap %5d  product %8.1f us  %6.0f GB/s | %s" % (L, eps, c, t, nbytes / t / 1e3, alone[c]),
              flush=True)
    del plans, hm
    torch.cuda.empty_cache()
