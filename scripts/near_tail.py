"""Product time vs the share of near-field bytes launched after the coupling
(PanelPlan(near_tail=f)).  Usage: python scripts/near_tail.py level:eps ..."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_08429_b200 import cli, geometry, h2  # noqa: E402

fracs = [float(f) for f in os.environ.get("FRACS", "0,0.15,0.3,0.45,0.6").split(",")]
for spec in sys.argv[1:]:
    L, eps = spec.split(":")
    L, eps = int(L), float(eps)
    mesh = geometry.build_sphere_mesh(L)
    hm, _, _ = cli.build_h2_operator(mesh, cli.default_config(eps=eps))
    nbytes = h2.storage_report(hm)["total"] + 16 * mesh.nt
    x = torch.randn(mesh.nt, dtype=torch.float64, device="cuda")
    ref = None
    res = {f: [] for f in fracs}
    plans = {}
    for f in fracs:
        p = h2.PanelPlan(hm, near_tail=f)
        p.capture()
        plans[f] = p
    reps = 50 if L <= 7 else 10
    for rnd in range(3):
        for f in fracs:
            p = plans[f]
            y = torch.empty_like(x)
            for _ in range(3):
                p.run(x, y)
            torch.cuda.synchronize()
            if ref is None:
                ref = y.clone()
            err = float((y - ref).norm() / ref.norm())
            assert err < 1e-14, err
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                p.run(x, y)
            b.record()
            torch.cuda.synchronize()
            res[f].append(a.elapsed_time(b) / reps * 1e3)
    for f in fracs:
        t = min(res[f])
        print("L%d eps %g near_tail %.2f  product %8.1f us  %6.0f GB/s" % (L, eps, f, t, nbytes / t / 1e3), flush=True)
    del plans, hm
    torch.cuda.empty_cache()
