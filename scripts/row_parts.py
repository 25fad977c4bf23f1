"""Product time vs the number of row parts (independent coupling / backward / leaf chains)
(PanelPlan(parts=p)).  Usage: python scripts/row_parts.py level:eps ..."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_08429_b200 import cli, geometry, h2  # noqa: E402

fracs = [int(f) for f in os.environ.get("PARTS", "1,2,4,8").split(",")]
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
        p = h2.PanelPlan(hm, parts=f)
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
        pb = plans[f]._pbounds
        print("L%d eps %g parts %d (%d)  product %8.1f us  %6.0f GB/s" % (L, eps, f, 1 if pb is None else len(pb), t,
                                                                        nbytes / t / 1e3), flush=True)
    del plans, hm
    torch.cuda.empty_cache()
