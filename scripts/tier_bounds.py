"""Product time for explicit tier boundaries (PanelPlan(tiers=[...])) next
to the DP choice.  Usage: python scripts/tier_bounds.py level:eps 'b1,b2;b1,b2,b3;...'"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_08429_b200 import cli, geometry, h2  # noqa: E402

spec, sets = sys.argv[1], sys.argv[2]
L, eps = spec.split(":")
L, eps = int(L), float(eps)
mesh = geometry.build_sphere_mesh(L)
hm, _, _ = cli.build_h2_operator(mesh, cli.default_config(eps=eps))
nbytes = h2.storage_report(hm)["total"] + 16 * mesh.nt
x = torch.randn(mesh.nt, dtype=torch.float64, device="cuda")
cands = ["auto"] + [[int(v) for v in s.split(",")] for s in sets.split(";")]
plans = []
for c in cands:
    p = h2.PanelPlan(hm, tiers=c)
    p.capture()
    plans.append(p)
reps = 50 if L <= 7 else 10
res = [[] for _ in cands]
ref = None
for rnd in range(3):
    for i, p in enumerate(plans):
        y = torch.empty_like(x)
        for _ in range(3):
            p.run(x, y)
        torch.cuda.synchronize()
        if ref is None:
            ref = y.clone()
        assert float((y - ref).norm() / ref.norm()) < 1e-13
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            p.run(x, y)
        b.record()
        torch.cuda.synchronize()
        res[i].append(a.elapsed_time(b) / reps * 1e3)
for c, p, r in zip(cands, plans, res):
    t = min(r)
    print("L%d eps %g tiers %-14s (col %s)  product %8.1f us  %6.0f GB/s" % (
        L, eps, c if c == "auto" else ",".join(map(str, c)), p.tiers["col"] if p.tiers else None, t,
        nbytes / t / 1e3), flush=True)
