"""Product time for values of one h2 module constant (plan-construction
parameters under study).  Usage: python scripts/modvar.py NAME v1,v2,... level:eps ... (cubeL:eps for the cube)"""
import ast
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_08429_b200 import cli, geometry, h2, tiers  # noqa: E402

name, vals = sys.argv[1], sys.argv[2].split(",")


def conv(v):
    try:
        return ast.literal_eval(v)
    except (ValueError, SyntaxError):
        return v


vals = [conv(v) for v in vals]
for spec in sys.argv[3:]:
    L, eps = spec.split(":")
    cube = L.startswith("cube")
    L, eps = int(L[4:] if cube else L), float(eps)
    mesh = geometry.build_cube_mesh(L) if cube else geometry.build_sphere_mesh(L)
    hm, _, _ = cli.build_h2_operator(mesh, cli.default_config(eps=eps))
    nbytes = h2.storage_report(hm)["total"] + 16 * mesh.nt
    x = torch.randn(mesh.nt, dtype=torch.float64, device="cuda")
    plans, res, ref = [], [[] for _ in vals], None
    mod = next(m for m in (h2, tiers) if hasattr(m, name))
    old = getattr(mod, name)
    for v in vals:
        setattr(mod, name, v)
        p = h2.PanelPlan(hm)
        p.capture()
        plans.append(p)
    setattr(mod, name, old)
    reps = 50 if L <= 7 else 10
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
    from paper_1810_08429_b200.device import stream_handle
    import numpy as np
    flush = torch.empty(32 << 20, dtype=torch.float64, device="cuda")
    for v, r, p in zip(vals, res, plans):
        big = max((P for P in p.phases if P.name == "coupling"), key=lambda P: P.bytes)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
        for e0, e1 in ev:
            flush.zero_()
            e0.record()
            p._launch(big, stream_handle())
            e1.record()
        torch.cuda.synchronize()
        tb = np.median([e0.elapsed_time(e1) for e0, e1 in ev]) * 1e3
        bb = big.bytes + 8 * big.in_elems + 8 * big.out_elems
        print("L%d eps %g %s=%-10s product %8.1f us  %6.0f GB/s   largest coupling launch alone %6.1f us %6.0f GB/s"
              % (L, eps, name, v, min(r), nbytes / min(r) / 1e3, tb, bb / tb / 1e3), flush=True)
    del plans, hm
    torch.cuda.empty_cache()
