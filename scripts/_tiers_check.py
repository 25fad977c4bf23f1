import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1810_08429_b200 import cli, geometry, h2
for L, eps in [(4, 1e-4), (6, 1e-6)]:
    mesh = geometry.build_sphere_mesh(L)
    hm, _, _ = cli.build_h2_operator(mesh, cli.default_config(level=L, eps=eps))
    x = torch.randn(mesh.nt, dtype=torch.float64, device="cuda")
    ys = {}
    for mode in ["off", "auto", "0,1,2,3,4,5,6,7,8,9,10", "3,7", "2,5,8"]:
        os.environ["GC_TIERS"] = mode
        t0 = time.perf_counter()
        p = h2.PanelPlan(hm)
        p.capture()
        torch.cuda.synchronize()
        tp = time.perf_counter() - t0
        y = torch.empty_like(x)
        p.run(x, y)
        for _ in range(5): p.run(x, y)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(50): p.run(x, y)
        e1.record(); torch.cuda.synchronize()
        ys[mode] = y.clone()
        ys_s = torch.empty_like(x); p.run(x, ys_s, serial=True)
        rel = ((y - ys["off"]).norm() / ys["off"].norm()).item()
        print(L, mode, p.tiers, "plan %.3fs" % tp, "%.1f us" % (e0.elapsed_time(e1) * 1e3 / 50), "rel %.2e" % rel,
              "graph==serial", bool(torch.equal(y, ys_s)), flush=True)
