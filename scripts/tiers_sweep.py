import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1810_08429_b200 import cli, geometry, h2
L, eps = int(sys.argv[1]), float(sys.argv[2])
confs = sys.argv[3].split(";")
mesh = (geometry.build_cube_mesh if os.environ.get("GC_SWEEP_GEO") == "cube" else geometry.build_sphere_mesh)(L)
hm, _, _ = cli.build_h2_operator(mesh, cli.default_config(level=L, eps=eps))
nbytes = h2.storage_report(hm)["total"] + 16 * mesh.nt
x = torch.randn(mesh.nt, dtype=torch.float64, device="cuda")
ref = None
for conf in confs:
    for kv in conf.split():
        k, v = kv.split("=")
        os.environ[k] = v
    p = h2.PanelPlan(hm); p.capture()
    y = torch.empty_like(x)
    for _ in range(5): p.run(x, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for r in range(3):
        torch.cuda.synchronize(); e0.record()
        for _ in range(50): p.graph.replay()
        e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3 / 50)
    ref = y.clone() if ref is None else ref
    rel = ((y - ref).norm() / ref.norm()).item()
    t = min(ts)
    print("L%d %-40s tiers=%s  %.1f us  %.0f GB/s  rel %.1e" % (L, conf, p.tiers and (p.tiers["col"], p.tiers["row"]), t, nbytes / t / 1e3, rel), flush=True)
