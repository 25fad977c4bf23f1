"""Host cost of plan construction and graph capture, first and second time
in a process (bench.py's sequence: warm-up assembly + plan, then timed)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1810_08429_b200 import cli, geometry, h2
L = int(sys.argv[1]); eps = float(sys.argv[2]); geo = sys.argv[3] if len(sys.argv) > 3 else "sphere"
mesh = geometry.build_sphere_mesh(L) if geo == "sphere" else geometry.build_cube_mesh(L)
cfg = cli.default_config(eps=eps)
for rep in range(3):
    hm, tree, bt = cli.build_h2_operator(mesh, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = h2.PanelPlan(hm)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    p.capture()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print("rep %d: plan %.3f s  capture %.3f s" % (rep, t1 - t0, t2 - t1), flush=True)
    del p, hm
