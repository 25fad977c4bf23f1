"""cProfile of one warm C2 assembly (build_h2_operator + plan), top entries."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1810_08429_b200 import cli, geometry, h2
L = int(sys.argv[1]) if len(sys.argv) > 1 else 6
mesh = geometry.build_sphere_mesh(L)
cfg = cli.default_config(eps=1e-6)
hm, _, _ = cli.build_h2_operator(mesh, cfg)
h2.plan(hm)
del hm
import gc; gc.collect()
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
tm = {}
hm, _, _ = cli.build_h2_operator(mesh, cfg, timings=tm)
h2.plan(hm)
torch.cuda.synchronize()
pr.disable()
print("total %.3f s" % (time.perf_counter() - t0), {k: round(v, 4) for k, v in tm.items()})
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
pstats.Stats(pr).sort_stats("cumulative").print_stats(45)
st = pstats.Stats(pr)
st.print_callers("argsort")
st.print_callers("reduce")
st.print_callers("_amin")
