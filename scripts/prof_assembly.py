import cProfile, pstats, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1810_08429_b200 import cli, geometry
L = int(sys.argv[1]) if len(sys.argv) > 1 else 6
mesh = geometry.build_sphere_mesh(L)
cfg = cli.default_config(eps=1e-6)
for _ in range(2):
    hm = cli.build_h2_operator(mesh, cfg)[0]; torch.cuda.synchronize(); del hm
t = time.time()
pr = cProfile.Profile(); pr.enable()
hm = cli.build_h2_operator(mesh, cfg)[0]; torch.cuda.synchronize()
pr.disable()
print("wall %.3f" % (time.time() - t))
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
