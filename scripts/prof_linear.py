"""cProfile of a linear-basis GCA-H2 build (sphere L5)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1810_08429_b200 import cli, geometry
mesh = geometry.build_sphere_mesh(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
cfg = cli.default_config(eps=1e-4, basis="linear")
cli.build_h2_operator(mesh, cfg)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
t0 = time.perf_counter()
cli.build_h2_operator(mesh, cfg)
torch.cuda.synchronize()
pr.disable()
print("total %.3f" % (time.perf_counter() - t0))
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
