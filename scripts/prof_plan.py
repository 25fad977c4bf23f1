"""cProfile of the host-side plan construction (h2.PanelPlan) and of the
cluster/block tree builders at a given level."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1810_08429_b200 import cli, clustering, geometry, h2
L = int(sys.argv[1]); eps = float(sys.argv[2]); geo = sys.argv[3] if len(sys.argv) > 3 else "sphere"
mesh = geometry.build_sphere_mesh(L) if geo == "sphere" else geometry.build_cube_mesh(L)
hm, tree, bt = cli.build_h2_operator(mesh, cli.default_config(eps=eps))
torch.cuda.synchronize()
for what, fn in [("plan", lambda: h2.PanelPlan(hm)),
                 ("cluster_tree", lambda: clustering.build_cluster_tree(mesh, "constant", 16))]:
    pr = cProfile.Profile()
    t0 = time.time()
    pr.enable()
    fn()
    pr.disable()
    torch.cuda.synchronize()
    print("==== %s %.2fs" % (what, time.time() - t0))
    pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
