import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import golden, mesh_for, eps_of
from paper_1810_08429_b200 import cli
name = sys.argv[1]
g = golden(name); mesh = mesh_for(name)
hm, tree, bt = cli.build_h2_operator(mesh, cli.default_config(eps=eps_of(name)))
for side, basis in (("row", hm.row_basis), ("col", hm.col_basis)):
    nodes = basis.nodes()
    gi = g[side + "_node"].tolist(); gr = g[side + "_rank"].tolist()
    print(side, "nodes equal", [b.cluster.index for b in nodes] == gi)
    off = 0; ref = {}
    for i, r in zip(gi, gr):
        ref[i] = g[side + "_piv"][off:off + r]; off += r
    bad = 0
    for b in nodes:
        rp = ref[b.cluster.index]
        if not np.array_equal(b.pivots, rp):
            bad += 1
            if bad <= 5:
                print("  node", b.cluster.index, "rank", b.rank, len(rp), "first diff at", next((k for k in range(min(b.rank, len(rp))) if b.pivots[k] != rp[k]), None), "set equal", set(b.pivots) == set(rp))
    print(side, "mismatching nodes", bad, "of", len(nodes))
