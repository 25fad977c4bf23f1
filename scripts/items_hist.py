import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1810_08429_b200 import cli, geometry, h2
L = int(sys.argv[1]); eps = float(sys.argv[2])
hm, _, _ = cli.build_h2_operator(geometry.build_sphere_mesh(L), cli.default_config(eps=eps))
p = h2.plan(hm)
phs = [n.phase for n in p.nodes if n.phase is not None]
big = max(phs, key=lambda P: P.bytes)
it = big.items.cpu().numpy().reshape(-1, 8)
el = it[:, 3] * it[:, 4]
print("largest phase", big.name, big.height, "items", len(it), "MB", big.bytes / 1e6, "ring", big.ring, "pair", big.pair)
print("item elems: min %d p10 %d median %d p90 %d max %d mean %.0f" % (el.min(), *np.percentile(el, [10, 50, 90]).astype(int), el.max(), el.mean()))
direct = (it[:, 5] & 4) != 0
print("direct items", direct.sum(), "split items", (~direct).sum())
print("T values", np.unique(it[:, 3], return_counts=True))
h, e = np.histogram(el, bins=12)
print(list(zip(e.astype(int), h)))
print("sum elems", el.sum(), "per 888 slots", el.sum() / 888)
