"""Developer parity probe against the real reference (baseline/_ref).
Not a test: the committed tests use oracle/ + tests/golden only."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
import greencross.geometry as RG, greencross.assembly as RA, greencross.gca as RGCA, greencross.h2 as RH
import greencross.clustering as RC, greencross.quadrature as RQ
from paper_1810_08429_b200 import geometry as G, assembly as A, gca, h2, cli, clustering as C, _native

L = int(sys.argv[1]) if len(sys.argv) > 1 else 3
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-4
mesh = G.build_sphere_mesh(L); rmesh = RG.build_sphere_mesh(L)
n = mesh.nt
rng = np.random.default_rng(0)
# 1. evaluator seam
ev = A.galerkin_pair_evaluator("slp", mesh, "constant", 3, 5)
rev = RA.galerkin_pair_evaluator("slp", rmesh, "constant", 3, 5)
cls = RA.galerkin_classify(rmesh)
rows = rng.integers(0, n, 20000); cols = rng.integers(0, n, 20000)
# add singular pairs
st = rmesh.vertex_stars()
extra_r, extra_c = [], []
for t in range(0, n, max(1, n // 200)):
    for v in rmesh.triangles[t]:
        for s in st[v]:
            extra_r.append(t); extra_c.append(s)
rows = np.concatenate([rows, extra_r]); cols = np.concatenate([cols, extra_c])
case, px, py = cls(rows, cols)
for k in range(4):
    m = case == k
    if not m.any(): continue
    a = ev(k, rows[m], cols[m], px[m], py[m]).ravel()
    b = rev(k, rows[m], cols[m], px[m], py[m]).ravel()
    print("pair case %d n=%d maxrel %.3e" % (k, m.sum(), np.max(np.abs(a - b) / np.abs(b))))
# 2. dense block
idx = np.arange(min(n, 512))
t0 = time.time(); D = A.assemble_galerkin_block("slp", mesh, "constant", idx, idx).values; t1 = time.time()
RD = RA.assemble_galerkin_block("slp", rmesh, "constant", idx, idx).values; t2 = time.time()
print("dense %d: maxrel %.3e  (dev %.3fs ref %.3fs)" % (len(idx), np.max(np.abs(D - RD)) / np.max(np.abs(RD)), t1 - t0, t2 - t1))
# 3. full H2
cfg = cli.default_config(level=L, eps=eps)
tm = {}
t0 = time.time(); hm, tree, bt = cli.build_h2_operator(mesh, cfg, timings=tm); t1 = time.time()
print("device build %.3fs" % (t1 - t0), {k: round(v, 4) for k, v in tm.items()})
rtree = RC.build_cluster_tree(rmesh, "constant", 16); rbt = RC.build_block_tree(rtree, eta=1.0)
rm, cm = RGCA.coupling_marks(rbt)
t0 = time.time()
rrb = RGCA.build_cluster_basis(rtree, rmesh, "constant", 3, 0.5, eps, "row", (3, 5), rm)
rcb = RGCA.build_cluster_basis(rtree, rmesh, "constant", 3, 0.5, eps, "col", (3, 5), cm)
t1 = time.time()
rh = RGCA.build_h2(rbt, rrb, rcb, rmesh, "slp", "constant", "galerkin", (3, 5))
t2 = time.time()
print("ref bases %.2fs build_h2 %.2fs" % (t1 - t0, t2 - t1))
print("perm equal", np.array_equal(tree.perm, rtree.perm))
for side, mine, ref in (("row", hm.row_basis, rrb), ("col", hm.col_basis, rcb)):
    nodes_m = {bn.cluster.index: bn for bn in mine.nodes()}
    nodes_r = {bn.cluster.index: bn for bn in ref.nodes()}
    assert set(nodes_m) == set(nodes_r), "materialized sets differ"
    bad_set = bad_ord = 0; vmax = 0.0
    for i, br in nodes_r.items():
        bm = nodes_m[i]
        if not np.array_equal(bm.pivots, br.pivots):
            bad_ord += 1
            if set(bm.pivots.tolist()) != set(br.pivots.tolist()): bad_set += 1
            continue
        if br.v is not None:
            vmax = max(vmax, np.max(np.abs(bm.v - br.v)) / max(np.max(np.abs(br.v)), 1e-300))
        if br.transfer is not None:
            vmax = max(vmax, np.max(np.abs(bm.transfer - br.transfer)) / max(np.max(np.abs(br.transfer)), 1e-300))
    print("%s basis: %d nodes, pivot order mismatches %d (set %d), V/transfer maxrel %.3e" % (side, len(nodes_r), bad_ord, bad_set, vmax))
cm_ = max(np.max(np.abs(a.values - b.values)) / np.max(np.abs(b.values)) for a, b in zip(hm.coupling, rh.coupling) if a.values.shape == b.values.shape)
nm_ = max(np.max(np.abs(a.values - b.values)) / np.max(np.abs(b.values)) for a, b in zip(hm.nearfield, rh.nearfield))
print("coupling blocks %d/%d maxrel %.3e ; near %d/%d maxrel %.3e" % (len(hm.coupling), len(rh.coupling), cm_, len(hm.nearfield), len(rh.nearfield), nm_))
print("storage", h2.storage_report(hm) == RH.storage_report(rh))
for trans in (False, True):
    errs = []
    for _ in range(5):
        x = rng.standard_normal(n)
        y = (h2.mvm_t if trans else h2.mvm)(hm, x); ry = (RH.mvm_t if trans else RH.mvm)(rh, x)
        errs.append(np.linalg.norm(y - ry) / np.linalg.norm(ry))
    print("mvm%s rel err max %.3e" % ("_t" if trans else "", max(errs)))
print("launches", _native.launch_count())
