"""Generate the golden fixtures from the reference implementation itself.

Run in the build container (the reference is importable there):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--dlp | --linear | --mvm20 ...]
(each flag writes only that family of fixtures; none = the base set)
Outputs tests/golden/*.npz.  The GPU box has no /root/reference; the tests
read only these committed files.
"""

import os
import sys

import numpy as np

_REF = "/root/reference/pkg/src"
if not os.path.isdir(_REF):   # on the GPU host: the stock install the reference arm uses
    _REF = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "baseline", "_ref")
sys.path.insert(0, _REF)
from greencross import assembly as A  # noqa: E402
from greencross import clustering as C  # noqa: E402
from greencross import gca as GC  # noqa: E402
from greencross import geometry as G  # noqa: E402
from greencross import h2 as H  # noqa: E402
from greencross import quadrature as Q  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def cube(level):
    s = G.build_sphere_mesh(level)
    v = s.vertices
    return G.TriangleMesh(v / np.abs(v).max(axis=1, keepdims=True), s.triangles)


def pair_tasks(mesh, n_disjoint, seed, kind="slp"):
    """Random disjoint tasks plus every singular pair of a triangle subset."""
    rng = np.random.default_rng(seed)
    rows = list(rng.integers(0, mesh.nt, n_disjoint))
    cols = list(rng.integers(0, mesh.nt, n_disjoint))
    stars = mesh.vertex_stars()
    for t in rng.choice(mesh.nt, 24, replace=False):
        for v in mesh.triangles[t]:
            for s in stars[v]:
                rows.append(int(t))
                cols.append(int(s))
    rows, cols = np.array(rows), np.array(cols)
    case, px, py = Q.classify_pairs(mesh.triangles[rows], mesh.triangles[cols])
    ev = A.galerkin_pair_evaluator(kind, mesh, "constant", 3, 5)
    vals = np.empty(len(rows))
    for k in range(4):
        m = case == k
        if m.any():
            vals[m] = ev(k, rows[m], cols[m], px[m], py[m]).ravel()
    return dict(rows=rows, cols=cols, case=case, px=px, py=py, values=vals)


def pipeline(mesh, eps, seed, nsample=40):
    tree = C.build_cluster_tree(mesh, "constant", 16)
    bt = C.build_block_tree(tree, eta=1.0)
    rm, cm = GC.coupling_marks(bt)
    rb = GC.build_cluster_basis(tree, mesh, "constant", 3, 0.5, eps, "row", (3, 5), rm)
    cb = GC.build_cluster_basis(tree, mesh, "constant", 3, 0.5, eps, "col", (3, 5), cm)
    hm = GC.build_h2(bt, rb, cb, mesh, "slp", "constant", "galerkin", (3, 5))
    nodes = tree.nodes()
    leaves = bt.leaves()
    out = dict(perm=tree.perm.astype(np.int32),
               start=np.array([n.start for n in nodes], np.int32),
               stop=np.array([n.stop for n in nodes], np.int32),
               lower=np.array([n.box.lower for n in nodes]),
               upper=np.array([n.box.upper for n in nodes]),
               leaf_row=np.array([l.row.index for l in leaves], np.int32),
               leaf_col=np.array([l.col.index for l in leaves], np.int32),
               leaf_adm=np.array([l.state == "admissible" for l in leaves]))
    for side, basis in (("row", rb), ("col", cb)):
        bns = basis.nodes()
        out[side + "_node"] = np.array([b.cluster.index for b in bns], np.int32)
        out[side + "_rank"] = np.array([b.rank for b in bns], np.int32)
        out[side + "_piv"] = np.concatenate([b.pivots for b in bns]).astype(np.int32)
        # transfers / leaf bases of a few nodes for value checks
        rng = np.random.default_rng(seed + (side == "col"))
        pick = rng.choice(len(bns), min(12, len(bns)), replace=False)
        vals, meta = [], []
        for i in pick:
            b = bns[i]
            m = b.v if b.v is not None else b.transfer
            kind = 0 if b.v is not None else 1
            if m is None:
                continue
            meta.append((b.cluster.index, kind, m.shape[0], m.shape[1]))
            vals.append(m.ravel())
        out[side + "_mat_meta"] = np.array(meta, np.int64).reshape(-1, 4)
        out[side + "_mat_vals"] = np.concatenate(vals) if vals else np.zeros(0)
    rng = np.random.default_rng(seed)
    for name, blocks in (("coup", hm.coupling), ("near", hm.nearfield)):
        pick = np.sort(rng.choice(len(blocks), min(nsample, len(blocks)), replace=False))
        out[name + "_pick"] = pick.astype(np.int32)
        out[name + "_shape"] = np.array([blocks[i].values.shape for i in pick], np.int32)
        out[name + "_vals"] = np.concatenate([blocks[i].values.ravel() for i in pick])
    xs = np.random.default_rng(seed + 7).standard_normal((2, mesh.nt))
    out["x"] = xs
    out["mvm"] = np.stack([H.mvm(hm, x) for x in xs])
    out["mvm_t"] = np.stack([H.mvm_t(hm, x) for x in xs])
    rep = H.storage_report(hm)
    out["storage_keys"] = np.array(list(rep.keys()))
    out["storage_vals"] = np.array(list(rep.values()), np.int64)
    out["exec_tasks"] = np.array([s["tasks"] for s in hm.exec_stats], np.int64)
    return out


def factors(mesh, seed):
    """Green factors (row and column side) of leaves and of internal nodes
    on the reference's own row lists, plus ACA results on them."""
    tree = C.build_cluster_tree(mesh, "constant", 16)
    nodes = tree.nodes()
    rng = np.random.default_rng(seed)
    leaves = [n for n in nodes if n.is_leaf()]
    inner = [n for n in nodes if not n.is_leaf() and n.size <= 64]
    chosen = list(rng.choice(len(leaves), 4, replace=False))
    out = {"node": [], "side": [], "rows": [], "nrows": [], "A": [], "piv": [], "npiv": [], "V": []}
    for node in [leaves[i] for i in chosen] + inner[:3]:
        rows = np.asarray(node.indices)
        for side in ("row", "col"):
            rule = Q.green_box_rule(node.box, 0.5 * node.box.diameter(), 3)
            stub = GC._Rows(rows, node.box)
            a = (A.green_row_factor(stub, rule, mesh, "constant") if side == "row" else
                 A.green_col_factor((stub, stub), rule, mesh, "constant"))
            it = GC.aca_interpolation(a, 1e-6)
            out["node"].append(node.index)
            out["side"].append(side == "col")
            out["rows"].append(rows)
            out["nrows"].append(len(rows))
            out["A"].append(a.ravel())
            out["piv"].append(it.pivots)
            out["npiv"].append(len(it.pivots))
            out["V"].append(it.v.ravel())
    return {k: (np.concatenate(v) if k in ("rows", "A", "piv", "V") else np.array(v))
            for k, v in out.items()}


def aca_kats():
    rng = np.random.default_rng(2024)
    mats, shapes, eps, pivs, npiv, vs = [], [], [], [], [], []
    q1, _ = np.linalg.qr(rng.standard_normal((60, 20)))
    q2, _ = np.linalg.qr(rng.standard_normal((20, 20)))
    cases = [(np.eye(8), 1e-12), (np.outer(np.arange(1.0, 7.0), [2.0, -1.0, 0.5]), 1e-12),
             (rng.standard_normal((200, 24)), 1e-6), (np.zeros((10, 4)), 1e-8),
             (q1 @ np.diag(10.0 ** -np.arange(20.0)) @ q2.T, 1e-3),
             (rng.standard_normal((37, 108)), 1e-4)]
    for a, e in cases:
        it = GC.aca_interpolation(a, e)
        mats.append(a.ravel())
        shapes.append(a.shape)
        eps.append(e)
        pivs.append(it.pivots)
        npiv.append(len(it.pivots))
        vs.append(it.v.ravel())
    return dict(A=np.concatenate(mats), shape=np.array(shapes), eps=np.array(eps),
                piv=np.concatenate(pivs), npiv=np.array(npiv), V=np.concatenate(vs))


def dlp_pipeline(mesh, eps, seed):
    """The reference's GCA-H2 of the double-layer operator (same nested
    bases, dlp coupling and near-field blocks): matvecs and sampled blocks."""
    tree = C.build_cluster_tree(mesh, "constant", 16)
    bt = C.build_block_tree(tree, eta=1.0)
    rm, cm = GC.coupling_marks(bt)
    rb = GC.build_cluster_basis(tree, mesh, "constant", 3, 0.5, eps, "row", (3, 5), rm)
    cb = GC.build_cluster_basis(tree, mesh, "constant", 3, 0.5, eps, "col", (3, 5), cm)
    hm = GC.build_h2(bt, rb, cb, mesh, "dlp", "constant", "galerkin", (3, 5))
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((3, mesh.nt))
    y = np.array([H.mvm(hm, v) for v in x])
    pick = rng.choice(len(hm.nearfield), 8, replace=False)
    near_r = np.array([hm.nearfield[i].row.index for i in pick], np.int32)
    near_c = np.array([hm.nearfield[i].col.index for i in pick], np.int32)
    near_v = np.concatenate([hm.nearfield[i].values.ravel() for i in pick])
    return dict(x=x, mvm=y, near_row=near_r, near_col=near_c, near_values=near_v)


def lin_pair_tasks(mesh, n_disjoint, seed, kind):
    """Linear-basis pair integrals (B, 3, 3) from the reference's evaluator."""
    g = pair_tasks(mesh, n_disjoint, seed)
    ev = A.galerkin_pair_evaluator(kind, mesh, "linear", 3, 5)
    vals = np.empty((len(g["rows"]), 3, 3))
    for k in range(4):
        m = g["case"] == k
        if m.any():
            vals[m] = ev(k, g["rows"][m], g["cols"][m], g["px"][m], g["py"][m])
    g["values"] = vals
    return g


def lin_pipeline(mesh, eps, seed):
    """The reference's GCA-H2 with the linear basis: vertex tree, bases
    (pivot vertices), sampled blocks and matvecs."""
    tree = C.build_cluster_tree(mesh, "linear", 16)
    bt = C.build_block_tree(tree, eta=1.0)
    rm, cm = GC.coupling_marks(bt)
    rb = GC.build_cluster_basis(tree, mesh, "linear", 3, 0.5, eps, "row", (3, 5), rm)
    cb = GC.build_cluster_basis(tree, mesh, "linear", 3, 0.5, eps, "col", (3, 5), cm)
    hm = GC.build_h2(bt, rb, cb, mesh, "slp", "linear", "galerkin", (3, 5))
    nodes = tree.nodes()
    leaves = bt.leaves()
    out = dict(perm=tree.perm.astype(np.int32),
               start=np.array([n.start for n in nodes], np.int32),
               stop=np.array([n.stop for n in nodes], np.int32),
               lower=np.array([n.box.lower for n in nodes]),
               upper=np.array([n.box.upper for n in nodes]),
               leaf_row=np.array([l.row.index for l in leaves], np.int32),
               leaf_col=np.array([l.col.index for l in leaves], np.int32),
               leaf_adm=np.array([l.state == "admissible" for l in leaves]))
    for side, basis in (("row", rb), ("col", cb)):
        bns = basis.nodes()
        out[side + "_node"] = np.array([b.cluster.index for b in bns], np.int32)
        out[side + "_rank"] = np.array([b.rank for b in bns], np.int32)
        out[side + "_piv"] = np.concatenate([b.pivots for b in bns]).astype(np.int32)
    # Green factors of a few leaves (row side) for the linear basis
    rng = np.random.default_rng(seed)
    fl = [n for n in nodes if n.is_leaf()]
    pick = rng.choice(len(fl), 4, replace=False)
    facs = []
    for i in pick:
        node = fl[i]
        rule = Q.green_box_rule(node.box, 0.5 * node.box.diameter(), 3)
        facs.append(A.green_row_factor(node, rule, mesh, "linear", (3, 5)).ravel())
    out["factor_nodes"] = np.array([fl[i].index for i in pick], np.int32)
    out["factors"] = np.concatenate(facs)
    x = rng.standard_normal((3, mesh.nv))
    out["x"] = x
    out["mvm"] = np.array([H.mvm(hm, v) for v in x])
    out["storage_keys"] = np.array(list(H.storage_report(hm).keys()))
    out["storage_vals"] = np.array(list(H.storage_report(hm).values()))
    return out


def main_linear_h2():
    np.savez_compressed(os.path.join(OUT, "h2_lin_sphere3_eps1e-4.npz"),
                        **lin_pipeline(G.build_sphere_mesh(3), 1e-4, 43))
    np.savez_compressed(os.path.join(OUT, "h2_lin_cube3_eps1e-6.npz"), **lin_pipeline(cube(3), 1e-6, 44))


def main_linear():
    s3 = G.build_sphere_mesh(3)
    for kind in ("slp", "dlp"):
        np.savez_compressed(os.path.join(OUT, "pairs_lin_%s_sphere3.npz" % kind),
                            **lin_pair_tasks(s3, 300, 41, kind))
    s2 = G.build_sphere_mesh(2)
    dofs = np.arange(s2.nv)
    rng = np.random.default_rng(42)
    r = rng.choice(s2.nv, 7, replace=False)
    c = rng.choice(s2.nv, 9, replace=False)
    np.savez_compressed(os.path.join(OUT, "dense_lin_sphere2.npz"),
                        slp=A.assemble_galerkin_block("slp", s2, "linear", dofs, dofs).values,
                        dlp=A.assemble_galerkin_block("dlp", s2, "linear", dofs, dofs).values,
                        sub_rows=r, sub_cols=c,
                        sub=A.assemble_galerkin_block("slp", s2, "linear", r, c).values,
                        table_rows=r, table=A.triangle_table(r, s2).rows)


def main_collocation():
    s3 = G.build_sphere_mesh(3)
    rng = np.random.default_rng(51)
    rows = list(rng.integers(0, s3.nv, 400))
    cols = list(rng.integers(0, s3.nt, 400))
    stars = s3.vertex_stars()
    for v in rng.choice(s3.nv, 20, replace=False):
        for t in stars[v]:
            rows.append(int(v))
            cols.append(int(t))
    rows, cols = np.array(rows), np.array(cols)
    case, px, py = A.collocation_classify(s3)(rows, cols)
    out = dict(rows=rows, cols=cols, case=case, py=py)
    for kind in ("slp", "dlp"):
        ev = A.collocation_evaluator(kind, s3, 3, 5)
        vals = np.empty((len(rows), 1, 3))
        for k in (0, 1):
            m = case == k
            vals[m] = ev(k, rows[m], cols[m], px[m], py[m])
        out[kind] = vals
    np.savez_compressed(os.path.join(OUT, "colloc_pairs_sphere3.npz"), **out)
    s2 = G.build_sphere_mesh(2)
    dofs = np.arange(s2.nv)
    np.savez_compressed(os.path.join(OUT, "colloc_dense_sphere2.npz"),
                        slp=A.assemble_collocation_block("slp", s2, "linear", dofs, dofs).values,
                        dlp=A.assemble_collocation_block("dlp", s2, "linear", dofs, dofs).values)
    # the reference's collocation GCA-H2 (cli.build_h2_operator, disc="collocation")
    import greencross.cli as CL
    mesh = G.build_sphere_mesh(3)
    cfg = CL.ExperimentConfig(level=3, geometry="plane", basis="linear", disc="collocation", eta=1.0,
                              m=3, delta_factor=0.5, eps=1e-4, leaf_size=16, q_reg=3, q_sing=5,
                              lam=0.5, source=(2.0, 0.0, 0.0), seed=0)
    hm, tree, bt = CL.build_h2_operator(mesh, cfg)
    res = dict(perm=tree.perm.astype(np.int32))
    for side, basis in (("row", hm.row_basis), ("col", hm.col_basis)):
        bns = basis.nodes()
        res[side + "_node"] = np.array([b.cluster.index for b in bns], np.int32)
        res[side + "_rank"] = np.array([b.rank for b in bns], np.int32)
        res[side + "_piv"] = np.concatenate([b.pivots for b in bns]).astype(np.int32)
    x = rng.standard_normal((3, mesh.nv))
    res["x"] = x
    res["mvm"] = np.array([H.mvm(hm, v) for v in x])
    np.savez_compressed(os.path.join(OUT, "h2_colloc_sphere3_eps1e-4.npz"), **res)


def curved_pipeline(mesh, basis, eps, seed):
    tree = C.build_cluster_tree(mesh, basis, 16)
    bt = C.build_block_tree(tree, eta=1.0)
    rm, cm = GC.coupling_marks(bt)
    rb = GC.build_cluster_basis(tree, mesh, basis, 3, 0.5, eps, "row", (3, 5), rm)
    cb = GC.build_cluster_basis(tree, mesh, basis, 3, 0.5, eps, "col", (3, 5), cm)
    hm = GC.build_h2(bt, rb, cb, mesh, "slp", basis, "galerkin", (3, 5))
    nodes = tree.nodes()
    out = dict(perm=tree.perm.astype(np.int32),
               lower=np.array([n.box.lower for n in nodes]), upper=np.array([n.box.upper for n in nodes]))
    for side, b in (("row", rb), ("col", cb)):
        bns = b.nodes()
        out[side + "_node"] = np.array([x.cluster.index for x in bns], np.int32)
        out[side + "_rank"] = np.array([x.rank for x in bns], np.int32)
        out[side + "_piv"] = np.concatenate([x.pivots for x in bns]).astype(np.int32)
    rng = np.random.default_rng(seed)
    fl = [n for n in nodes if n.is_leaf()]
    pick = rng.choice(len(fl), 3, replace=False)
    facs = []
    for i in pick:
        node = fl[i]
        rule = Q.green_box_rule(node.box, 0.5 * node.box.diameter(), 3)
        facs.append(A.green_row_factor(node, rule, mesh, basis, (3, 5)).ravel())
    out["factor_nodes"] = np.array([fl[i].index for i in pick], np.int32)
    out["factors"] = np.concatenate(facs)
    n = mesh.nt if basis == "constant" else mesh.nv
    x = rng.standard_normal((2, n))
    out["x"] = x
    out["mvm"] = np.array([H.mvm(hm, v) for v in x])
    return out


def main_curved():
    c3 = G.to_curved(G.build_sphere_mesh(3), project_to_unit_sphere=True)
    c2 = G.to_curved(G.build_sphere_mesh(2), project_to_unit_sphere=True)
    out = {}
    g = pair_tasks(c3, 300, 61)
    out.update({"rows": g["rows"], "cols": g["cols"], "case": g["case"], "px": g["px"], "py": g["py"]})
    for kind in ("slp", "dlp"):
        for basis, w in (("constant", 1), ("linear", 3)):
            ev = A.galerkin_pair_evaluator(kind, c3, basis, 3, 5)
            vals = np.empty((len(g["rows"]), w, w))
            for k in range(4):
                m = g["case"] == k
                vals[m] = ev(k, g["rows"][m], g["cols"][m], g["px"][m], g["py"][m])
            out["%s_%s" % (kind, basis)] = vals
    np.savez_compressed(os.path.join(OUT, "curved_pairs_sphere3.npz"), **out)
    idx, dofs = np.arange(c2.nt), np.arange(c2.nv)
    np.savez_compressed(os.path.join(OUT, "curved_dense_sphere2.npz"),
                        slp_constant=A.assemble_galerkin_block("slp", c2, "constant", idx, idx).values,
                        dlp_linear=A.assemble_galerkin_block("dlp", c2, "linear", dofs, dofs).values,
                        colloc_dlp=A.assemble_collocation_block("dlp", c2, "linear", dofs, dofs).values,
                        mass_linear=A.mass_block(c2, "linear", dofs, dofs).values)
    np.savez_compressed(os.path.join(OUT, "curved_h2_constant_sphere3.npz"),
                        **curved_pipeline(c3, "constant", 1e-4, 62))
    c4 = G.to_curved(G.build_sphere_mesh(4), project_to_unit_sphere=True)
    np.savez_compressed(os.path.join(OUT, "curved_h2_linear_sphere4.npz"),
                        **curved_pipeline(c4, "linear", 1e-4, 63))


def main_dlp():
    s3 = G.build_sphere_mesh(3)
    np.savez_compressed(os.path.join(OUT, "pairs_dlp_sphere3.npz"), **pair_tasks(s3, 600, 31, "dlp"))
    np.savez_compressed(os.path.join(OUT, "pairs_dlp_cube3.npz"), **pair_tasks(cube(3), 300, 32, "dlp"))
    s2 = G.build_sphere_mesh(2)
    idx = np.arange(s2.nt)
    np.savez_compressed(os.path.join(OUT, "dense_dlp_sphere2.npz"),
                        values=A.assemble_galerkin_block("dlp", s2, "constant", idx, idx).values)
    np.savez_compressed(os.path.join(OUT, "h2_dlp_sphere4_eps1e-6.npz"),
                        **dlp_pipeline(G.build_sphere_mesh(4), 1e-6, 33))


def main():
    s3 = G.build_sphere_mesh(3)
    np.savez_compressed(os.path.join(OUT, "pairs_sphere3.npz"), **pair_tasks(s3, 600, 11))
    c3 = cube(3)
    np.savez_compressed(os.path.join(OUT, "pairs_cube3.npz"), **pair_tasks(c3, 300, 12))
    s2 = G.build_sphere_mesh(2)
    idx = np.arange(s2.nt)
    np.savez_compressed(os.path.join(OUT, "dense_sphere2.npz"),
                        values=A.assemble_galerkin_block("slp", s2, "constant", idx, idx).values)
    np.savez_compressed(os.path.join(OUT, "factors_sphere4.npz"), **factors(G.build_sphere_mesh(4), 5))
    np.savez_compressed(os.path.join(OUT, "aca_kats.npz"), **aca_kats())
    np.savez_compressed(os.path.join(OUT, "h2_sphere4_eps1e-4.npz"),
                        **pipeline(G.build_sphere_mesh(4), 1e-4, 21))
    np.savez_compressed(os.path.join(OUT, "h2_cube4_eps1e-6.npz"), **pipeline(cube(4), 1e-6, 22))
    np.savez_compressed(os.path.join(OUT, "h2_sphere5_eps1e-6.npz"),
                        **pipeline(G.build_sphere_mesh(5), 1e-6, 23))


def main_mvm20():
    """SURVEY 8(c) parity protocol on C1 (sphere L4, eps 1e-4, CLI defaults):
    the reference's mvm / mvm_t of 20 seeded N(0,1) vectors
    (np.random.default_rng(0), the reference tests' convention).  x is
    regenerated in the test; only the products are stored."""
    mesh = G.build_sphere_mesh(4)
    tree = C.build_cluster_tree(mesh, "constant", 16)
    bt = C.build_block_tree(tree, eta=1.0)
    rm, cm = GC.coupling_marks(bt)
    rb = GC.build_cluster_basis(tree, mesh, "constant", 3, 0.5, 1e-4, "row", (3, 5), rm)
    cb = GC.build_cluster_basis(tree, mesh, "constant", 3, 0.5, 1e-4, "col", (3, 5), cm)
    hm = GC.build_h2(bt, rb, cb, mesh, "slp", "constant", "galerkin", (3, 5))
    xs = np.random.default_rng(0).standard_normal((20, mesh.nt))
    np.savez_compressed(os.path.join(OUT, "mvm20_sphere4_eps1e-4.npz"),
                        mvm=np.stack([H.mvm(hm, x) for x in xs]),
                        mvm_t=np.stack([H.mvm_t(hm, x) for x in xs]))


def node_hashes(bns):
    """Per basis node: 32-bit digests of the pivot list in order and of the
    sorted pivot set (blake2b of the little-endian int32 bytes).  Stored
    instead of the pivots themselves at the benchmark sizes (C4 holds about
    6 M pivots per side); tests/bench_fixtures.py recomputes them."""
    import hashlib

    def h(a):
        return int.from_bytes(hashlib.blake2b(np.asarray(a, "<i4").tobytes(), digest_size=4).digest(), "little")
    return (np.array([h(b.pivots) for b in bns], np.uint32),
            np.array([h(np.sort(b.pivots)) for b in bns], np.uint32))


def digest(*arrays):
    import hashlib
    d = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        d.update(str(a.dtype.str).encode() + str(a.shape).encode())
        d.update(a.tobytes())
    return d.hexdigest()


BENCH = {   # C2 sphere L6 eps 1e-6, C3 cube L7 eps 1e-6, C4 sphere L8 eps 1e-8
    "c2": (lambda: G.build_sphere_mesh(6), 1e-6),
    "c3": (lambda: cube(7), 1e-6),
    "c4": (lambda: G.build_sphere_mesh(8), 1e-8),
}


def bench_pipeline(name, full_build):
    """Reference structure at a benchmark mesh (north_star: trees, pivot sets
    and block structure bit-exact on the same mesh; entries and matvecs
    within 1e-10).  Trees, block leaves and per-node pivot digests in full;
    V / transfer matrices of sampled nodes; sampled coupling blocks
    assembled at the reference's own pivots and near-field blocks, both by
    the reference's assemble_galerkin_block (bitwise equal to the H2
    blocks, test_assembly.py:220-226 / executor invariance).  With
    ``full_build`` (C2) also the reference's own build_h2 and mvm / mvm_t of
    three np.random.default_rng(0) vectors."""
    import time
    make, eps = BENCH[name]
    t0 = time.time()
    mesh = make()
    tree = C.build_cluster_tree(mesh, "constant", 16)
    t1 = time.time()
    bt = C.build_block_tree(tree, eta=1.0)
    t2 = time.time()
    print("%s: cluster tree %.1f s, block tree %.1f s" % (name, t1 - t0, t2 - t1), flush=True)
    nodes = tree.nodes()
    leaves = bt.leaves()
    perm = tree.perm.astype(np.int32)
    start = np.array([n.start for n in nodes], np.int32)
    stop = np.array([n.stop for n in nodes], np.int32)
    lower = np.array([n.box.lower for n in nodes])
    upper = np.array([n.box.upper for n in nodes])
    lrow = np.array([lf.row.index for lf in leaves], np.int32)
    lcol = np.array([lf.col.index for lf in leaves], np.int32)
    ladm = np.array([lf.state == "admissible" for lf in leaves])
    out = dict(nt=mesh.nt, eps=eps, n_nodes=len(nodes), n_leaves=len(leaves), n_adm=int(ladm.sum()),
               perm_sha=digest(perm), tree_sha=digest(start, stop), box_sha=digest(lower, upper),
               leaves_sha=digest(lrow, lcol, ladm), perm_head=perm[:256])
    rm, cm = GC.coupling_marks(bt)
    bases = {}
    for side, marks in (("row", rm), ("col", cm)):
        t = time.time()
        basis = GC.build_cluster_basis(tree, mesh, "constant", 3, 0.5, eps, side, (3, 5), marks)
        print("%s: %s basis %.1f s" % (name, side, time.time() - t), flush=True)
        bases[side] = basis
        bns = basis.nodes()
        ho, hs = node_hashes(bns)
        out[side + "_node"] = np.array([b.cluster.index for b in bns], np.int32)
        out[side + "_rank"] = np.array([b.rank for b in bns], np.int16)
        out[side + "_hash_order"] = ho
        out[side + "_hash_set"] = hs
        out[side + "_piv_sha"] = digest(np.concatenate([b.pivots for b in bns]).astype(np.int32))
        rng = np.random.default_rng(100 + (side == "col"))
        # a few nodes at every tree height, their pivots and matrices
        pick = rng.choice(len(bns), min(24, len(bns)), replace=False)
        meta, vals, pivs = [], [], []
        for i in pick:
            b = bns[int(i)]
            m = b.v if b.v is not None else b.transfer
            if m is None:
                continue
            meta.append((b.cluster.index, 0 if b.v is not None else 1, m.shape[0], m.shape[1], b.rank))
            vals.append(m.ravel())
            pivs.append(b.pivots.astype(np.int32))
        out[side + "_mat_meta"] = np.array(meta, np.int64).reshape(-1, 5)
        out[side + "_mat_vals"] = np.concatenate(vals)
        out[side + "_mat_piv"] = np.concatenate(pivs)
    # sampled blocks at the reference's own pivots / clusters
    rng = np.random.default_rng(7)
    adm_idx = np.flatnonzero(ladm)
    near_idx = np.flatnonzero(~ladm)
    t = time.time()
    for key, pool, k in (("coup", adm_idx, 24), ("near", near_idx, 24)):
        pick = np.sort(rng.choice(pool, k, replace=False))
        shapes, vals = [], []
        for i in pick:
            lf = leaves[int(i)]
            if key == "coup":
                r = bases["row"].node(lf.row).pivots
                c = bases["col"].node(lf.col).pivots
            else:
                r, c = lf.row.indices, lf.col.indices
            v = A.assemble_galerkin_block("slp", mesh, "constant", r, c).values
            shapes.append(v.shape)
            vals.append(v.ravel())
        out[key + "_leaf"] = pick.astype(np.int64)
        out[key + "_shape"] = np.array(shapes, np.int32)
        out[key + "_vals"] = np.concatenate(vals)
    print("%s: sampled blocks %.1f s" % (name, time.time() - t), flush=True)
    if full_build:
        t = time.time()
        hm = GC.build_h2(bt, bases["row"], bases["col"], mesh, "slp", "constant", "galerkin", (3, 5))
        print("%s: build_h2 %.1f s" % (name, time.time() - t), flush=True)
        xs = np.random.default_rng(0).standard_normal((3, mesh.nt))
        out["mvm"] = np.stack([H.mvm(hm, x) for x in xs])
        out["mvm_t"] = np.stack([H.mvm_t(hm, x) for x in xs])
        rep = H.storage_report(hm)
        out["storage_keys"] = np.array(list(rep.keys()))
        out["storage_vals"] = np.array(list(rep.values()), np.int64)
        out["exec_tasks"] = np.array([s["tasks"] for s in hm.exec_stats], np.int64)
        out["exec_batches"] = np.array([s["batches"] for s in hm.exec_stats], np.int64)
    out["total_s"] = time.time() - t0
    return out


def main_bench(names, full):
    import platform
    for name in names:
        res = bench_pipeline(name, full and name == "c2")
        res["host"] = np.array(platform.processor() or platform.machine())
        np.savez_compressed(os.path.join(OUT, "bench_%s.npz" % name), **res)
        print("%s: done in %.1f s" % (name, res["total_s"]), flush=True)


def main_solvers():
    """C1 (sphere L4, CLI defaults): the reference's cg_solve, cgnr_solve and
    spectral_error_estimate on its own GCA-H2 operators (h2.py:144-253):
    iterates and residual histories, the eps 1e-6 operator as the 'exact'
    one against the eps 1e-4 approximation."""
    mesh = G.build_sphere_mesh(4)
    ops = {}
    for eps in (1e-4, 1e-6):
        tree = C.build_cluster_tree(mesh, "constant", 16)
        bt = C.build_block_tree(tree, eta=1.0)
        rm, cm = GC.coupling_marks(bt)
        rb = GC.build_cluster_basis(tree, mesh, "constant", 3, 0.5, eps, "row", (3, 5), rm)
        cb = GC.build_cluster_basis(tree, mesh, "constant", 3, 0.5, eps, "col", (3, 5), cm)
        ops[eps] = H.as_operator(GC.build_h2(bt, rb, cb, mesh, "slp", "constant", "galerkin", (3, 5)))
    b = np.random.default_rng(5).standard_normal(mesh.nt)
    cg = H.cg_solve(ops[1e-4], b, tol=1e-10, max_iter=300)
    cgnr = H.cgnr_solve(ops[1e-4], b, tol=1e-8, max_iter=300)
    err, rel = H.spectral_error_estimate(ops[1e-6], ops[1e-4], mesh.nt, iters=30, seed=3)
    np.savez_compressed(os.path.join(OUT, "solvers_sphere4.npz"), b=b, cg_x=cg.x, cg_res=cg.residuals,
                        cg_conv=cg.converged, cgnr_x=cgnr.x, cgnr_res=cgnr.residuals, cgnr_conv=cgnr.converged,
                        spec_err=err, spec_rel=rel)


if __name__ == "__main__":
    if "--solvers" in sys.argv:
        main_solvers()
    elif "--bench" in sys.argv:
        # --bench c2 [c3 c4] [--no-build]; --out DIR redirects (used on the
        # GPU host to check that its SIMD dispatch yields the same fixtures)
        if "--out" in sys.argv:
            OUT = sys.argv[sys.argv.index("--out") + 1]
        main_bench([a for a in sys.argv[1:] if a in BENCH], "--no-build" not in sys.argv)
    elif "--mvm20" in sys.argv:
        main_mvm20()
    elif "--dlp" in sys.argv:
        main_dlp()
    elif "--linear" in sys.argv:
        main_linear()
    elif "--linear-h2" in sys.argv:
        main_linear_h2()
    elif "--collocation" in sys.argv:
        main_collocation()
    elif "--curved" in sys.argv:
        main_curved()
    else:
        main()
