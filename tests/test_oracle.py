"""The CPU oracle (oracle/port.py) against fixtures generated from the
reference itself (tests/golden/make_golden.py).  Bitwise where the oracle
restates the reference's operation order; this pins the checker that the
GPU parity tests rely on."""

import numpy as np
import pytest

from conftest import PIPELINES, eps_of, golden, mesh_for
from oracle import port as P
from paper_1810_08429_b200.geometry import build_sphere_mesh

# frozen coplanar pair-integral values of the reference's test suite
# (pkg/tests/test_quadrature.py:11-19), q = 8, 5e-6 relative
T1 = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
PAIR_ORACLES = {
    3: (T1, 7.98214469042526e-02),
    2: (np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.4, -0.8, 0.0]]), 2.8659934531e-02),
    1: (np.array([[0.0, 0.0, 0.0], [-1.0, -0.2, 0.0], [-0.5, -1.0, 0.0]]), 1.6892968088e-02),
    0: (T1 + np.array([2.0, 0.5, 0.0]), 9.6850829651e-03),
}


def _affine_pair(case, q, t1, t2):
    x, y, w = P.sauter(case, q) if case else _disjoint(q)
    X = t1[0] + np.outer(x[:, 0], t1[1] - t1[0]) + np.outer(x[:, 1], t1[2] - t1[0])
    Y = t2[0] + np.outer(y[:, 0], t2[1] - t2[0]) + np.outer(y[:, 1], t2[2] - t2[0])
    r = np.linalg.norm(X - Y, axis=1)
    area = lambda t: 0.5 * np.linalg.norm(np.cross(t[1] - t[0], t[2] - t[0]))
    return 4.0 * area(t1) * area(t2) * float(w @ (1.0 / (P.FOUR_PI * r)))


def _disjoint(q):
    p, w = P.triangle_rule(q)
    n = len(p)
    return np.repeat(p, n, axis=0), np.tile(p, (n, 1)), np.outer(w, w).ravel()


@pytest.mark.parametrize("case", [0, 1, 2, 3])
def test_frozen_pair_oracles(case):
    t2, target = PAIR_ORACLES[case]
    assert abs(_affine_pair(case, 8, T1, t2) - target) / target < 5e-6


@pytest.mark.parametrize("case,sub", [(3, 6), (2, 10), (1, 2)])
def test_sauter_sizes_and_weights(case, sub):
    for q in (2, 3, 5):
        x, y, w = P.sauter(case, q)
        assert len(w) == sub * q ** 4 and x.shape == y.shape == (len(w), 2)
        assert abs(w.sum() - 0.25) < 1e-13


@pytest.mark.parametrize("name", ["pairs_sphere3.npz", "pairs_cube3.npz"])
def test_pair_values_bitwise(name):
    g = golden(name)
    mesh = mesh_for(name.replace("pairs_", "x_"))
    nodes, gram = P.chart_nodes(mesh.vertices, mesh.triangles)
    case, px, py = P.classify(mesh.triangles[g["rows"]], mesh.triangles[g["cols"]])
    assert np.array_equal(case, g["case"]) and np.array_equal(px, g["px"])
    assert np.array_equal(py, g["py"])
    for k in range(4):
        m = case == k
        got = P.pair_values(nodes, gram, k, g["rows"][m], g["cols"][m], px[m], py[m])
        assert np.array_equal(got, g["values"][m]), "case %d" % k


def test_dense_sphere2_bitwise():
    mesh = build_sphere_mesh(2)
    nodes, gram = P.chart_nodes(mesh.vertices, mesh.triangles)
    idx = np.arange(mesh.nt)
    assert np.array_equal(P.block(nodes, gram, mesh.triangles, idx, idx),
                          golden("dense_sphere2.npz")["values"])


def test_green_factors_and_aca_bitwise():
    g = golden("factors_sphere4.npz")
    mesh = build_sphere_mesh(4)
    nodes, gram = P.chart_nodes(mesh.vertices, mesh.triangles)
    t = P.Tree(mesh.vertices, mesh.triangles, 16)
    ro = ao = po = 0
    for i, node in enumerate(g["node"]):
        R = int(g["nrows"][i])
        rows = g["rows"][ro:ro + R]
        a = P.green_factor(nodes, gram, rows, t.lower[node], t.upper[node], t.diam[node],
                           "col" if g["side"][i] else "row")
        assert np.array_equal(a.ravel(), g["A"][ao:ao + a.size])
        piv, v = P.aca(a, 1e-6)
        r = int(g["npiv"][i])
        assert np.array_equal(piv, g["piv"][po:po + r])
        assert np.array_equal(v.ravel(), g["V"][ao // 108 * 0 + _voff(g, i):_voff(g, i) + R * r])
        ro += R
        ao += a.size
        po += r


def _voff(g, i):
    return int(sum(int(g["nrows"][j]) * int(g["npiv"][j]) for j in range(i)))


def test_aca_kats_bitwise():
    g = golden("aca_kats.npz")
    ao = po = vo = 0
    for (n, w), e, r in zip(g["shape"], g["eps"], g["npiv"]):
        a = g["A"][ao:ao + n * w].reshape(n, w)
        piv, v = P.aca(a, e)
        assert np.array_equal(piv, g["piv"][po:po + r])
        assert np.array_equal(v.ravel(), g["V"][vo:vo + n * r])
        ao, po, vo = ao + n * w, po + r, vo + n * r


@pytest.mark.parametrize("name", PIPELINES)
def test_trees_and_block_leaves(name):
    g = golden(name)
    mesh = mesh_for(name)
    t = P.Tree(mesh.vertices, mesh.triangles, 16)
    assert np.array_equal(t.perm, g["perm"])
    assert np.array_equal(np.array(t.start), g["start"]) and np.array_equal(np.array(t.stop), g["stop"])
    assert np.array_equal(t.lower, g["lower"]) and np.array_equal(t.upper, g["upper"])
    lv = np.array(P.block_leaves(t), dtype=np.int64)
    assert np.array_equal(lv[:, 0], g["leaf_row"]) and np.array_equal(lv[:, 1], g["leaf_col"])
    assert np.array_equal(lv[:, 2].astype(bool), g["leaf_adm"])


def test_oracle_bases_and_blocks_sphere4():
    name = "h2_sphere4_eps1e-4.npz"
    g = golden(name)
    mesh = mesh_for(name)
    h = P.H2(mesh.vertices, mesh.triangles, eps_of(name), assemble=False)
    for side in ("row", "col"):
        order = [int(i) for i in g[side + "_node"]]
        assert sorted(order) == sorted(k for k in h.bases[side] if k != "_roots")
        piv = np.concatenate([h.bases[side][i]["piv"] for i in order])
        assert np.array_equal(piv, g[side + "_piv"])
    # sampled block values, bitwise
    adm = [(i, j) for i, j, a in h.leaves if a]
    near = [(i, j) for i, j, a in h.leaves if not a]
    for key, blocks in (("coup", adm), ("near", near)):
        off = 0
        for bi, shp in zip(g[key + "_pick"][:8], g[key + "_shape"][:8]):
            i, j = blocks[bi]
            r = h.bases["row"][i]["piv"] if key == "coup" else h.t.dofs(i)
            c = h.bases["col"][j]["piv"] if key == "coup" else h.t.dofs(j)
            vals = P.block(h.nodes, h.gram, h.tris, r, c)
            assert np.array_equal(vals.ravel(), g[key + "_vals"][off:off + vals.size])
            off += int(np.prod(shp))


# ---------------------------------------------------------------- double layer

@pytest.mark.parametrize("name,mesh_name", [("pairs_dlp_sphere3.npz", "x_sphere3"),
                                            ("pairs_dlp_cube3.npz", "x_cube3")])
def test_dlp_pair_values_bitwise(name, mesh_name):
    """Double-layer pair integrals (assembly.py:194-201): the oracle equals
    the reference bit for bit in every case."""
    g = golden(name)
    mesh = mesh_for(mesh_name)
    nodes, gram = P.chart_nodes(mesh.vertices, mesh.triangles)
    normals = P.chart_normals(mesh.vertices, mesh.triangles)
    case, px, py = P.classify(mesh.triangles[g["rows"]], mesh.triangles[g["cols"]])
    assert np.array_equal(case, g["case"])
    for k in range(4):
        m = case == k
        got = P.pair_values(nodes, gram, k, g["rows"][m], g["cols"][m], px[m], py[m],
                            kind="dlp", normals=normals)
        assert np.array_equal(got, g["values"][m]), "case %d" % k


def test_dlp_dense_sphere2_bitwise():
    mesh = build_sphere_mesh(2)
    nodes, gram = P.chart_nodes(mesh.vertices, mesh.triangles)
    normals = P.chart_normals(mesh.vertices, mesh.triangles)
    idx = np.arange(mesh.nt)
    got = P.block(nodes, gram, mesh.triangles, idx, idx, kind="dlp", normals=normals)
    assert np.array_equal(got, golden("dense_dlp_sphere2.npz")["values"])


# ---------------------------------------------------------------- linear basis

@pytest.mark.parametrize("kind", ["slp", "dlp"])
def test_linear_pair_values_bitwise(kind):
    """Linear-basis 3x3 pair integrals (assembly.py:122-135, 175-214)."""
    g = golden("pairs_lin_%s_sphere3.npz" % kind)
    mesh = mesh_for("x_sphere3")
    nodes, gram = P.chart_nodes(mesh.vertices, mesh.triangles)
    normals = P.chart_normals(mesh.vertices, mesh.triangles)
    for k in range(4):
        m = g["case"] == k
        got = P.pair_values_linear(nodes, gram, k, g["rows"][m], g["cols"][m], g["px"][m], g["py"][m],
                                   kind=kind, normals=normals)
        assert np.array_equal(got, g["values"][m]), "case %d" % k


def test_linear_dense_blocks_and_table_bitwise():
    g = golden("dense_lin_sphere2.npz")
    mesh = build_sphere_mesh(2)
    nodes, gram = P.chart_nodes(mesh.vertices, mesh.triangles)
    normals = P.chart_normals(mesh.vertices, mesh.triangles)
    dofs = np.arange(mesh.nv)
    assert np.array_equal(P.triangle_table(g["table_rows"], mesh.triangles, mesh.nv), g["table"])
    assert np.array_equal(P.block_linear(nodes, gram, mesh.triangles, dofs, dofs), g["slp"])
    assert np.array_equal(P.block_linear(nodes, gram, mesh.triangles, dofs, dofs, kind="dlp",
                                         normals=normals), g["dlp"])
    assert np.array_equal(P.block_linear(nodes, gram, mesh.triangles, g["sub_rows"], g["sub_cols"]),
                          g["sub"])


def test_linear_triangle_table_host_matches_oracle():
    from paper_1810_08429_b200 import linear
    mesh = build_sphere_mesh(3)
    rng = np.random.default_rng(8)
    for n in (1, 7, 40, mesh.nv):
        idx = rng.choice(mesh.nv, n, replace=False)
        assert np.array_equal(linear.triangle_table(idx, mesh),
                              P.triangle_table(idx, mesh.triangles, mesh.nv))


# ---------------------------------------------------------------- collocation

def test_collocation_values_and_blocks_bitwise():
    g = golden("colloc_pairs_sphere3.npz")
    mesh = mesh_for("x_sphere3")
    nodes, gram = P.chart_nodes(mesh.vertices, mesh.triangles)
    normals = P.chart_normals(mesh.vertices, mesh.triangles)
    case, py = P.collocation_classify(mesh.triangles, g["rows"], g["cols"])
    assert np.array_equal(case, g["case"]) and np.array_equal(py, g["py"])
    for kind in ("slp", "dlp"):
        for k in (0, 1):
            m = case == k
            got = P.collocation_values(nodes, gram, mesh.vertices, k, g["rows"][m], g["cols"][m], py[m],
                                       kind=kind, normals=normals)
            assert np.array_equal(got, g[kind][m]), (kind, k)
    d = golden("colloc_dense_sphere2.npz")
    s2 = build_sphere_mesh(2)
    n2, g2 = P.chart_nodes(s2.vertices, s2.triangles)
    nn2 = P.chart_normals(s2.vertices, s2.triangles)
    dofs = np.arange(s2.nv)
    assert np.array_equal(P.block_collocation(n2, g2, s2.vertices, s2.triangles, dofs, dofs), d["slp"])
    assert np.array_equal(P.block_collocation(n2, g2, s2.vertices, s2.triangles, dofs, dofs, kind="dlp",
                                              normals=nn2), d["dlp"])


# ---------------------------------------------------------------- curved charts

def _curved3():
    from paper_1810_08429_b200.geometry import to_curved
    return to_curved(build_sphere_mesh(3), project_to_unit_sphere=True)


def test_curved_pair_values_bitwise():
    """Curved (quadratic) charts: pair integrals with point Gramians from the
    interpolated node normals (assembly.py:189-205), all four cases, both
    kernels and bases."""
    g = golden("curved_pairs_sphere3.npz")
    m = _curved3()
    nodes, normals = P.chart_curved(m.vertices, m.triangles, m.midpoints, m.tri_edges)
    for kind in ("slp", "dlp"):
        for k in range(4):
            sel = g["case"] == k
            args = (nodes, None, k, g["rows"][sel], g["cols"][sel], g["px"][sel], g["py"][sel])
            got = P.pair_values(*args, kind=kind, normals=normals)
            assert np.array_equal(got, g["%s_constant" % kind][sel][:, 0, 0]), (kind, k)
            got = P.pair_values_linear(*args, kind=kind, normals=normals)
            assert np.array_equal(got, g["%s_linear" % kind][sel]), (kind, k)


def test_curved_chart_pack_and_trees_bitwise():
    """Host curved geometry (to_curved, chart_pack, control points) and the
    cluster trees built on it, constant and linear, vs the reference."""
    from paper_1810_08429_b200 import clustering, geometry
    m = _curved3()
    pack = geometry.chart_pack(m)
    nodes, normals = P.chart_curved(m.vertices, m.triangles, m.midpoints, m.tri_edges)
    assert np.array_equal(pack.nodes, nodes) and np.array_equal(pack.normals, normals)
    g = golden("curved_h2_constant_sphere3.npz")
    t = clustering.build_cluster_tree(m, "constant", 16)
    assert np.array_equal(t.perm, g["perm"])
    assert np.array_equal(t.flat.lower, g["lower"]) and np.array_equal(t.flat.upper, g["upper"])
    m4 = geometry.to_curved(build_sphere_mesh(4), project_to_unit_sphere=True)
    g = golden("curved_h2_linear_sphere4.npz")
    t = clustering.build_cluster_tree(m4, "linear", 16)
    assert np.array_equal(t.perm, g["perm"])
    assert np.array_equal(t.flat.lower, g["lower"]) and np.array_equal(t.flat.upper, g["upper"])
