"""Host-side mirror (meshes, rule tables, classification, trees, block
trees, configuration, errors) against the reference fixtures: bit-exact."""

import os

import numpy as np
import pytest

from conftest import PIPELINES, golden, mesh_for
from oracle import port as P
from paper_1810_08429_b200 import cli, clustering, geometry, quadrature as Q
from paper_1810_08429_b200.errors import (ConfigError, MeshFormatError, SizeLimitError)


@pytest.mark.parametrize("level", [0, 1, 2, 3, 4])
def test_sphere_mesh_matches_oracle_charts(level):
    m = geometry.build_sphere_mesh(level)
    assert m.nt == 8 * 4 ** level
    nodes, gram = P.chart_nodes(m.vertices, m.triangles)
    pack = geometry.chart_pack(m)
    assert np.array_equal(pack.nodes, nodes) and np.array_equal(pack.gram, gram)
    assert np.allclose(np.linalg.norm(m.vertices, axis=1), 1.0, atol=1e-15)


def test_cube_mesh_is_closed_and_on_the_cube():
    c = geometry.build_cube_mesh(3)
    assert c.nt == 512 and np.allclose(np.abs(c.vertices).max(axis=1), 1.0)
    assert len(c.edges) == 3 * c.nt // 2


def test_level_cap_lifted_to_9():
    assert geometry.LEVEL_CAP == 9
    with pytest.raises(SizeLimitError):
        geometry.build_sphere_mesh(10)


def test_mesh_roundtrip(tmp_path):
    m = geometry.build_cube_mesh(2)
    path = os.path.join(tmp_path, "m.txt")
    geometry.write_mesh(m, path)
    r = geometry.read_mesh(path)
    assert np.array_equal(r.vertices, m.vertices) and np.array_equal(r.triangles, m.triangles)
    with open(path, "a") as fh:
        fh.write("1 2\n")
    with pytest.raises(MeshFormatError):
        geometry.read_mesh(path)


def test_mesh_validation():
    v = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]])
    with pytest.raises(MeshFormatError):
        geometry.TriangleMesh(v, np.array([[0, 1, 2]]))          # open surface
    with pytest.raises(MeshFormatError):
        geometry.TriangleMesh(v, np.array([[0, 1, 5]]))          # bad index


@pytest.mark.parametrize("case", [1, 2, 3])
@pytest.mark.parametrize("q", [2, 3, 5])
def test_sauter_tables_bitwise(case, q):
    a = Q.sauter_rule(case, q)
    x, y, w = P.sauter(case, q)
    assert np.array_equal(a.x, x) and np.array_equal(a.y, y) and np.array_equal(a.w, w)


def test_triangle_gauss_and_box_rule():
    for q in (1, 2, 4, 7):
        p, w = Q.triangle_gauss(q)
        op, ow = P.triangle_rule(q)
        assert np.array_equal(p, op) and np.array_equal(w, ow)
        assert abs(w.sum() - 0.5) < 1e-14
    rng = np.random.default_rng(0)
    for _ in range(5):
        lo = rng.standard_normal(3)
        hi = lo + rng.random(3)
        a = Q.green_box_rule((lo, hi), 0.3, 3)
        z, wz, nz = P.box_rule(lo, hi, 0.3, 3)
        assert np.array_equal(a.points, z) and np.array_equal(a.weights, wz)
        assert np.array_equal(a.normals, nz)
    r = Q.green_box_rule((np.zeros(3), np.ones(3)), 0.5, 2)
    assert abs(r.weights.sum() - 24.0) < 1e-12 and r.k == 24


def test_classification_matches_oracle():
    rng = np.random.default_rng(3)
    pool = np.array([(0, 1, 2), (2, 1, 5), (3, 4, 2), (3, 4, 5), (1, 2, 6), (0, 5, 6),
                     (7, 8, 9), (2, 0, 1), (1, 0, 3), (0, 3, 2)])
    r = pool[rng.integers(0, len(pool), 3000)]
    c = pool[rng.integers(0, len(pool), 3000)]
    for a, b in zip(Q.classify_pairs(r, c), P.classify(r, c)):
        assert np.array_equal(a, b)
    distinct = [t for t in pool if tuple(t) != (2, 0, 1)]     # one ordering per vertex set
    for t in distinct:
        for s in distinct:
            case = Q.classify_pair(t, s)
            k = {"identical": 3, "edge": 2, "vertex": 1, "disjoint": 0}[case.kind]
            tp, sp = np.asarray(t)[list(case.row_perm)], np.asarray(s)[list(case.col_perm)]
            assert np.array_equal(tp[:k], sp[:k])


@pytest.mark.parametrize("name", PIPELINES)
def test_cluster_and_block_tree_bitwise(name):
    g = golden(name)
    mesh = mesh_for(name)
    tree = clustering.build_cluster_tree(mesh, "constant", leaf_size=16)
    f = tree.flat
    assert np.array_equal(tree.perm, g["perm"])
    assert np.array_equal(f.start, g["start"]) and np.array_equal(f.stop, g["stop"])
    assert np.array_equal(f.lower, g["lower"]) and np.array_equal(f.upper, g["upper"])
    assert [n.index for n in tree.nodes()] == list(range(len(f)))
    bt = clustering.build_block_tree(tree, eta=1.0)
    lr, lc = bt.flat.leaves()
    st = bt.flat.state[bt.flat.leaf_ids]
    assert np.array_equal(lr, g["leaf_row"]) and np.array_equal(lc, g["leaf_col"])
    assert np.array_equal(st == 0, g["leaf_adm"])
    lv = bt.leaves()
    assert len(lv) == len(lr) and lv[5].row.index == lr[5]
    s = bt.stats()
    assert s["admissible"] == int(g["leaf_adm"].sum()) and s["leaves"] == len(lr)


@pytest.mark.parametrize("level,basis,eta", [(3, "constant", 1.0), (4, "linear", 0.7), (4, "constant", 2.5)])
def test_native_block_tree_equals_array_builder(level, basis, eta):
    """gc_block_tree (the library's host routine) builds exactly the nodes,
    order, keys and parents of the numpy array-at-a-time builder."""
    mesh = geometry.build_sphere_mesh(level)
    tree = clustering.build_cluster_tree(mesh, basis, 16)
    a = clustering.build_block_tree(tree, eta=eta).flat
    b = clustering._build_block_tree_arrays(tree, eta=eta).flat
    for k in ("row", "col", "state", "level", "key", "parent_of", "leaf_ids"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


@pytest.mark.parametrize("n,leaf", [(2048, 16), (8194, 16), (1000, 7), (5, 16), (131072, 16)])
def test_tree_topology_matches_the_host_builder(n, leaf):
    """The device cluster tree lays out every depth from the dof count and
    leaf size alone (clustering._tree_topology); the shape must equal the
    host builder's on any point set of that size."""
    rng = np.random.default_rng(n)
    pts = rng.standard_normal((n, 3))

    class _Pts:                       # minimal support data: points as zero-size boxes
        pass
    start, stop, left, right, parent, depth, depths = clustering._tree_topology(n, leaf)
    orig = clustering._support_data
    clustering._support_data = lambda mesh, kind: (pts, pts, pts)
    try:
        flat = clustering.build_cluster_tree(_Pts(), "constant", leaf).flat
    finally:
        clustering._support_data = orig
    for k, v in (("start", start), ("stop", stop), ("left", left), ("right", right), ("parent", parent),
                 ("depth", depth)):
        assert np.array_equal(getattr(flat, k), v), k
    front = np.concatenate([ids for ids, _ in depths])
    assert np.array_equal(np.sort(front), np.arange(len(start)))      # every node in one frontier
    for ids, split in depths:
        assert np.all(np.diff(start[ids]) > 0)                          # start order
        assert np.array_equal(split, (stop[ids] - start[ids]) > leaf)


def test_block_tree_tiles_the_matrix(sphere3):
    tree = clustering.build_cluster_tree(sphere3, "constant", 16)
    bt = clustering.build_block_tree(tree, eta=1.0)
    cover = np.zeros((sphere3.nt, sphere3.nt), dtype=np.int64)
    for b in bt.leaves():
        cover[b.row.start:b.row.stop, b.col.start:b.col.stop] += 1
        if b.state == clustering.ADMISSIBLE:
            assert clustering.admissible(b.row.box, b.col.box, 1.0)
    assert np.all(cover == 1)


def test_tree_validation(sphere2):
    with pytest.raises(ConfigError):
        clustering.build_cluster_tree(sphere2, "quadratic", 16)
    with pytest.raises(ConfigError):
        clustering.build_cluster_tree(sphere2, "constant", 0)
    t = clustering.build_cluster_tree(sphere2, "constant", 16)
    with pytest.raises(ConfigError):
        clustering.build_block_tree(t, eta=0.0)


def test_config_validation():
    cfg = cli.default_config()
    assert (cfg.eta, cfg.m, cfg.leaf_size, cfg.q_reg, cfg.q_sing) == (1.0, 3, 16, 3, 5)
    for bad in (dict(eps=0.0), dict(m=0), dict(eta=-1.0), dict(q_reg=0), dict(lam=1.5),
                dict(disc="collocation")):
        with pytest.raises(ConfigError):
            cli.default_config(**bad)


@pytest.mark.parametrize("name,mesh_name", [("h2_lin_sphere3_eps1e-4.npz", "x_sphere3"),
                                            ("h2_lin_cube3_eps1e-6.npz", "x_cube3")])
def test_linear_vertex_tree_and_block_tree_bitwise(name, mesh_name):
    """The linear basis clusters vertices (support boxes from the vertex
    stars, clustering.py:107-128): tree and block leaves bit-exact."""
    g = golden(name)
    mesh = mesh_for(mesh_name)
    tree = clustering.build_cluster_tree(mesh, "linear", leaf_size=16)
    f = tree.flat
    assert np.array_equal(tree.perm, g["perm"])
    assert np.array_equal(f.start, g["start"]) and np.array_equal(f.stop, g["stop"])
    assert np.array_equal(f.lower, g["lower"]) and np.array_equal(f.upper, g["upper"])
    bt = clustering.build_block_tree(tree, eta=1.0)
    lr, lc = bt.flat.leaves()
    assert np.array_equal(lr, g["leaf_row"]) and np.array_equal(lc, g["leaf_col"])
    assert np.array_equal(bt.flat.state[bt.flat.leaf_ids] == 0, g["leaf_adm"])


def test_bench_scaling_config_arguments(monkeypatch):
    """bench.py defaults: C2 is the headline workload and every line also
    carries the scaling configuration C4 (BASELINE configs[3])."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    a = bench.parse()
    assert (a.level, a.eps, a.gpus) == (6, 1e-6, 1)
    assert (a.scale_level, a.scale_eps) == (8, 1e-8)
    assert bench.workload(a)["triangles"] == 32768
    assert "524288 triangles" in bench.scaling_workload(a) and "configs[3]" in bench.scaling_workload(a)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--scale-level", "7", "--scale-eps", "1e-6"])
    b = bench.parse()
    assert "configs[3]" not in bench.scaling_workload(b)
