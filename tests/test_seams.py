"""The device seams inside greencross itself (the evaluator
contract of batchexec.py:70-76 and the Green-factor functions resolved as
module attributes at gca.py:188-190).

The stock reference installed for the reference arm (baseline/_ref, it
ships to the GPU box) runs its own pipeline - cli.build_h2_operator with its
BatchExecutor thread pool, capacity sealing and ordered scatter, its
build_cluster_basis recursion and its host ACA - with only three module
attributes replaced by this package's device functions:
greencross.assembly.galerkin_pair_evaluator, green_row_factor and
green_col_factor (INTEGRATION.md option 2).  The result must equal the
reference's own fixtures (tests/golden/h2_sphere4_eps1e-4.npz, made by the
unpatched reference)."""

import os
import sys

import numpy as np
import pytest

from conftest import ROOT, golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - GPU box only
    pytest.skip("no CUDA device", allow_module_level=True)

_REF = os.path.join(ROOT, "baseline", "_ref")
if not os.path.isdir(os.path.join(_REF, "greencross")):  # pragma: no cover
    pytest.skip("baseline/_ref (the stock reference install) is absent", allow_module_level=True)


@pytest.fixture(scope="module")
def greencross():
    sys.path.insert(0, _REF)
    try:
        import greencross
        from greencross import assembly, batchexec, cli, clustering, gca, geometry, h2  # noqa: F401
        yield greencross
    finally:
        sys.path.remove(_REF)


def _adapters():
    """Device seam functions taking greencross objects (its TriangleMesh,
    its _Rows stubs and BoundingBox, its GreenRule) - the shim a greencross
    maintainer would register."""
    from paper_1810_08429_b200 import assembly as dev_asm
    from paper_1810_08429_b200 import geometry as dev_geo
    cache = {}

    def ours(mesh):
        m = cache.get(id(mesh))
        if m is None:
            m = cache[id(mesh)] = (mesh, dev_geo.TriangleMesh(mesh.vertices, mesh.triangles))
        return m[1]

    def galerkin_pair_evaluator(kind, mesh, basis, q_reg, q_sing):
        return dev_asm.galerkin_pair_evaluator(kind, ours(mesh), basis, q_reg, q_sing)

    def green_row_factor(cluster, rule, mesh, basis, orders=(3, 5)):
        return dev_asm.green_row_factor(cluster, rule, ours(mesh), basis, orders)

    def green_col_factor(pair, rule, mesh, basis, orders=(3, 5)):
        return dev_asm.green_col_factor(pair, rule, ours(mesh), basis, orders)
    return galerkin_pair_evaluator, green_row_factor, green_col_factor


def test_greencross_pipeline_on_device_seams(greencross, monkeypatch):
    """cli.build_h2_operator of the stock reference at C1 (sphere L4, eps
    1e-4, 8 executor threads) with the device evaluator and Green factors:
    trees and block leaves bit-exact, pivot sets bit-exact (the reference's
    own host ACA runs on the device factors), block entries and the
    reference's own mvm / mvm_t within 1e-12 of the unpatched reference."""
    from greencross import assembly, cli, h2
    ev, row, col = _adapters()
    monkeypatch.setattr(assembly, "galerkin_pair_evaluator", ev)
    monkeypatch.setattr(assembly, "green_row_factor", row)
    monkeypatch.setattr(assembly, "green_col_factor", col)
    g = golden("h2_sphere4_eps1e-4.npz")
    mesh = greencross.geometry.build_sphere_mesh(4)
    cfg = cli.ExperimentConfig(level=4, geometry="plane", basis="constant", disc="galerkin", eta=1.0, m=3,
                               delta_factor=0.5, eps=1e-4, leaf_size=16, q_reg=3, q_sing=5, lam=0.5,
                               source=(2.0, 0.0, 0.0), seed=0)
    hm, tree, bt = cli.build_h2_operator(mesh, cfg)
    assert np.array_equal(tree.perm, g["perm"])
    leaves = bt.leaves()
    assert np.array_equal([lf.row.index for lf in leaves], g["leaf_row"])
    assert np.array_equal([lf.col.index for lf in leaves], g["leaf_col"])
    for side, basis in (("row", hm.row_basis), ("col", hm.col_basis)):
        nodes = basis.nodes()
        assert [b.cluster.index for b in nodes] == g[side + "_node"].tolist()
        assert [b.rank for b in nodes] == g[side + "_rank"].tolist()
        off = 0
        for b, r in zip(nodes, g[side + "_rank"]):
            assert np.array_equal(np.sort(b.pivots), np.sort(g[side + "_piv"][off:off + r]))
            off += r
    for key, blocks in (("coup", hm.coupling), ("near", hm.nearfield)):
        off = 0
        for i, shp in zip(g[key + "_pick"], g[key + "_shape"]):
            ref = g[key + "_vals"][off:off + int(np.prod(shp))].reshape(shp)
            off += int(np.prod(shp))
            v = blocks[int(i)].values
            assert v.shape == tuple(shp)
            if key == "near":
                assert np.max(np.abs(v - ref)) <= 1e-12 * np.max(np.abs(ref))
    for x, y, yt in zip(g["x"], g["mvm"], g["mvm_t"]):
        assert np.linalg.norm(h2.mvm(hm, x) - y) <= 1e-12 * np.linalg.norm(y)
        assert np.linalg.norm(h2.mvm_t(hm, x) - yt) <= 1e-12 * np.linalg.norm(yt)
    assert [s["tasks"] for s in hm.exec_stats] == g["exec_tasks"].tolist()


def test_greencross_executor_threads_and_capacity_invariant(greencross, monkeypatch):
    """The reference's BatchExecutor driving the device evaluator from its
    thread pool: results bitwise independent of the thread count and the
    sealing capacity (the executor contract, batchexec.py:10-13 and
    test_batchexec.py:127-140), and equal to the device dense block."""
    from greencross import assembly
    from paper_1810_08429_b200 import assembly as dev_asm
    ev, _, _ = _adapters()
    monkeypatch.setattr(assembly, "galerkin_pair_evaluator", ev)
    mesh = greencross.geometry.build_sphere_mesh(3)
    rng = np.random.default_rng(2)
    rows = rng.choice(mesh.nt, 120, replace=False)
    cols = rng.choice(mesh.nt, 90, replace=False)
    outs = []
    for threads, capacity in ((1, 4096), (8, 512), (8, 97)):
        ex = assembly.make_galerkin_executor("slp", mesh, "constant", (3, 5), capacity, threads)
        bid = ex.register_block(len(rows), len(cols))
        assembly.enqueue_galerkin_tasks(ex, mesh, "constant", rows, cols, bid)
        outs.append(ex.finalize()[bid])
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    from paper_1810_08429_b200 import geometry as dev_geo
    ours = dev_asm.assemble_galerkin_block("slp", dev_geo.TriangleMesh(mesh.vertices, mesh.triangles),
                                           "constant", rows, cols).values
    assert np.array_equal(outs[0], ours)
