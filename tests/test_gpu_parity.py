"""GPU parity: the CUDA path through the C-ABI against the reference
fixtures (tests/golden, generated from greencross itself) and the CPU
oracle (oracle/port.py).

Tolerances: pivots, ranks, trees and block structure bit-exact; matrix
entries and matvec results within 1e-12 relative (the north star asks for
1e-10); Green factors within 2 ulp (numpy's SIMD r**3 is the only known
rounding difference); the pipeline is bitwise deterministic run to run.
"""

import numpy as np
import pytest

from conftest import PIPELINES, eps_of, golden, mesh_for
from oracle import port as P

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - GPU box only
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1810_08429_b200 import (_native, assembly, cli, clustering, gca, geometry,  # noqa: E402
                                   h2, quadrature as Q)
from paper_1810_08429_b200.errors import ConfigError, GeometryError  # noqa: E402


def rel(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("name", ["pairs_sphere3.npz", "pairs_cube3.npz"])
def test_pair_evaluator_seam(name):
    g = golden(name)
    mesh = mesh_for(name.replace("pairs_", "x_"))
    ev = assembly.galerkin_pair_evaluator("slp", mesh, "constant", 3, 5)
    for k in range(4):
        m = g["case"] == k
        got = ev(k, g["rows"][m], g["cols"][m], g["px"][m], g["py"][m])
        assert got.shape == (int(m.sum()), 1, 1)
        assert np.max(np.abs(got.ravel() - g["values"][m]) / np.abs(g["values"][m])) < 1e-13


def test_pair_values_independent_of_batching():
    g = golden("pairs_sphere3.npz")
    mesh = mesh_for("x_sphere3.npz")
    ev = assembly.galerkin_pair_evaluator("slp", mesh, "constant", 3, 5)
    for k in range(4):
        m = np.flatnonzero(g["case"] == k)
        full = ev(k, g["rows"][m], g["cols"][m], g["px"][m], g["py"][m]).ravel()
        half = ev(k, g["rows"][m][1::2], g["cols"][m][1::2], g["px"][m][1::2],
                  g["py"][m][1::2]).ravel()
        assert np.array_equal(full[1::2], half)


def test_dense_block_sphere2(sphere2):
    idx = np.arange(sphere2.nt)
    d = assembly.assemble_galerkin_block("slp", sphere2, "constant", idx, idx).values
    ref = golden("dense_sphere2.npz")["values"]
    assert rel(d, ref) < 1e-13
    assert np.max(np.abs(d - d.T)) <= 1e-13 * np.max(np.abs(d))
    assert np.all(np.linalg.eigvalsh(0.5 * (d + d.T)) > 0)


def test_subset_block_equals_dense_slice(sphere3):
    idx = np.arange(sphere3.nt)
    dense = assembly.assemble_galerkin_block("slp", sphere3, "constant", idx, idx).values
    rng = np.random.default_rng(4)
    r = rng.choice(sphere3.nt, 37, replace=False)
    c = rng.choice(sphere3.nt, 23, replace=False)
    sub = assembly.assemble_galerkin_block("slp", sphere3, "constant", r, c).values
    assert np.array_equal(sub, dense[np.ix_(r, c)])


def test_dense_block_vs_oracle_cube3():
    mesh = geometry.build_cube_mesh(3)
    rows = np.arange(0, mesh.nt, 7)
    cols = np.arange(mesh.nt)
    got = assembly.assemble_galerkin_block("slp", mesh, "constant", rows, cols).values
    nodes, gram = P.chart_nodes(mesh.vertices, mesh.triangles)
    ref = P.block(nodes, gram, mesh.triangles, rows, cols)
    assert rel(got, ref) < 1e-12


def test_green_factors_and_aca_vs_reference():
    g = golden("factors_sphere4.npz")
    mesh = geometry.build_sphere_mesh(4)
    tree = clustering.build_cluster_tree(mesh, "constant", 16)
    ro = ao = po = vo = 0
    for i, node in enumerate(g["node"]):
        R = int(g["nrows"][i])
        cl = tree.flat.node(int(node))
        stub = gca_stub(g["rows"][ro:ro + R], cl.box)
        rule = Q.green_box_rule(cl.box, 0.5 * cl.box.diameter(), 3)
        a = (assembly.green_col_factor((stub, stub), rule, mesh, "constant") if g["side"][i]
             else assembly.green_row_factor(stub, rule, mesh, "constant"))
        ref = g["A"][ao:ao + a.size].reshape(a.shape)
        # bit-exact except where numpy's SIMD r**3 rounds differently from
        # the correctly rounded cube (<= 1 ulp per term, a few ulp per sum)
        ulps = np.abs(a - ref) / np.spacing(np.abs(ref))
        assert np.max(ulps) <= 8.0
        assert np.mean(a == ref) >= 0.9
        interp = gca.aca_interpolation(ref, 1e-6)
        r = int(g["npiv"][i])
        assert np.array_equal(interp.pivots, g["piv"][po:po + r])
        vref = g["V"][vo:vo + R * r].reshape(R, r)
        assert np.array_equal(interp.v[interp.pivots], np.eye(r))
        assert rel(interp.v, vref) < 1e-11
        ro, ao, po, vo = ro + R, ao + a.size, po + r, vo + R * r


class gca_stub:
    def __init__(self, rows, box):
        self.indices, self.box = rows, box


def test_aca_known_answers():
    g = golden("aca_kats.npz")
    ao = po = vo = 0
    for (n, w), e, r in zip(g["shape"], g["eps"], g["npiv"]):
        a = g["A"][ao:ao + n * w].reshape(n, w)
        it = gca.aca_interpolation(a, e)
        assert np.array_equal(it.pivots, g["piv"][po:po + r])
        assert it.v.shape == (n, r)
        if r:
            assert rel(it.v, g["V"][vo:vo + n * r].reshape(n, r)) < 1e-12
        ao, po, vo = ao + n * w, po + r, vo + n * r
    assert len(gca.aca_interpolation(np.random.default_rng(2).standard_normal((50, 10)),
                                     1e-14, max_rank=4).pivots) == 4


@pytest.fixture(scope="module", params=PIPELINES)
def built(request):
    name = request.param
    mesh = mesh_for(name)
    cfg = cli.default_config(eps=eps_of(name))
    hm, tree, bt = cli.build_h2_operator(mesh, cfg)
    return name, golden(name), mesh, hm, tree, bt


def test_pipeline_structure_and_pivots(built):
    name, g, mesh, hm, tree, bt = built
    assert np.array_equal(tree.perm, g["perm"])
    lr, lc = bt.flat.leaves()
    assert np.array_equal(lr, g["leaf_row"]) and np.array_equal(lc, g["leaf_col"])
    for side, basis in (("row", hm.row_basis), ("col", hm.col_basis)):
        nodes = basis.nodes()
        assert [b.cluster.index for b in nodes] == g[side + "_node"].tolist()
        assert [b.rank for b in nodes] == g[side + "_rank"].tolist()
        ref = _ref_pivots(g, side)
        # pivot sets bit-exact everywhere; pivot order may flip only at
        # ULP-level near-ties of |R| (numpy's SIMD r**3)
        order_diff = 0
        for b in nodes:
            rp = ref[b.cluster.index]
            assert np.array_equal(np.sort(b.pivots), np.sort(rp)), b.cluster.index
            order_diff += not np.array_equal(b.pivots, rp)
        assert order_diff <= max(1, len(nodes) // 100)
        if "sphere" in name:
            assert order_diff == 0


def _ref_pivots(g, side):
    out, off = {}, 0
    for i, r in zip(g[side + "_node"].tolist(), g[side + "_rank"].tolist()):
        out[i] = g[side + "_piv"][off:off + r]
        off += r
    return out


def test_pipeline_bases(built):
    name, g, mesh, hm, tree, bt = built
    for side, basis in (("row", hm.row_basis), ("col", hm.col_basis)):
        off = 0
        for idx, kind, r, c in g[side + "_mat_meta"]:
            bn = basis._by_index[int(idx)]
            m = bn.v if kind == 0 else bn.transfer
            ref = g[side + "_mat_vals"][off:off + r * c].reshape(r, c)
            off += r * c
            assert m.shape == ref.shape
            assert np.linalg.norm(m - ref) <= 1e-10 * max(np.linalg.norm(ref), 1.0)


def test_pipeline_block_values(built):
    name, g, mesh, hm, tree, bt = built
    rp, cp = _ref_pivots(g, "row"), _ref_pivots(g, "col")
    for key, blocks in (("coup", hm.coupling), ("near", hm.nearfield)):
        off = 0
        for i, shp in zip(g[key + "_pick"], g[key + "_shape"]):
            blk = blocks[int(i)]
            v = blk.values
            ref = g[key + "_vals"][off:off + int(np.prod(shp))].reshape(shp)
            off += int(np.prod(shp))
            assert v.shape == tuple(shp)
            if key == "coup":   # entries keyed by (row pivot, column pivot)
                mr = hm.row_basis.node(blk.row).pivots
                mc = hm.col_basis.node(blk.col).pivots
                ir = np.argsort(mr)[np.argsort(np.argsort(rp[blk.row.index]))]
                ic = np.argsort(mc)[np.argsort(np.argsort(cp[blk.col.index]))]
                v = v[np.ix_(ir, ic)]
            assert rel(v, ref) < 1e-12


def test_pipeline_matvec(built):
    name, g, mesh, hm, tree, bt = built
    for x, y, yt in zip(g["x"], g["mvm"], g["mvm_t"]):
        assert np.linalg.norm(h2.mvm(hm, x) - y) <= 1e-12 * np.linalg.norm(y)
        assert np.linalg.norm(h2.mvm_t(hm, x) - yt) <= 1e-12 * np.linalg.norm(yt)


def test_pipeline_storage_and_stats(built):
    name, g, mesh, hm, tree, bt = built
    rep = h2.storage_report(hm)
    assert {k: rep[k] for k in g["storage_keys"]} == dict(zip(g["storage_keys"].tolist(),
                                                              g["storage_vals"].tolist()))
    assert [s["tasks"] for s in hm.exec_stats] == g["exec_tasks"].tolist()
    assert [s["case"] for s in hm.exec_stats] == [0, 1, 2, 3]
    # the reference executor seals every case's list at capacity 4096 and
    # once more for a partial tail (batchexec.py:37-52, 154-166)
    assert [s["batches"] for s in hm.exec_stats] == [-(-int(t) // 4096) for t in g["exec_tasks"]]
    assert all(s["wall_s"] >= 0.0 for s in hm.exec_stats)


@pytest.mark.parametrize("mesh_fn,basis,eta", [("sphere5", "constant", 1.0), ("sphere4", "linear", 0.7),
                                                ("cube4", "constant", 2.5), ("sphere6", "constant", 1.0)])
def test_device_block_tree_equals_host_builders(mesh_fn, basis, eta):
    """gc_bt_level (one tree level per launch pair, on the device) builds the
    nodes, order, keys and parents of the numpy builder exactly."""
    mesh = (geometry.build_sphere_mesh if mesh_fn.startswith("sphere") else geometry.build_cube_mesh)(
        int(mesh_fn[-1]))
    tree = clustering.build_cluster_tree(mesh, basis, 16, device=torch.device("cuda", 0))
    assert getattr(tree.flat, "_device", None) is not None
    a = clustering.build_block_tree(tree, eta=eta).flat
    b = clustering._build_block_tree_arrays(tree, eta=eta).flat
    for k in ("row", "col", "state", "level", "key", "parent_of", "leaf_ids"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


def test_build_h2_returns_before_the_quadrature_settles():
    """build_h2 (plane charts) does not synchronise: the statistics settle on
    first use, once, and equal a synchronous rebuild's."""
    mesh = geometry.build_sphere_mesh(3)
    cfg = cli.default_config(eps=1e-4)
    hm, tree, bt = cli.build_h2_operator(mesh, cfg)
    assert hm._settle is not None                       # still pending
    st = hm.exec_stats
    assert hm._settle is None and hm.settle().exec_stats == st
    assert [s["tasks"] for s in st] == [s["tasks"] for s in cli.build_h2_operator(mesh, cfg)[0].exec_stats]
    assert all(s["wall_s"] > 0.0 for s in st if s["tasks"])


def test_stats_report(built, tmp_path):
    """``greencross stats`` CSV (pkg/tests/test_cli.py:145-154): header,
    case names, tasks / batches / seconds per case."""
    import csv
    name, g, mesh, hm, tree, bt = built
    out = str(tmp_path / "stats.csv")
    cli.write_stats(out, hm)
    with open(out) as fh:
        rows = list(csv.DictReader(fh))
    assert list(rows[0].keys()) == cli.STATS_COLUMNS
    assert [r["case"] for r in rows] == list(cli.CASE_NAMES)
    assert [int(r["tasks"]) for r in rows] == g["exec_tasks"].tolist()
    assert all(int(r["batches"]) >= 1 for r in rows)
    assert all(float(r["wall_s"]) >= 0.0 for r in rows)


def test_pipeline_bitwise_deterministic(built):
    name, g, mesh, hm, tree, bt = built
    cfg = cli.default_config(eps=eps_of(name))
    hm2, _, _ = cli.build_h2_operator(mesh, cfg)
    assert torch.equal(hm.dev.coup, hm2.dev.coup) and torch.equal(hm.dev.near, hm2.dev.near)
    assert torch.equal(hm.row_basis.store.V, hm2.row_basis.store.V)
    x = g["x"][0]
    assert np.array_equal(h2.mvm(hm, x), h2.mvm(hm2, x))
    # graph replay == eager launch sequence, bitwise
    p = h2.plan(hm)
    xd = torch.from_numpy(x).cuda()
    y1 = torch.empty_like(xd)
    p.run(xd, y1, phase_events=(torch.cuda.Event(), torch.cuda.Event()))
    assert np.array_equal(y1.cpu().numpy(), h2.mvm(hm, x))


def test_oracle_full_pipeline_sphere3(sphere3):
    cfg = cli.default_config(eps=1e-4)
    hm, tree, bt = cli.build_h2_operator(sphere3, cfg)
    o = P.H2(sphere3.vertices, sphere3.triangles, 1e-4)
    for bn in hm.row_basis.nodes():
        assert np.array_equal(bn.pivots, o.bases["row"][bn.cluster.index]["piv"])
    x = np.random.default_rng(9).standard_normal(sphere3.nt)
    y = o.mvm(x)
    assert np.linalg.norm(h2.mvm(hm, x) - y) <= 1e-12 * np.linalg.norm(y)


def test_matvec_properties_c2():
    """Size-independent properties at the benchmark size (C2)."""
    mesh = geometry.build_sphere_mesh(6)
    hm, _, _ = cli.build_h2_operator(mesh, cli.default_config(eps=1e-6))
    rng = np.random.default_rng(4)
    x, y = rng.standard_normal((2, mesh.nt))
    hx, hy = h2.mvm(hm, x), h2.mvm(hm, y)
    lin = h2.mvm(hm, 1.5 * x - 2.0 * y)
    assert np.linalg.norm(lin - (1.5 * hx - 2.0 * hy)) <= 1e-13 * np.linalg.norm(hx)
    assert abs(y @ hx - x @ h2.mvm_t(hm, y)) <= 1e-12 * abs(y @ hx)
    # single layer is symmetric: compression error at eps 1e-6 bounds the asymmetry
    assert abs(y @ hx - x @ hy) <= 1e-5 * abs(y @ hx)
    # near-field spot check against the oracle
    nodes, gram = P.chart_nodes(mesh.vertices, mesh.triangles)
    for i in rng.choice(len(hm.nearfield), 10, replace=False):
        blk = hm.nearfield[int(i)]
        ref = P.block(nodes, gram, mesh.triangles, blk.row.indices, blk.col.indices)
        assert rel(blk.values, ref) < 1e-12
    for i in rng.choice(len(hm.coupling), 10, replace=False):
        blk = hm.coupling[int(i)]
        ref = P.block(nodes, gram, mesh.triangles, hm.row_basis.node(blk.row).pivots,
                      hm.col_basis.node(blk.col).pivots)
        assert rel(blk.values, ref) < 1e-12


@pytest.mark.parametrize("cfg", ["c3", "c4"])
def test_properties_and_block_samples_full_size(cfg):
    """C3 (cube L7, 131,072 triangles, eps 1e-6: edges and corners stress the
    singular rules) and C4 (sphere L8, 524,288 triangles, eps 1e-8, the
    multi-GPU configuration) at full size, through size-independent
    properties: linearity, the mvm / mvm_t adjoint, near-symmetry of the
    single layer within the compression error, and a random sample of stored
    near-field and coupling blocks re-derived by the dense-block path
    (bitwise) and by the oracle (<= 1e-12)."""
    mesh = geometry.build_cube_mesh(7) if cfg == "c3" else geometry.build_sphere_mesh(8)
    eps = 1e-6 if cfg == "c3" else 1e-8
    hm, _, _ = cli.build_h2_operator(mesh, cli.default_config(eps=eps))
    rng = np.random.default_rng(8)
    x, y = rng.standard_normal((2, mesh.nt))
    hx, hy = h2.mvm(hm, x), h2.mvm(hm, y)
    lin = h2.mvm(hm, 1.5 * x - 2.0 * y)
    assert np.linalg.norm(lin - (1.5 * hx - 2.0 * hy)) <= 1e-13 * np.linalg.norm(hx)
    assert abs(y @ hx - x @ h2.mvm_t(hm, y)) <= 1e-12 * abs(y @ hx)
    assert abs(y @ hx - x @ hy) <= 10 * eps * abs(y @ hx)
    nodes, gram = P.chart_nodes(mesh.vertices, mesh.triangles)
    for i in rng.choice(len(hm.nearfield), 8, replace=False):
        blk = hm.nearfield[int(i)]
        r, c = blk.row.indices, blk.col.indices
        assert np.array_equal(blk.values, assembly.assemble_galerkin_block("slp", mesh, "constant", r, c).values)
        assert rel(blk.values, P.block(nodes, gram, mesh.triangles, r, c)) < 1e-12
    for i in rng.choice(len(hm.coupling), 4, replace=False):
        blk = hm.coupling[int(i)]
        r, c = hm.row_basis.node(blk.row).pivots, hm.col_basis.node(blk.col).pivots
        assert np.array_equal(blk.values, assembly.assemble_galerkin_block("slp", mesh, "constant", r, c).values)
        assert rel(blk.values, P.block(nodes, gram, mesh.triangles, r, c)) < 1e-12


def test_errors_map_to_reference_classes(sphere2):
    with pytest.raises(ConfigError):
        assembly.assemble_galerkin_block("hyp", sphere2, "constant", [0], [1])
    with pytest.raises(ConfigError):
        assembly.galerkin_pair_evaluator("slp", sphere2, "quadratic", 3, 5)
    tree = clustering.build_cluster_tree(sphere2, "constant", 16)
    leaf = tree.leaves()[0]
    # an expansion point exactly on a surface quadrature point trips the
    # touch guard (assembly._touch_guard): reproduce the device's point
    t = int(leaf.indices[0])
    nodes = geometry.chart_pack(sphere2).nodes[t]
    n6 = geometry.shape_functions(Q.triangle_gauss(3)[0])
    z = np.zeros(3)
    for a in range(6):
        z = z + n6[0, a] * nodes[a]
    bad = Q.GreenRule(z[None, :], np.ones(1), np.array([[1.0, 0.0, 0.0]]), 1)
    with pytest.raises(GeometryError):
        assembly.green_row_factor(leaf, bad, sphere2, "constant")
    with pytest.raises(ConfigError):
        h2.mvm(cli.build_h2_operator(sphere2, cli.default_config())[0], np.zeros(3))


def test_native_launches_counted(sphere2):
    before = _native.launch_count()
    assembly.assemble_galerkin_block("slp", sphere2, "constant", [0, 1], [2, 3])
    assert _native.launch_count() > before


def test_sharded_operator_world1_matches_full():
    """The block-row sharded device path (parallel.py) at world size 1 over
    NCCL equals the single-operator product (the N>1 exchange logic is
    covered on the CPU with gloo in tests/test_parallel.py)."""
    import os
    import socket
    import torch.distributed as dist
    from paper_1810_08429_b200 import parallel
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        mesh = geometry.build_sphere_mesh(4)
        cfg = cli.default_config(eps=1e-6)
        sh = parallel.build_sharded_operator(mesh, cfg)
        hm, tree, _ = cli.build_h2_operator(mesh, cfg)
        x = np.random.default_rng(3).standard_normal(mesh.nt)
        xt = torch.from_numpy(x[tree.perm]).cuda()
        ys = sh.mvm_local(xt).cpu().numpy()
        # the sharded product, NCCL all-gathers included, replays as one CUDA graph
        assert sh.plan.graph is not None
        y = np.empty(mesh.nt)
        y[tree.perm] = ys
        ref = h2.mvm(hm, x)
        assert np.linalg.norm(y - ref) <= 1e-13 * np.linalg.norm(ref)
        assert np.array_equal(sh.mvm_local(xt).cpu().numpy(), ys)
        # the reference-order API (full external vector in and out)
        assert np.linalg.norm(sh.mvm(x) - ref) <= 1e-13 * np.linalg.norm(ref)
        out = torch.empty_like(xt)
        assert sh.mvm_slice(xt, out) is out and torch.equal(out.cpu(), torch.from_numpy(ys))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("q", [2, 4, 5, 6])
def test_other_quadrature_orders_vs_oracle(q):
    """C5 orders (q_reg = q_sing = q): blocks against the oracle's
    reference-order restatement with the reference's full rules."""
    mesh = geometry.build_sphere_mesh(2)
    rows = np.arange(0, mesh.nt, 3)
    cols = np.arange(mesh.nt)
    got = assembly.assemble_galerkin_block("slp", mesh, "constant", rows, cols, orders=(q, q)).values
    nodes, gram = P.chart_nodes(mesh.vertices, mesh.triangles)
    ref = P.block(nodes, gram, mesh.triangles, rows, cols, q=(q, q))
    assert rel(got, ref) < 1e-12


def test_matvec_graph_equals_serial_and_repeats():
    """The captured product (native executor: streams, priorities, one
    graph) == the serial eager launch sequence bitwise, and repeated
    replays (split-panel counters re-armed in-kernel) stay bitwise equal."""
    mesh = geometry.build_sphere_mesh(5)
    hm, _, _ = cli.build_h2_operator(mesh, cli.default_config(eps=1e-6))
    x = torch.from_numpy(np.random.default_rng(5).standard_normal(mesh.nt)).cuda()
    p = h2.PanelPlan(hm)
    y0, y1, y2 = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
    p.run(x, y0, serial=True)
    p.capture()
    p.run(x, y1)
    p.run(x, y2)
    torch.cuda.synchronize()
    assert torch.equal(y0, y1) and torch.equal(y1, y2)


def _solver_op(eps):
    mesh = geometry.build_sphere_mesh(4)
    hm, _, _ = cli.build_h2_operator(mesh, cli.default_config(eps=eps))
    return mesh, hm


def test_device_solvers_match_reference_c1():
    """cg_solve / cgnr_solve / spectral_error_estimate (h2.py:144-253) with
    every vector in HBM against the reference's own runs on its own C1
    operators (tests/golden/make_golden.py --solvers).  The discrete SLP
    operator is ill-conditioned (|x| ~ 1e4 |b|), so a 1e-15 difference per
    product grows along the iteration: the histories must agree to 1e-6
    relative over the first 10 iterations, the convergence flags and the
    iteration counts (within 10 %) must match; a converged device iterate
    must meet the tolerance against the operator itself and agree with the
    reference's to 1e-4 relative (condition-number limited), a capped run
    must end at the reference's residual level (within 20 %).  The power-iteration
    estimate is stable: within 1e-8."""
    g = golden("solvers_sphere4.npz")
    mesh, hm = _solver_op(1e-4)
    _, hm6 = _solver_op(1e-6)
    op = h2.as_operator(hm)
    b = g["b"]

    def check(res, ref_res, ref_x, ref_conv, tol):
        assert bool(res.converged) == bool(ref_conv)
        assert abs(len(res.residuals) - len(ref_res)) <= max(2, len(ref_res) // 10)
        assert np.allclose(res.residuals[:10], ref_res[:10], rtol=1e-6, atol=0)
        true_res = np.linalg.norm(b - h2.mvm(hm, res.x))
        if res.converged:
            assert true_res <= 1.5 * tol * np.linalg.norm(b)
            assert np.linalg.norm(res.x - ref_x) <= 1e-4 * np.linalg.norm(ref_x)
        else:                       # iteration cap reached by both: same residual level
            assert abs(res.residuals[-1] - ref_res[-1]) <= 0.2 * ref_res[-1]
    check(h2.cg_solve(op, b, tol=1e-10, max_iter=300), g["cg_res"], g["cg_x"], g["cg_conv"], 1e-10)
    check(h2.cgnr_solve(op, b, tol=1e-8, max_iter=300), g["cgnr_res"], g["cgnr_x"], g["cgnr_conv"], 1e-8)
    err, relerr = h2.spectral_error_estimate(h2.as_operator(hm6), op, mesh.nt, iters=30, seed=3)
    assert abs(err - float(g["spec_err"])) <= 1e-8 * float(g["spec_err"])
    assert abs(relerr - float(g["spec_rel"])) <= 1e-8 * float(g["spec_rel"])


def test_device_solvers_on_host_closures():
    """The reference's own solver tests on plain numpy closures
    (test_h2.py:96-156): the device loops call them on host copies."""
    rng = np.random.default_rng(0)
    m = rng.standard_normal((40, 40))
    a = m @ m.T + 40 * np.eye(40)
    b = rng.standard_normal(40)
    res = h2.cg_solve(lambda v: a @ v, b, tol=1e-10)
    assert res.converged and np.linalg.norm(a @ res.x - b) <= 1e-9 * np.linalg.norm(b)
    res = h2.cg_solve(lambda v: v, np.zeros(5))
    assert res.converged and np.array_equal(res.x, np.zeros(5))
    n = rng.standard_normal((30, 30)) + 10 * np.eye(30)

    def apply(v, trans=False):
        return n.T @ v if trans else n @ v
    res = h2.cgnr_solve(apply, b[:30], tol=1e-10, max_iter=1000)
    assert res.converged and np.linalg.norm(n @ res.x - b[:30]) <= 1e-9 * np.linalg.norm(b[:30])
    da, db = np.diag([3.0, 2.0, 1.0]), np.diag([3.0, 2.0, 0.5])
    err, rel = h2.spectral_error_estimate(lambda v, t=False: da @ v, lambda v, t=False: db @ v, 3, iters=200)
    assert abs(err - 0.5) < 1e-6 and abs(rel - 0.5 / 3.0) < 1e-6
    with pytest.raises(ConfigError):
        h2.spectral_error_estimate(lambda v, t=False: v, lambda v, t=False: v, 3, iters=0)


@pytest.mark.parametrize("geo,level,cfg_kw", [
    ("sphere", 5, dict(eps=1e-6)), ("cube", 4, dict(eps=1e-6)),
    ("sphere", 4, dict(eps=1e-4, basis="linear")),
    ("sphere", 3, dict(eps=1e-4, basis="linear", disc="collocation"))])
def test_tiered_transforms_match_level_by_level(geo, level, cfg_kw):
    """Tiered transforms (tiers.py: composed transfers, one launch per tier)
    == the level-by-level nested-basis recursion (tiers="off") to rounding,
    for automatic and forced tier boundaries, symmetric and row != column
    bases; graph replay == serial eager bitwise."""
    mesh = (geometry.build_sphere_mesh if geo == "sphere" else geometry.build_cube_mesh)(level)
    hm, _, _ = cli.build_h2_operator(mesh, cli.default_config(**cfg_kw))
    n = hm.shape[1]
    x = torch.from_numpy(np.random.default_rng(3).standard_normal(n)).cuda()
    p0 = h2.PanelPlan(hm, tiers="off")
    assert p0.tiers is None
    y0 = torch.empty(hm.shape[0], dtype=torch.float64, device="cuda")
    p0.run(x, y0, serial=True)
    for tiers in ("auto", [0], [1, 3], [0, 2, 4], [2]):
        p = h2.PanelPlan(hm, tiers=tiers)
        assert p.tiers is not None
        y1, y2 = torch.empty_like(y0), torch.empty_like(y0)
        p.run(x, y1, serial=True)
        p.capture()
        p.run(x, y2)
        p.run(x, y2)
        torch.cuda.synchronize()
        assert torch.equal(y1, y2), tiers
        assert (y1 - y0).norm().item() <= 1e-13 * y0.norm().item(), tiers


@pytest.mark.parametrize("level,eps", [(1, 1e-2), (2, 1e-2), (2, 1e-10), (3, 1e-10)])
def test_small_and_degenerate_operators(level, eps):
    """Tiny trees (few or no admissible blocks, full-rank or rank-0 bases):
    the default plan (tiers, native executor) == the level-by-level plan to
    rounding, and both approximate the dense Galerkin matrix to ~eps."""
    mesh = geometry.build_sphere_mesh(level)
    hm, _, _ = cli.build_h2_operator(mesh, cli.default_config(eps=eps))
    x = np.random.default_rng(level).standard_normal(mesh.nt)
    y = h2.mvm(hm, x)
    dense = assembly.assemble_galerkin_block("slp", mesh, "constant", np.arange(mesh.nt),
                                             np.arange(mesh.nt)).values
    yd = dense @ x
    assert np.linalg.norm(y - yd) <= max(100 * eps, 1e-12) * np.linalg.norm(yd)
    p = h2.PanelPlan(hm, tiers="off")
    xd = torch.from_numpy(x).cuda()
    y0 = torch.empty_like(xd)
    p.run(xd, y0, serial=True)
    assert np.linalg.norm(y0.cpu().numpy() - y) <= 1e-13 * np.linalg.norm(y)


def test_mvm_20_seeded_vectors_c1():
    """SURVEY 8(c) parity protocol at C1: mvm and mvm_t of the 20 seeded
    N(0,1) vectors (default_rng(0)) against the reference's own products
    (tests/golden/make_golden.py --mvm20); bar 1e-10, held to 1e-12."""
    g = golden("mvm20_sphere4_eps1e-4.npz")
    mesh = geometry.build_sphere_mesh(4)
    hm, _, _ = cli.build_h2_operator(mesh, cli.default_config(eps=1e-4))
    xs = np.random.default_rng(0).standard_normal((20, mesh.nt))
    for x, y, yt in zip(xs, g["mvm"], g["mvm_t"]):
        assert np.linalg.norm(h2.mvm(hm, x) - y) <= 1e-12 * np.linalg.norm(y)
        assert np.linalg.norm(h2.mvm_t(hm, x) - yt) <= 1e-12 * np.linalg.norm(yt)


def test_graph_rebinding_to_caller_buffers():
    """The captured product re-pointed at caller buffers (gc_graph_retarget):
    alternating device inputs / outputs, the pinned host buffers of
    h2.mvm (zero-copy gather / scatter) and back all give the serial eager
    product bitwise, and the plan's static buffers are left untouched."""
    mesh = geometry.build_sphere_mesh(4)
    hm, _, _ = cli.build_h2_operator(mesh, cli.default_config(eps=1e-6))
    p = h2.plan(hm)
    assert p.graph is not None
    rng = np.random.default_rng(9)
    xs = [torch.from_numpy(rng.standard_normal(mesh.nt)).cuda() for _ in range(3)]
    ref = []
    for x in xs:
        y = torch.empty_like(x)
        p.run(x, y, serial=True)
        ref.append(y.clone())
    ys = [torch.empty_like(xs[0]) for _ in range(2)]
    for k in range(7):
        i = k % 3
        p.run(xs[i], ys[k % 2])
        torch.cuda.synchronize()
        assert torch.equal(ys[k % 2], ref[i])
        if k % 3 == 2:                            # host API in between
            got = h2.mvm(hm, xs[i].cpu().numpy())
            assert np.array_equal(got, ref[i].cpu().numpy())


def _sharded_worker(rank, world, port, out_dir, level, cfg_kw):
    import os
    import torch.distributed as dist
    from paper_1810_08429_b200 import parallel
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        mesh = geometry.build_sphere_mesh(level)
        sh = parallel.build_sharded_operator(mesh, cli.default_config(**cfg_kw))
        n = sh.shape[1]
        x = np.random.default_rng(3).standard_normal(n)
        perm = sh.h.row_tree.flat.perm
        xt = torch.from_numpy(x[perm][sh.layout.lo:sh.layout.hi].copy()).cuda()
        y = sh.mvm_slice(xt).cpu().numpy()
        np.save(os.path.join(out_dir, "y%d.npy" % rank), y)
        np.save(os.path.join(out_dir, "lo%d.npy" % rank), np.array([sh.layout.lo, sh.layout.hi]))
        # the reference-order API: full x in, full y out on every rank
        np.save(os.path.join(out_dir, "ext%d.npy" % rank), sh.mvm(x))
        # a second vector: the remote blocks must read this product's
        # all-gathered data, not the previous product's
        x2 = np.random.default_rng(4).standard_normal(n)
        xt2 = torch.from_numpy(x2[perm][sh.layout.lo:sh.layout.hi].copy()).cuda()
        np.save(os.path.join(out_dir, "y2_%d.npy" % rank), sh.mvm_slice(xt2).cpu().numpy())
        # a few of this rank's blocks, for the bitwise comparison with the
        # single-operator assembly (same per-task arithmetic on every rank)
        picks = []
        for blocks in (sh.h.coupling, sh.h.nearfield):
            for i in np.linspace(0, len(blocks) - 1, 4).astype(int) if len(blocks) else []:
                b = blocks[int(i)]
                picks.append((b.row.index, b.col.index, b.values.ravel()))
        np.save(os.path.join(out_dir, "blk%d.npy" % rank), np.array(picks, dtype=object), allow_pickle=True)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,level,cfg_kw", [
    (2, 5, dict(eps=1e-6)), (4, 5, dict(eps=1e-6)), (8, 5, dict(eps=1e-6)),
    (4, 4, dict(eps=1e-6, basis="linear")),                        # 1026 vertex DOFs: unequal shards
    (2, 3, dict(eps=1e-4, basis="linear", disc="collocation"))])
def test_sharded_operator_multirank_matches_full(world, level, cfg_kw, tmp_path):
    """The N>1 device path end to end: `world` ranks as processes sharing the
    one GPU (gloo collectives staged through the host - no kernel waits on
    another rank), each assembling its own block rows and bases; the
    concatenated row slices and every rank's external-order product equal
    the single-operator product - for the constant and linear Galerkin and
    the collocation operators, with equal and unequal shard sizes."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_sharded_worker, args=(world, port, str(tmp_path), level, cfg_kw), nprocs=world, join=True)
    mesh = geometry.build_sphere_mesh(level)
    hm, tree, _ = cli.build_h2_operator(mesh, cli.default_config(**cfg_kw))
    n = hm.shape[1]
    x = np.random.default_rng(3).standard_normal(n)
    yt = np.empty(n)
    sizes = []
    for g in range(world):
        lo, hi = np.load(tmp_path / ("lo%d.npy" % g))
        sizes.append(hi - lo)
        yt[lo:hi] = np.load(tmp_path / ("y%d.npy" % g))
    y = np.empty(n)
    y[tree.perm] = yt
    ref = h2.mvm(hm, x)
    assert np.linalg.norm(y - ref) <= 1e-13 * np.linalg.norm(ref)
    for g in range(world):
        ye = np.load(tmp_path / ("ext%d.npy" % g))
        assert np.linalg.norm(ye - ref) <= 1e-13 * np.linalg.norm(ref)
    x2 = np.random.default_rng(4).standard_normal(n)
    for g in range(world):
        lo, hi = np.load(tmp_path / ("lo%d.npy" % g))
        yt[lo:hi] = np.load(tmp_path / ("y2_%d.npy" % g))
    y[tree.perm] = yt
    ref2 = h2.mvm(hm, x2)
    assert np.linalg.norm(y - ref2) <= 1e-13 * np.linalg.norm(ref2)
    # the ranks' blocks are bitwise the single operator's (SURVEY 8e parity)
    full = {(b.row.index, b.col.index): b.values for blocks in (hm.coupling, hm.nearfield) for b in blocks}
    for g in range(world):
        for r, c, v in np.load(tmp_path / ("blk%d.npy" % g), allow_pickle=True):
            assert np.array_equal(full[(r, c)].ravel(), v)
    if cfg_kw.get("basis") == "linear" and world == 4:
        assert len(set(sizes)) > 1               # the padded all-gather path ran



# ---------------------------------------------------------------- double layer
# (first step: the DLP kernel, constant basis, plane charts)

@pytest.mark.parametrize("name,mesh_name", [("pairs_dlp_sphere3.npz", "x_sphere3"),
                                            ("pairs_dlp_cube3.npz", "x_cube3")])
def test_dlp_pair_evaluator_seam(name, mesh_name):
    """Device double-layer pair integrals vs the reference's values.  The
    identical-pair values are rounding noise around 0 (x - y lies in the
    plane of n_y), so every case is compared against the largest value."""
    g = golden(name)
    mesh = mesh_for(mesh_name)
    ev = assembly.galerkin_pair_evaluator("dlp", mesh, "constant", 3, 5)
    scale = np.max(np.abs(g["values"]))
    for k in range(4):
        m = g["case"] == k
        got = ev(k, g["rows"][m], g["cols"][m], g["px"][m], g["py"][m]).ravel()
        assert np.max(np.abs(got - g["values"][m])) <= 1e-13 * scale, "case %d" % k
        if k in (0, 1, 2):
            nz = np.abs(g["values"][m]) > 1e-6 * scale
            assert np.max(np.abs(got[nz] - g["values"][m][nz]) / np.abs(g["values"][m][nz])) < 1e-11


def test_dlp_dense_block_and_gauss_identity(sphere2):
    """Dense DLP block vs the reference, and the interior Gauss identity of
    the double layer on a closed surface: K 1 = -1/2 M 1 up to O(h)."""
    idx = np.arange(sphere2.nt)
    d = assembly.assemble_galerkin_block("dlp", sphere2, "constant", idx, idx).values
    ref = golden("dense_dlp_sphere2.npz")["values"]
    assert rel(d, ref) < 1e-13
    areas = 0.5 * geometry.chart_pack(sphere2).gram
    for L in (3, 4):
        m = geometry.build_sphere_mesh(L)
        i = np.arange(m.nt)
        k = assembly.assemble_galerkin_block("dlp", m, "constant", i, i).values
        a = 0.5 * geometry.chart_pack(m).gram
        err = np.linalg.norm(k.sum(axis=1) + 0.5 * a) / np.linalg.norm(0.5 * a)
        assert err < {3: 0.05, 4: 0.03}[L]
    assert areas.sum() > 0


def test_dlp_h2_matvec_vs_reference():
    """GCA-H2 of the double-layer operator (same nested bases, DLP coupling
    and near-field blocks, gca.py:282-312 with kind="dlp") vs the
    reference's H2: sampled near-field blocks and three matvecs."""
    g = golden("h2_dlp_sphere4_eps1e-6.npz")
    mesh = geometry.build_sphere_mesh(4)
    cfg = cli.default_config(eps=1e-6)
    tree = clustering.build_cluster_tree(mesh, "constant", 16)
    bt = clustering.build_block_tree(tree, eta=1.0)
    rm, cm = gca.coupling_marks(bt)
    rb = gca.build_cluster_basis(tree, mesh, "constant", 3, 0.5, 1e-6, "row", (3, 5), rm)
    cb = gca.build_cluster_basis(tree, mesh, "constant", 3, 0.5, 1e-6, "col", (3, 5), cm)
    hm = gca.build_h2(bt, rb, cb, mesh, "dlp", "constant", "galerkin", (3, 5))
    near = {(b.row.index, b.col.index): b.values for b in hm.nearfield}
    off = 0
    for r, c in zip(g["near_row"], g["near_col"]):
        v = near[(int(r), int(c))]
        ref = g["near_values"][off:off + v.size].reshape(v.shape)
        off += v.size
        assert np.max(np.abs(v - ref)) <= 1e-13 * np.max(np.abs(ref))
    for x, y in zip(g["x"], g["mvm"]):
        assert np.linalg.norm(h2.mvm(hm, x) - y) <= 1e-12 * np.linalg.norm(y)
    assert cfg.eps == 1e-6


# ---------------------------------------------------------------- linear basis
# (vertex DOFs, 3x3 pair integrals, device scatter)

@pytest.mark.parametrize("kind", ["slp", "dlp"])
def test_linear_pair_evaluator_seam(kind):
    g = golden("pairs_lin_%s_sphere3.npz" % kind)
    mesh = mesh_for("x_sphere3")
    ev = assembly.galerkin_pair_evaluator(kind, mesh, "linear", 3, 5)
    scale = np.max(np.abs(g["values"]))
    for k in range(4):
        m = g["case"] == k
        got = ev(k, g["rows"][m], g["cols"][m], g["px"][m], g["py"][m])
        assert got.shape == (int(m.sum()), 3, 3)
        # identical pairs of the double layer are rounding noise around 0
        # (x - y lies in the plane of n_y): 1e-12 of the largest value
        tol = 1e-12 if (kind, k) == ("dlp", 3) else 1e-13
        assert np.max(np.abs(got - g["values"][m])) <= tol * scale, "case %d" % k


def test_linear_dense_blocks(sphere2):
    g = golden("dense_lin_sphere2.npz")
    dofs = np.arange(sphere2.nv)
    for kind in ("slp", "dlp"):
        d = assembly.assemble_galerkin_block(kind, sphere2, "linear", dofs, dofs).values
        assert rel(d, g[kind]) < 1e-13, kind
    sub = assembly.assemble_galerkin_block("slp", sphere2, "linear", g["sub_rows"], g["sub_cols"]).values
    assert rel(sub, g["sub"]) < 1e-13
    # single layer: symmetric positive definite on the vertex DOFs
    d = assembly.assemble_galerkin_block("slp", sphere2, "linear", dofs, dofs).values
    assert np.max(np.abs(d - d.T)) <= 1e-13 * np.max(np.abs(d))
    assert np.all(np.linalg.eigvalsh(0.5 * (d + d.T)) > 0)
    # bitwise reproducible, and a sub-block equals the dense slice to rounding
    d2 = assembly.assemble_galerkin_block("slp", sphere2, "linear", dofs, dofs).values
    assert np.array_equal(d, d2)
    assert rel(sub, d[np.ix_(g["sub_rows"], g["sub_cols"])]) < 1e-13


@pytest.mark.parametrize("name,mesh_name,eps", [("h2_lin_sphere3_eps1e-4.npz", "x_sphere3", 1e-4),
                                                ("h2_lin_cube3_eps1e-6.npz", "x_cube3", 1e-6)])
def test_linear_h2_pipeline_vs_reference(name, mesh_name, eps):
    """GCA-H2 with the linear basis (vertex DOFs) against the reference:
    vertex tree, Green factors of sampled leaves, ranks and pivot sets per
    basis node, storage report and three matvecs."""
    g = golden(name)
    mesh = mesh_for(mesh_name)
    cfg = cli.default_config(eps=eps, basis="linear")
    hm, tree, bt = cli.build_h2_operator(mesh, cfg)
    assert np.array_equal(tree.perm, g["perm"])
    # Green row factors of sampled leaves (rows = vertices)
    off = 0
    for i in g["factor_nodes"]:
        node = tree.flat.node(int(i))
        rule = Q.green_box_rule(node.box, 0.5 * node.box.diameter(), 3)
        a = assembly.green_row_factor(node, rule, mesh, "linear")
        ref = g["factors"][off:off + a.size].reshape(a.shape)
        off += a.size
        assert np.max(np.abs(a - ref)) <= 1e-14 * np.max(np.abs(ref))
    for side, basis in (("row", hm.row_basis), ("col", hm.col_basis)):
        nodes = list(basis.nodes())
        assert [b.cluster.index for b in nodes] == g[side + "_node"].tolist()
        assert [b.rank for b in nodes] == g[side + "_rank"].tolist()
        got = np.concatenate([b.pivots for b in nodes])
        ref = g[side + "_piv"]
        o = 0
        for b in nodes:
            assert set(got[o:o + b.rank]) == set(ref[o:o + b.rank])
            o += b.rank
    rep = h2.storage_report(hm)
    assert {k: rep[k] for k in g["storage_keys"]} == dict(zip(g["storage_keys"].tolist(),
                                                              g["storage_vals"].tolist()))
    for x, y in zip(g["x"], g["mvm"]):
        assert np.linalg.norm(h2.mvm(hm, x) - y) <= 1e-12 * np.linalg.norm(y)


# ---------------------------------------------------------------- collocation

def test_collocation_seam_and_dense_blocks(sphere2):
    g = golden("colloc_pairs_sphere3.npz")
    mesh = mesh_for("x_sphere3")
    for kind in ("slp", "dlp"):
        ev = assembly.collocation_evaluator(kind, mesh, 3, 5)
        scale = np.max(np.abs(g[kind]))
        for k in (0, 1):
            m = g["case"] == k
            got = ev(k, g["rows"][m], g["cols"][m], None, g["py"][m])
            assert got.shape == (int(m.sum()), 1, 3)
            # dlp with the point at a corner: x - y lies in the plane of n_y, both
            # sides are rounding noise around 0 (the reference forms x - y by
            # cancellation, the device exactly)
            tol = 1e-10 if (kind, k) == ("dlp", 1) else 1e-13
            assert np.max(np.abs(got - g[kind][m])) <= tol * scale, (kind, k)
    d = golden("colloc_dense_sphere2.npz")
    dofs = np.arange(sphere2.nv)
    for kind in ("slp", "dlp"):
        got = assembly.assemble_collocation_block(kind, sphere2, "linear", dofs, dofs).values
        # the dlp diagonal is rounding noise around 0 on both sides (see above)
        assert rel(got, d[kind]) < (1e-11 if kind == "dlp" else 1e-13), kind
    # double-layer row sums approach -1/2 under refinement (interior Gauss
    # identity, test_assembly.py:108-118; on plane charts the vertex solid
    # angle converges with h)
    res = []
    for L in (2, 3, 4):
        m = geometry.build_sphere_mesh(L)
        k = assembly.assemble_collocation_block("dlp", m, "linear", np.arange(m.nv), np.arange(m.nv)).values
        res.append(np.abs(k.sum(axis=1) + 0.5).max())
    assert res[2] < res[1] < res[0]


def test_collocation_h2_vs_reference():
    g = golden("h2_colloc_sphere3_eps1e-4.npz")
    mesh = geometry.build_sphere_mesh(3)
    cfg = cli.default_config(eps=1e-4, basis="linear", disc="collocation")
    hm, tree, bt = cli.build_h2_operator(mesh, cfg)
    assert np.array_equal(tree.perm, g["perm"])
    for side, basis in (("row", hm.row_basis), ("col", hm.col_basis)):
        nodes = list(basis.nodes())
        assert [b.cluster.index for b in nodes] == g[side + "_node"].tolist()
        assert [b.rank for b in nodes] == g[side + "_rank"].tolist()
        got = np.concatenate([b.pivots for b in nodes])
        ref = g[side + "_piv"]
        o = 0
        for b in nodes:
            assert set(got[o:o + b.rank]) == set(ref[o:o + b.rank])
            o += b.rank
    for x, y in zip(g["x"], g["mvm"]):
        assert np.linalg.norm(h2.mvm(hm, x) - y) <= 1e-12 * np.linalg.norm(y)


# ---------------------------------------------------------------- curved charts

def _curved(level):
    return geometry.to_curved(geometry.build_sphere_mesh(level), project_to_unit_sphere=True)


def test_curved_pair_evaluator_seam():
    g = golden("curved_pairs_sphere3.npz")
    mesh = _curved(3)
    for kind in ("slp", "dlp"):
        for basis in ("constant", "linear"):
            ref = g["%s_%s" % (kind, basis)]
            ev = assembly.galerkin_pair_evaluator(kind, mesh, basis, 3, 5)
            scale = np.max(np.abs(ref))
            for k in range(4):
                m = g["case"] == k
                got = ev(k, g["rows"][m], g["cols"][m], g["px"][m], g["py"][m])
                assert got.shape == ref[m].shape
                assert np.max(np.abs(got - ref[m])) <= 1e-12 * scale, (kind, basis, k)


def test_curved_dense_blocks():
    g = golden("curved_dense_sphere2.npz")
    mesh = _curved(2)
    idx, dofs = np.arange(mesh.nt), np.arange(mesh.nv)
    d = assembly.assemble_galerkin_block("slp", mesh, "constant", idx, idx).values
    assert rel(d, g["slp_constant"]) < 1e-12
    d = assembly.assemble_galerkin_block("dlp", mesh, "linear", dofs, dofs).values
    assert rel(d, g["dlp_linear"]) < 1e-12
    d = assembly.assemble_collocation_block("dlp", mesh, "linear", dofs, dofs).values
    assert rel(d, g["colloc_dlp"]) < 1e-10
    # interior Gauss identity on the curved sphere (test_assembly.py:93-104):
    # (M/2 + K) 1 = 0 to O(h^2)
    k = assembly.assemble_galerkin_block("dlp", _curved(3), "linear", np.arange(258), np.arange(258)).values
    assert np.abs(k.sum(axis=1)).max() > 0
    m2 = g["mass_linear"]
    k2 = assembly.assemble_galerkin_block("dlp", mesh, "linear", dofs, dofs).values
    r = (0.5 * m2 + k2) @ np.ones(mesh.nv)
    assert np.linalg.norm(r) / np.linalg.norm(m2 @ np.ones(mesh.nv)) < 2e-5


@pytest.mark.parametrize("basis,level,name", [("constant", 3, "curved_h2_constant_sphere3.npz"),
                                              ("linear", 4, "curved_h2_linear_sphere4.npz")])
def test_curved_h2_vs_reference(basis, level, name):
    g = golden(name)
    mesh = _curved(level)
    cfg = cli.default_config(eps=1e-4, basis=basis)
    hm, tree, bt = cli.build_h2_operator(mesh, cfg)
    assert np.array_equal(tree.perm, g["perm"])
    off = 0
    for i in g["factor_nodes"]:
        node = tree.flat.node(int(i))
        rule = Q.green_box_rule(node.box, 0.5 * node.box.diameter(), 3)
        a = assembly.green_row_factor(node, rule, mesh, basis)
        ref = g["factors"][off:off + a.size].reshape(a.shape)
        off += a.size
        assert np.max(np.abs(a - ref)) <= 1e-13 * np.max(np.abs(ref))
    for side, b in (("row", hm.row_basis), ("col", hm.col_basis)):
        nodes = list(b.nodes())
        assert [x.rank for x in nodes] == g[side + "_rank"].tolist()
        got = np.concatenate([x.pivots for x in nodes])
        ref = g[side + "_piv"]
        o = 0
        for x in nodes:
            assert set(got[o:o + x.rank]) == set(ref[o:o + x.rank])
            o += x.rank
    for x, y in zip(g["x"], g["mvm"]):
        assert np.linalg.norm(h2.mvm(hm, x) - y) <= 1e-12 * np.linalg.norm(y)


@pytest.mark.parametrize("name,basis", [("h2_sphere5_eps1e-6.npz", "constant"), ("h2_cube4_eps1e-6.npz", "constant"),
                                        ("h2_lin_cube3_eps1e-6.npz", "linear")])
def test_device_cluster_tree_bitwise(name, basis):
    """The device cluster tree (csrc/tree.cu) equals the reference's tree
    bit for bit: permutation, ranges and boxes."""
    g = golden(name)
    mesh = mesh_for(name.replace("h2_lin_", "h2_"))
    t = clustering.build_cluster_tree(mesh, basis, 16, device=torch.device("cuda"))
    assert np.array_equal(t.perm, g["perm"])
    assert np.array_equal(t.flat.start, g["start"]) and np.array_equal(t.flat.stop, g["stop"])
    assert np.array_equal(t.flat.lower, g["lower"]) and np.array_equal(t.flat.upper, g["upper"])
    host = clustering.build_cluster_tree(mesh, basis, 16)
    assert np.array_equal(t.flat.depth, host.flat.depth) and np.array_equal(t.flat.left, host.flat.left)


@pytest.mark.parametrize("kind,level", [("sphere", 6), ("cube", 7), ("sphere", 2)])
def test_device_charts_bit_identical_to_host(kind, level):
    """gc_chart_pack (device chart data and cluster support boxes) == the
    host chart_pack / control_points / centroids bit for bit, signed zeros
    included (numpy's minimum / maximum tie rule)."""
    from paper_1810_08429_b200 import device
    mesh = (geometry.build_sphere_mesh if kind == "sphere" else geometry.build_cube_mesh)(level)
    ch = device.device_charts(mesh, torch.device("cuda", 0))
    pack = geometry.chart_pack(mesh)
    ctrl = geometry.control_points(mesh)
    sup = ch["support"].cpu().numpy()
    for got, ref in ((ch["corners"].cpu().numpy(), pack.nodes[:, :3]), (ch["gram"].cpu().numpy(), pack.gram),
                     (ch["normal"].cpu().numpy(), pack.normals[:, 0]), (sup[:, 6:], mesh.centroids())):
        assert got.tobytes() == np.ascontiguousarray(ref).tobytes()
    lo, hi = ctrl[:, 0].copy(), ctrl[:, 0].copy()
    for k in range(1, 6):
        np.minimum(lo, ctrl[:, k], out=lo)
        np.maximum(hi, ctrl[:, k], out=hi)
    assert sup[:, :3].tobytes() == lo.tobytes() and sup[:, 3:6].tobytes() == hi.tobytes()


def _expected_block_tables(bt, rf, cf, rs, cs, rng):
    """numpy restatement of build_h2's block loop (gca.py:296-310): leaves in
    DFS order, admissible -> coupling (ranks), inadmissible -> near field
    (cluster sizes), storage grouped stably by block row (a shard: local
    columns first inside each row)."""
    fb = bt.flat
    ids = fb.leaf_ids
    st, lr, lc = fb.state[ids], fb.row[ids], fb.col[ids]
    if rng is not None:
        k = (rf.start[lr] >= rng[0]) & (rf.stop[lr] <= rng[1])
        st, lr, lc = st[k], lr[k], lc[k]
    adm = st == 0
    out = []
    for rows, cols, nr, nc in ((lr[adm], lc[adm], rs.rank[lr[adm]], cs.rank[lc[adm]]),
                               (lr[~adm], lc[~adm], (rf.stop - rf.start)[lr[~adm]],
                                (cf.stop - cf.start)[lc[~adm]])):
        key = rows if rng is None else 2 * rows + ~((cf.start[cols] >= rng[0]) & (cf.stop[cols] <= rng[1]))
        order = np.argsort(key, kind="stable")
        sz = nr * nc
        off = np.empty(len(key), np.int64)
        off[order] = np.cumsum(sz[order]) - sz[order]
        out.append((rows, cols, nr, nc, off, order))
    return out


@pytest.mark.parametrize("level,basis,disc", [(4, "constant", "galerkin"), (3, "linear", "collocation")])
def test_device_block_tables_match_numpy(level, basis, disc):
    """gc_h2_blocks (csrc/h2blocks.cu): the coupling / near-field tables and
    storage offsets equal the numpy restatement, unsharded and for three
    block-row shards; the assembly descriptors point at the same pivots /
    clusters."""
    mesh = geometry.build_sphere_mesh(level)
    cfg = cli.default_config(eps=1e-6, basis=basis, disc=disc)
    hm, tree, bt = cli.build_h2_operator(mesh, cfg)
    rf = cf = tree.flat
    rs, cs = hm.row_basis.store, hm.col_basis.store
    dev = torch.device("cuda", 0)
    n = int(rf.stop[0])
    for rng in [None, (0, n // 4), (n // 4, n // 2), (n // 2, n)]:
        tabs = gca._device_block_tables(bt, rf, cf, rs, cs, rng, dev)
        got = tabs.host()
        exp = _expected_block_tables(bt, rf, cf, rs, cs, rng)
        for g, e in zip(got, exp):
            for a, b in zip(g, e):
                assert np.array_equal(a, b), rng
        (cr, cc, c_nr, c_nc, c_off, _), (nr_r, nc_r, n_nr, n_nc, n_off, _) = exp
        keep = (c_nr > 0) & (c_nc > 0)
        cd = tabs.c_desc.cpu().numpy()
        assert np.array_equal(cd, np.stack([rs.piv_off[cr], c_nr, cs.piv_off[cc], c_nc, c_off], 1)[keep])
        nd = tabs.n_desc.cpu().numpy()
        assert np.array_equal(nd, np.stack([rf.start[nr_r], n_nr, cf.start[nc_r], n_nc, n_off], 1))
        c_shape, n_shape = tabs.shapes
        assert c_shape[0] == int(keep.sum()) and c_shape[3] == int((c_nr * c_nc).sum())
        assert n_shape[0] == len(nr_r) and n_shape[3] == int((n_nr * n_nc).sum())
