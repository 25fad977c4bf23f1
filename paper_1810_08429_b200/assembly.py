"""Device-backed Galerkin assembly and Green factors behind the reference's seams.

Mirrors the hot-path entry points of ``greencross/assembly.py``:

* ``galerkin_pair_evaluator(kind, mesh, basis, q_reg, q_sing)`` returns an
  ``evaluate(case, rows, cols, px, py)`` with the executor contract of
  ``batchexec.py:70-76`` (values in canonical permuted order, shape (B,1,1),
  independent of batch composition), computed by ``gc_pair_eval``
  (``assembly.py:159-216``);
* ``assemble_galerkin_block`` - dense block on any index lists
  (``assembly.py:330-337``) through ``gc_assemble_blocks`` +
  ``gc_singular_flush``;
* ``green_row_factor`` / ``green_col_factor`` - the Green quadrature factor
  seam resolved by ``gca.build_cluster_basis`` (``assembly.py:420-455``)
  through ``gc_green_factor``.

Only the single-layer kernel with the piecewise-constant basis on plane
charts runs on the device (the configurations of BASELINE.json); other
kinds raise :class:`ConfigError`.  There is no host fallback.
"""

from collections import namedtuple

import numpy as np

from . import _native
from . import quadrature as quad
from .device import (DeviceMesh, DeviceRules, SingularQueue, check_mesh, empty, ptr,
                     require_device, stream_handle, to_dev, torch)
from .errors import ConfigError, GeometryError

FOUR_PI = 4.0 * np.pi
DenseBlock = namedtuple("DenseBlock", "rows cols values")
TriangleTable = namedtuple("TriangleTable", "rows")


def galerkin_classify(mesh):
    """Host twin of the device classifier (``assembly.py:150-156``)."""
    tris = mesh.triangles

    def classify(rows, cols):
        return quad.classify_pairs(tris[rows], tris[cols])

    return classify


def triangle_table(indices, mesh, basis="linear"):
    """Triangle table of vertex DOFs (``assembly.py:54-89``): rows
    (triangle, slot0, slot1, slot2) sorted by triangle."""
    if basis != "linear":
        raise ConfigError("triangle tables index vertex DOFs (linear basis)")
    from . import linear
    return TriangleTable(linear.triangle_table(indices, mesh))


def galerkin_pair_evaluator(kind, mesh, basis, q_reg, q_sing, device=None):
    """Batched device pair evaluator for the executor seam: values of shape
    (B, 1, 1) (constant basis) or (B, 3, 3) (linear basis, canonical permuted
    local order, ``batchexec.py:70-76``)."""
    if kind not in ("slp", "dlp"):
        raise ConfigError("unknown kernel kind %r" % (kind,))
    if basis not in ("constant", "linear"):
        raise ConfigError("unknown basis %r" % (basis,))
    check_mesh(mesh, kind, basis, linear_ok=True)
    dev = require_device(device)
    dmesh = DeviceMesh.get(mesh, q_reg, dev)
    if basis == "linear":
        from . import linear
        lrules = linear.LinearRules.get(q_reg, q_sing, dev)

        def evaluate_linear(case, rows, cols, px, py):
            if int(case) not in (0, 1, 2, 3):
                raise ConfigError("unknown pair case %r" % (case,))
            return linear.pair_values(dmesh, kind, lrules, rows, cols, dev)

        return evaluate_linear
    rules = DeviceRules.get(q_sing, dev, kind)
    geom = dmesh.geom_of(kind)
    if dmesh.curved:
        from . import linear
        return linear.curved_evaluator(dmesh, kind, q_reg, q_sing, 1, dev)

    def evaluate(case, rows, cols, px, py):
        case = int(case)
        if case not in (0, 1, 2, 3):
            raise ConfigError("unknown pair case %r" % (case,))
        b = len(rows)
        out = empty(b, dev)
        args = [to_dev(np.asarray(a, dtype=np.int64), dev) for a in (rows, cols, px, py)]
        with torch.cuda.device(dev):
            _native.call("gc_pair_eval", geom, rules.struct, case, b,
                         *[ptr(a) for a in args], ptr(out), stream_handle())
        return out.cpu().numpy().reshape(b, 1, 1)

    return evaluate


def device_block_assembly(dmesh, rules, queue, row_idx, col_idx, desc, out, stats=None, kind="slp",
                          d_desc=None, events=None, pending=None, shape=None):
    """Assemble blocks described by ``desc (nb,5)`` into the device buffer
    ``out`` (column-major per block); singular pairs are flushed at the end.
    ``kind`` "slp" / "dlp" picks the kernel (``rules`` must match it);
    ``d_desc`` is an already uploaded copy of ``desc``.  Returns the per-case
    task counts.  ``events``: a list that receives (start, after the block
    kernel, after the singular flush) CUDA events of this call.
    ``pending``: asynchronous mode (plane charts) - no host synchronisation;
    appends (device singular counts, total entries) to the list and returns
    None; the caller resolves the counts and checks the queue flags after
    its own synchronisation (:func:`resolve_counts`).  ``shape``: (blocks,
    max rows, max cols, entries) of a descriptor table that exists on the
    device only (``desc`` None)."""
    if getattr(rules, "kind", "slp") != kind:
        raise ConfigError("rules built for %r, assembling %r" % (rules.kind, kind))
    geom = dmesh.geom_of(kind)
    full = None
    if dmesh.curved:
        # curved charts: singular pairs take the full Sauter-Schwab rules
        from . import linear
        full = linear.LinearRules.get(dmesh.q_reg, rules.q_sing, out.device)
    if shape is not None:
        nb, max_rows, max_cols, total = (int(v) for v in shape[:4])
    else:
        nb = len(desc)
        if nb:
            max_rows, max_cols = int(desc[:, 1].max()), int(desc[:, 3].max())
            total = int((desc[:, 1] * desc[:, 3]).sum())
    if nb == 0:
        return [0, 0, 0, 0]
    if d_desc is None:
        d_desc = to_dev(desc.astype(np.int64), out.device)
    stream = stream_handle()
    with torch.cuda.device(out.device):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)] if events is not None else None
        if ev:
            ev[0].record()
        _native.call("gc_assemble_blocks", geom, nb, ptr(d_desc), max_rows, max_cols, ptr(row_idx),
                     ptr(col_idx), ptr(out), queue.struct, ptr(queue.flags), stream)
        if ev:
            ev[1].record()
        counts = (_native.c_i64 * 4)()
        if full is not None:
            _native.call("gc_curved_singular", geom, full.struct, queue.struct, 1, ptr(out), counts, stream)
        elif pending is not None:
            cdev = torch.zeros(4, dtype=torch.int32, device=out.device)
            _native.call("gc_singular_flush_async", geom, rules.struct, queue.struct, ptr(out), ptr(cdev),
                         stream)
        else:
            _native.call("gc_singular_flush", geom, rules.struct, queue.struct, ptr(out),
                         counts, stream)
        if ev:
            ev[2].record()
            events.append(ev)
    if pending is not None and full is None:
        pending.append((cdev, total))
        return None
    queue.check_flags()
    n_sing = [int(counts[k]) for k in range(4)]
    n_sing[0] = total - sum(n_sing[1:])
    return n_sing


def resolve_counts(pending, queue):
    """Per-case task counts of asynchronous device_block_assembly calls
    (after the caller's synchronisation); raises on a queue overflow."""
    queue.check_flags()
    out = []
    for cdev, total in pending:
        c = [int(v) for v in cdev.cpu().tolist()]
        out.append([total - sum(c[1:]), c[1], c[2], c[3]])
    return out


def assemble_galerkin_block(kind, mesh, basis, rows, cols, orders=(3, 5), capacity=None,
                            threads=None, device=None):
    """Dense Galerkin block G[rows, cols] (``assembly.py:330-337``); rows
    and columns are triangles (constant basis) or vertices (linear basis)."""
    check_mesh(mesh, kind, basis, linear_ok=True)
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    if len(np.unique(rows)) != len(rows) or len(np.unique(cols)) != len(cols):
        raise ConfigError("duplicate indices")
    nr, nc = len(rows), len(cols)
    if nr == 0 or nc == 0:
        return DenseBlock(rows, cols, np.zeros((nr, nc)))
    dev = require_device(device)
    dmesh = DeviceMesh.get(mesh, orders[0], dev)
    if basis == "linear":
        from . import linear
        out = empty(nr * nc, dev)
        linear.assemble_blocks(dmesh, kind, linear.LinearRules.get(orders[0], orders[1], dev), mesh,
                               [(rows, cols, 0)], out, dev)
        return DenseBlock(rows, cols, out.cpu().numpy().reshape(nc, nr).T.copy())
    rules = DeviceRules.get(orders[1], dev, kind)
    queue = SingularQueue.get(mesh, dev)
    out = empty(nr * nc, dev)
    desc = np.array([[0, nr, 0, nc, 0]], dtype=np.int64)
    device_block_assembly(dmesh, rules, queue, to_dev(rows, dev), to_dev(cols, dev), desc, out,
                          kind=kind)
    return DenseBlock(rows, cols, out.cpu().numpy().reshape(nc, nr).T.copy())


def collocation_classify(mesh):
    """``assembly.py:219-228``: rows are points (vertices), columns
    triangles; case 1 iff the point is a corner, py the rotation putting
    it first."""
    from . import linear
    return linear.collocation_classify(mesh)


def collocation_evaluator(kind, mesh, q_reg, q_sing, device=None):
    """Device single-integral evaluator (``assembly.py:231-276``): values
    (B, 1, 3) in the rotated column order."""
    if kind not in ("slp", "dlp"):
        raise ConfigError("unknown kernel kind %r" % (kind,))
    check_mesh(mesh, kind, "linear", linear_ok=True)
    from . import linear
    dev = require_device(device)
    dmesh = DeviceMesh.get(mesh, q_reg, dev)
    rules = linear.CollocationRules(q_reg, q_sing)

    def evaluate(case, rows, cols, px, py):
        if int(case) not in (0, 1):
            raise ConfigError("unknown collocation case %r" % (case,))
        return linear.collocation_values(dmesh, kind, rules, rows, cols, dev)

    return evaluate


def assemble_collocation_block(kind, mesh, basis, rows, cols, orders=(3, 5), capacity=None,
                               threads=None, device=None):
    """Collocation block g(x_i, .) phi_j (``assembly.py:352-362``): rows are
    surface points (vertex ids), columns linear-basis DOFs."""
    if basis != "linear":
        raise ConfigError("collocation rows pair with the linear basis")
    if kind not in ("slp", "dlp"):
        raise ConfigError("unknown kernel kind %r" % (kind,))
    check_mesh(mesh, kind, basis, linear_ok=True)
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    if len(np.unique(cols)) != len(cols):
        raise ConfigError("duplicate indices")
    nr, nc = len(rows), len(cols)
    if nr == 0 or nc == 0:
        return DenseBlock(rows, cols, np.zeros((nr, nc)))
    from . import linear
    dev = require_device(device)
    dmesh = DeviceMesh.get(mesh, orders[0], dev)
    out = empty(nr * nc, dev)
    linear.collocation_blocks(dmesh, kind, linear.CollocationRules(*orders), mesh, [(rows, cols, 0)], out, dev)
    return DenseBlock(rows, cols, out.cpu().numpy().reshape(nc, nr).T.copy())


# --------------------------------------------------------------------------
# Green factors

def green_factors_device(dmesh, side, K, rows, desc, dtau, z, sq, nz, total_rows, device,
                         check_flags=True, basis="constant"):
    """Factor matrices of a batch of nodes (device buffer, row-major per
    node); rows are triangles (constant basis) or vertices (linear basis).
    Raises GeometryError if an expansion point touches the surface."""
    out = empty(total_rows * 2 * K, device)
    flags = torch.zeros(1, dtype=torch.int32, device=device)
    with torch.cuda.device(device):
        _native.call("gc_green_factor", dmesh.geom_of("slp", basis), {"row": 0, "col": 1}.get(side, -1), K,
                     desc.numel() // 5,
                     ptr(desc), ptr(dtau), ptr(z), ptr(sq), ptr(nz), ptr(rows), ptr(out),
                     ptr(flags), stream_handle())
    if check_flags:
        touch_check(flags)
    return out, flags


def touch_check(flags):
    if int(flags.max().item()) & 1:
        raise GeometryError("expansion point touches the surface; "
                            "enlarge delta or the cluster box")


def _single_factor(side, cluster, rule, mesh, basis, orders, d_tau, device=None):
    check_mesh(mesh, "slp", basis, linear_ok=True)
    dev = require_device(device)
    dmesh = DeviceMesh.get(mesh, orders[0], dev)
    rows = np.asarray(cluster.indices, dtype=np.int64)
    K = int(rule.k)
    z = to_dev(np.asarray(rule.points, dtype=np.float64), dev)
    sq = to_dev(np.sqrt(np.asarray(rule.weights, dtype=np.float64)), dev)
    nz = to_dev(np.asarray(rule.normals, dtype=np.float64), dev)
    desc = to_dev(np.array([[0, len(rows), 0, 0, 0]], dtype=np.int64), dev)
    dtau = to_dev(np.array([d_tau]), dev)
    out, _ = green_factors_device(dmesh, side, K, to_dev(rows, dev), desc, dtau, z, sq, nz,
                                  len(rows), dev, basis=basis)
    return out.cpu().numpy().reshape(len(rows), 2 * K)


def green_row_factor(cluster, rule, mesh, basis, orders=(3, 5)):
    """Row factor A = [sqrt(w) g-moments, -d_tau sqrt(w) dg/dn-moments]
    (``assembly.py:420-439``); ``cluster`` needs ``.indices`` and ``.box``."""

    return _single_factor("row", cluster, rule, mesh, basis, orders, cluster.box.diameter())


def green_col_factor(pair, rule, mesh, basis, orders=(3, 5)):
    """Column factor B = [sqrt(w) dg/dn-moments, sqrt(w)/d_tau g-moments] of
    sigma under tau's rule (``assembly.py:442-455``)."""
    tau, sigma = pair
    if basis == "collocation":
        raise ConfigError("column factors integrate a Galerkin basis")
    return _single_factor("col", sigma, rule, mesh, basis, orders, tau.box.diameter())
