"""Piecewise-linear basis on the device.

The linear basis has one DOF per vertex (hat functions).  A Galerkin block
over DOF lists (rows, cols) is the sum, over every pair of triangles in the
rows' and columns' vertex stars, of a 3x3 matrix of pair integrals scattered
onto the pair's vertices (``assembly.py:279-304``, ``batchexec.py:178-209``).

Device path (``csrc/linear.cu``):

1. ``gc_lin_pairs`` - one thread per triangle pair: classification, the
   regular q^2 x q^2 rule for disjoint pairs, singular pairs queued;
2. ``gc_lin_singular`` - the reference's full Sauter-Schwab rules;
3. ``gc_lin_gather`` - one thread per block entry sums the contributions of
   its (row triangle, column triangle) pairs in a fixed order.

The host builds the triangle tables (``triangle_table``, same semantics as
``assembly.py:54-89``) and, per block, the CSR lists mapping each DOF to its
(table row, local corner) pairs.
"""

import numpy as np

from . import _native
from .device import empty, ptr, stream_handle, to_dev, torch
from .errors import ConfigError
from .quadrature import sauter_rule, triangle_gauss

_MAX_TASKS = 1 << 21          # triangle pairs per device batch (U: 9 doubles each)


def _star_csr(mesh):
    cache = mesh.__dict__.setdefault("_device_cache", {})
    if "star_csr" not in cache:
        flat = mesh.triangles.ravel()
        order = np.argsort(flat, kind="stable")
        ptr_ = np.searchsorted(flat[order], np.arange(mesh.nv + 1))
        cache["star_csr"] = (ptr_.astype(np.int64), (order // 3).astype(np.int64))
    return cache["star_csr"]


def _ranges(starts, lengths):
    lengths = np.asarray(lengths, dtype=np.int64)
    total = int(lengths.sum())
    if total == 0:
        return np.zeros(0, dtype=np.int64)
    heads = np.cumsum(lengths) - lengths
    return np.arange(total, dtype=np.int64) + np.repeat(np.asarray(starts, np.int64) - heads, lengths)


def triangle_table(indices, mesh):
    """(T, 4) rows (triangle, slot0, slot1, slot2) sorted by triangle; slot p
    is the 1-based position of the triangle's vertex p in ``indices`` or 0
    (``assembly.py:54-89``)."""
    indices = np.asarray(indices, dtype=np.int64)
    if len(np.unique(indices)) != len(indices):
        raise ConfigError("duplicate indices in triangle_table")
    if len(indices) == 0:
        return np.zeros((0, 4), dtype=np.int64)
    sp, st = _star_csr(mesh)
    tri = np.unique(st[_ranges(sp[indices], sp[indices + 1] - sp[indices])])
    corners = mesh.triangles[tri]
    order = np.argsort(indices, kind="stable")
    sidx = indices[order]
    loc = np.minimum(np.searchsorted(sidx, corners), len(sidx) - 1)
    hit = sidx[loc] == corners
    slot = np.where(hit, order[loc] + 1, 0)
    return np.column_stack([tri, slot]).astype(np.int64)


def _dof_lists(table, ndof):
    """CSR over the DOFs of a triangle table: per DOF the packed
    (table_row << 2 | corner) entries, in table order."""
    p, k = np.nonzero(table[:, 1:] > 0)
    dof = table[p, 1 + k] - 1
    order = np.argsort(dof, kind="stable")
    ptr_ = np.zeros(ndof + 1, dtype=np.int64)
    np.cumsum(np.bincount(dof, minlength=ndof), out=ptr_[1:])
    return ptr_, ((p[order] << 2) | k[order]).astype(np.int64)


class LinearRules:
    """Regular rule (weights + barycentric values of its points) and the
    reference's full Sauter-Schwab rules as SoA tables (x1, x2, y1, y2, w)."""

    def __init__(self, q_reg, q_sing, device):
        pts, wts = triangle_gauss(q_reg)
        self.w = np.ascontiguousarray(wts, dtype=np.float64)
        self.b = np.ascontiguousarray(np.stack([1.0 - pts[:, 0] - pts[:, 1], pts[:, 0], pts[:, 1]], 1))
        self.tables = [None] * 4
        self.struct = _native.GcRules()
        for case in (1, 2, 3):
            r = sauter_rule(case, q_sing)
            t = to_dev(np.concatenate([r.x[:, 0], r.x[:, 1], r.y[:, 0], r.y[:, 1], r.w]), device)
            self.tables[case] = t
            self.struct.table[case] = t.data_ptr()
            self.struct.npts[case] = len(r.w)

    @classmethod
    def get(cls, q_reg, q_sing, device):
        key = (str(device), int(q_reg), int(q_sing))
        if key not in _CACHE:
            _CACHE[key] = cls(int(q_reg), int(q_sing), device)
        return _CACHE[key]


_CACHE = {}


class _Queue:
    """Singular-pair queues sized for one batch (a triangle pair recurs in
    many linear blocks, so the per-mesh bound of SingularQueue does not
    hold)."""

    def __init__(self, cap, device):
        self.count = torch.zeros(4, dtype=torch.int32, device=device)
        self.flags = torch.zeros(1, dtype=torch.int32, device=device)
        self.tasks = [torch.empty((max(cap, 1) if k else 1, 4), dtype=torch.int64, device=device)
                      for k in range(4)]
        self.struct = _native.GcQueue()
        for k in range(4):
            self.struct.tasks[k] = self.tasks[k].data_ptr()
            self.struct.cap[k] = cap if k else 0
        self.struct.count = self.count.data_ptr()

    def check(self):
        if int(self.flags.item()) & 2:
            raise ConfigError("linear-basis singular queue overflow")


def pair_values(dmesh, kind, rules, rows, cols, device):
    """3x3 pair integrals (canonical permuted local order) of the triangle
    pairs (rows[i], cols[i]) - the evaluator seam for the linear basis."""
    n = len(rows)
    tasks = to_dev(np.stack([np.asarray(rows, np.int64), np.asarray(cols, np.int64)], 1), device)
    U = empty(9 * n, device)
    pp = torch.empty(n, dtype=torch.int32, device=device)
    q = _Queue(n, device)
    with torch.cuda.device(device):
        st = stream_handle()
        _native.call("gc_lin_pairs", dmesh.geom_of(kind), rules.w.ctypes.data, rules.b.ctypes.data, n,
                     ptr(tasks), ptr(U), ptr(pp), q.struct, ptr(q.flags), st)
        counts = (_native.c_i64 * 4)()
        _flush(dmesh, kind, rules, q, U, counts, st)
    q.check()
    return U.cpu().numpy().reshape(n, 3, 3)


def _flush(dmesh, kind, rules, q, U, counts, st):
    """Singular pairs of a batch: affine charts with the full rules
    (gc_lin_singular), curved charts evaluated point by point
    (gc_curved_singular)."""
    if dmesh.curved:
        _native.call("gc_curved_singular", dmesh.geom_of(kind), rules.struct, q.struct, 9, ptr(U), counts, st)
    else:
        _native.call("gc_lin_singular", dmesh.geom_of(kind), rules.struct, q.struct, ptr(U), counts, st)


def curved_evaluator(dmesh, kind, q_reg, q_sing, width, device):
    """Evaluator seam on curved charts: every case (the disjoint tensor rule
    included) through gc_curved_pairs; values (B,1,1) or (B,3,3)."""
    lr = LinearRules.get(q_reg, q_sing, device)
    pts, wts = triangle_gauss(q_reg)
    m = len(wts)
    x, y = np.repeat(pts, m, axis=0), np.tile(pts, (m, 1))
    reg = to_dev(np.concatenate([x[:, 0], x[:, 1], y[:, 0], y[:, 1], np.outer(wts, wts).ravel()]), device)

    def evaluate(case, rows, cols, px, py):
        case = int(case)
        if case not in (0, 1, 2, 3):
            raise ConfigError("unknown pair case %r" % (case,))
        n = len(rows)
        pk = np.asarray(px, np.int64) | (np.asarray(py, np.int64) << 8)
        tasks = to_dev(np.stack([np.asarray(rows, np.int64), np.asarray(cols, np.int64), pk,
                                 np.arange(n, dtype=np.int64)], 1), device)
        table, P = (reg, m * m) if case == 0 else (lr.tables[case], int(lr.struct.npts[case]))
        out = empty(width * max(n, 1), device)
        with torch.cuda.device(device):
            _native.call("gc_curved_pairs", dmesh.geom_of(kind), ptr(table), P, ptr(tasks), n, width, ptr(out),
                         stream_handle())
        return out[:width * n].cpu().numpy().reshape(n, 1 if width == 1 else 3, 1 if width == 1 else 3)

    return evaluate


def assemble_blocks(dmesh, kind, rules, mesh, blocks, out, device):
    """Linear-basis Galerkin blocks: ``blocks`` = list of (rows, cols,
    out_off) with vertex DOF lists; each block lands column-major in the
    device vector ``out`` at ``out_off``.  Returns per-case task counts."""
    totals = [0, 0, 0, 0]
    i = 0
    while i < len(blocks):
        # one device batch: consecutive blocks up to _MAX_TASKS pairs
        batch, ntask = [], 0
        while i < len(blocks):
            rows, cols, off = blocks[i]
            tr, tc = triangle_table(rows, mesh), triangle_table(cols, mesh)
            n = len(tr) * len(tc)
            if batch and ntask + n > _MAX_TASKS:
                break
            batch.append((rows, cols, off, tr, tc))
            ntask += n
            i += 1
        _run_batch(dmesh, kind, rules, batch, ntask, out, device, totals)
    return totals


def _run_batch(dmesh, kind, rules, batch, ntask, out, device, totals):
    tasks = np.empty((ntask, 2), dtype=np.int64)
    desc = np.empty((len(batch), 7), dtype=np.int64)
    rp, rl, cp, cl = [], [], [], []
    base = ro = co = 0
    for b, (rows, cols, off, tr, tc) in enumerate(batch):
        nr, nc, T, C = len(rows), len(cols), len(tr), len(tc)
        tasks[base:base + T * C, 0] = np.repeat(tr[:, 0], C)
        tasks[base:base + T * C, 1] = np.tile(tc[:, 0], T)
        p1, l1 = _dof_lists(tr, nr)
        p2, l2 = _dof_lists(tc, nc)
        desc[b] = (ro, nr, co, nc, off, base, C)
        rp.append(p1[:-1] + sum(len(x) for x in rl))
        rl.append(l1)
        cp.append(p2[:-1] + sum(len(x) for x in cl))
        cl.append(l2)
        ro += nr
        co += nc
        base += T * C
    rptr = np.concatenate(rp + [np.array([sum(len(x) for x in rl)], np.int64)])
    cptr = np.concatenate(cp + [np.array([sum(len(x) for x in cl)], np.int64)])
    rlist = np.concatenate(rl) if rl else np.zeros(1, np.int64)
    clist = np.concatenate(cl) if cl else np.zeros(1, np.int64)
    d_tasks = to_dev(tasks, device)
    U = empty(9 * max(ntask, 1), device)
    pp = torch.empty(max(ntask, 1), dtype=torch.int32, device=device)
    q = _Queue(ntask, device)
    d = [to_dev(a, device) for a in (desc, rptr, np.maximum(rlist, 0), cptr, np.maximum(clist, 0))]
    with torch.cuda.device(device):
        st = stream_handle()
        _native.call("gc_lin_pairs", dmesh.geom_of(kind), rules.w.ctypes.data, rules.b.ctypes.data, ntask,
                     ptr(d_tasks), ptr(U), ptr(pp), q.struct, ptr(q.flags), st)
        counts = (_native.c_i64 * 4)()
        _flush(dmesh, kind, rules, q, U, counts, st)
        _native.call("gc_lin_gather", len(batch), ptr(d[0]), ptr(d[1]), ptr(d[2]), ptr(d[3]), ptr(d[4]),
                     ptr(U), ptr(pp), ptr(out), st)
    q.check()
    sing = [int(counts[k]) for k in range(4)]
    sing[0] = ntask - sum(sing[1:])
    for k in range(4):
        totals[k] += sing[k]


# --------------------------------------------------------------------------
# collocation (assembly.py:219-276, 340-362): rows are surface points (the
# mesh vertices), columns the linear basis

class CollocationRules:
    """The regular rule of the chart points (weights, barycentrics) and the
    collapsed Gauss rule used when the point is a corner of the triangle
    (``quadrature.duffy_rule(0, q_sing)``)."""

    def __init__(self, q_reg, q_sing):
        pts, wts = triangle_gauss(q_reg)
        self.w = np.ascontiguousarray(wts, dtype=np.float64)
        self.b = np.ascontiguousarray(np.stack([1.0 - pts[:, 0] - pts[:, 1], pts[:, 0], pts[:, 1]], 1))
        sp, sw = triangle_gauss(q_sing)
        self.sw = np.ascontiguousarray(sw, dtype=np.float64)
        self.sp = np.ascontiguousarray(sp, dtype=np.float64)


def collocation_classify(mesh):
    """``assembly.py:219-228``: case 1 iff the point is a corner of the
    triangle, py = the rotation putting that corner first."""
    tris = mesh.triangles

    def classify(rows, cols):
        hit = tris[cols] == np.asarray(rows)[:, None]
        return hit.any(axis=1).astype(np.int64), np.zeros(len(rows), dtype=np.int64), np.argmax(hit, axis=1)

    return classify


def _col_call(dmesh, kind, rules, tasks_dev, n, U, pp, device):
    with torch.cuda.device(device):
        _native.call("gc_col_pairs", dmesh.geom_of(kind), ptr(dmesh.verts), rules.w.ctypes.data,
                     rules.b.ctypes.data, len(rules.sw), rules.sw.ctypes.data, rules.sp.ctypes.data, n,
                     ptr(tasks_dev), ptr(U), ptr(pp), stream_handle())


def collocation_values(dmesh, kind, rules, rows, cols, device):
    """(B, 1, 3) single integrals of the (point, triangle) tasks in the
    rotated column order - the collocation evaluator seam."""
    n = len(rows)
    tasks = to_dev(np.stack([np.asarray(rows, np.int64), np.asarray(cols, np.int64)], 1), device)
    U = empty(9 * max(n, 1), device)
    pp = torch.empty(max(n, 1), dtype=torch.int32, device=device)
    _col_call(dmesh, kind, rules, tasks, n, U, pp, device)
    return U.view(-1, 9)[:n, :3].cpu().numpy().reshape(n, 1, 3)


def collocation_blocks(dmesh, kind, rules, mesh, blocks, out, device):
    """Collocation blocks: ``blocks`` = (row points, column DOFs, out_off);
    column-major per block in ``out``.  Returns [regular, singular] task
    counts."""
    totals = [0, 0]
    i = 0
    while i < len(blocks):
        batch, ntask = [], 0
        while i < len(blocks):
            rows, cols, off = blocks[i]
            tc = triangle_table(cols, mesh)
            n = len(rows) * len(tc)
            if batch and ntask + n > _MAX_TASKS:
                break
            batch.append((np.asarray(rows, np.int64), cols, off, tc))
            ntask += n
            i += 1
        tasks = np.empty((ntask, 2), dtype=np.int64)
        desc = np.empty((len(batch), 7), dtype=np.int64)
        rp, rl, cp, cl = [], [], [], []
        base = ro = co = nrl = ncl = 0
        for b, (rows, cols, off, tc) in enumerate(batch):
            nr, nc, C = len(rows), len(cols), len(tc)
            tasks[base:base + nr * C, 0] = np.repeat(rows, C)
            tasks[base:base + nr * C, 1] = np.tile(tc[:, 0], nr)
            rp.append(np.arange(nr, dtype=np.int64) + nrl)
            rl.append(np.arange(nr, dtype=np.int64) << 2)           # row i: (task row i, corner 0)
            p2, l2 = _dof_lists(tc, nc)
            cp.append(p2[:-1] + ncl)
            cl.append(l2)
            desc[b] = (ro, nr, co, nc, off, base, C)
            nrl += nr
            ncl += len(l2)
            ro += nr
            co += nc
            base += nr * C
        rptr = np.concatenate(rp + [np.array([nrl], np.int64)])
        cptr = np.concatenate(cp + [np.array([ncl], np.int64)])
        d = [to_dev(a, device) for a in (desc, rptr, np.concatenate(rl), cptr,
                                          np.concatenate(cl) if ncl else np.zeros(1, np.int64))]
        d_tasks = to_dev(tasks, device)
        U = empty(9 * max(ntask, 1), device)
        pp = torch.empty(max(ntask, 1), dtype=torch.int32, device=device)
        _col_call(dmesh, kind, rules, d_tasks, ntask, U, pp, device)
        with torch.cuda.device(device):
            _native.call("gc_lin_gather", len(batch), ptr(d[0]), ptr(d[1]), ptr(d[2]), ptr(d[3]), ptr(d[4]),
                         ptr(U), ptr(pp), ptr(out), stream_handle())
        sing = int((mesh.triangles[tasks[:, 1]] == tasks[:, :1]).any(axis=1).sum()) if ntask else 0
        totals[0] += ntask - sing
        totals[1] += sing
    return totals
