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
        cache["star_corner"] = (order % 3).astype(np.int64)
    return cache["star_csr"]


class _Tables:
    """Triangle tables (``triangle_table``) of many DOF lists at once, plus
    the CSR from every DOF to its (table row, corner) entries - vectorised
    over all blocks.  ``points=True``: the rows are collocation points, each
    its own one-entry "table" row."""

    def __init__(self, mesh, dof_lists, points=False):
        lens = np.array([len(d) for d in dof_lists], dtype=np.int64)
        nb = len(lens)
        D = np.concatenate(dof_lists).astype(np.int64) if nb else np.zeros(0, np.int64)
        self.dof_off = np.r_[0, np.cumsum(lens)]
        P = np.arange(len(D), dtype=np.int64) - np.repeat(self.dof_off[:-1], lens)
        if points:
            self.T = lens.copy()
            self.toff = self.dof_off[:-1].copy()
            self.tri = D                                    # the point itself
            self.ptr = np.arange(len(D) + 1, dtype=np.int64)
            self.ent = P << 2
            return
        sp, st = _star_csr(mesh)
        sc = mesh.__dict__["_device_cache"]["star_corner"]
        deg = sp[D + 1] - sp[D]
        idx = _ranges(sp[D], deg)
        eb = np.repeat(np.repeat(np.arange(nb, dtype=np.int64), lens), deg)
        ep = np.repeat(P, deg)
        et, ek = st[idx], sc[idx]
        key = eb * mesh.nt + et
        ukey, inv = np.unique(key, return_inverse=True)
        tb = ukey // mesh.nt
        self.T = np.bincount(tb, minlength=nb).astype(np.int64)
        self.toff = np.r_[0, np.cumsum(self.T)][:-1]
        self.tri = ukey % mesh.nt
        gdof = self.dof_off[eb] + ep                        # global DOF index of every entry
        order = np.lexsort((inv, gdof))
        self.ent = (((inv - self.toff[eb]) << 2) | ek)[order].astype(np.int64)
        self.ptr = np.r_[0, np.cumsum(np.bincount(gdof, minlength=len(D)))].astype(np.int64)


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
    return _assemble(dmesh, kind, mesh, blocks, out, device, rules=rules)


def _dedupe(lists, keys):
    """Index of every list into the distinct lists (by key when given)."""
    if any(k is None for k in keys):
        return np.arange(len(lists), dtype=np.int64), lists
    first, idx = {}, np.empty(len(keys), dtype=np.int64)
    for i, k in enumerate(keys):
        j = first.get(k)
        if j is None:
            j = first[k] = len(first)
        idx[i] = j
    uniq = [None] * len(first)
    for i, k in enumerate(keys):
        if uniq[idx[i]] is None:
            uniq[idx[i]] = lists[i]
    return idx, uniq


class _Select:
    """Per-block view of the distinct tables: dof offset, dof count, table
    size and offset of each block's list."""

    def __init__(self, t, idx):
        self.dof_off = t.dof_off[:-1][idx]
        self.n = np.diff(t.dof_off)[idx]
        self.T = t.T[idx]
        self.toff = t.toff[idx]


def _assemble(dmesh, kind, mesh, blocks, out, device, rules=None, crules=None):
    """Shared block driver: vectorised tables, batches of <= _MAX_TASKS
    triangle (or point x triangle) pairs derived on the device from block
    descriptors, pair kernels, singular flush, deterministic gather."""
    totals = [0, 0, 0, 0]
    if not blocks:
        return totals
    colloc = crules is not None
    # one table per distinct DOF list: blocks of one block row share the row
    # list (blocks may carry (rows, cols, off, row_key, col_key))
    ridx, rlists = _dedupe([b[0] for b in blocks], [b[3] if len(b) > 3 else None for b in blocks])
    cidx, clists = _dedupe([b[1] for b in blocks], [b[4] if len(b) > 4 else None for b in blocks])
    tr_u = _Tables(mesh, rlists, points=colloc)
    tc_u = _Tables(mesh, clists)
    tr, tc = _Select(tr_u, ridx), _Select(tc_u, cidx)
    nr = tr.n
    nc = tc.n
    offs = np.array([b[2] for b in blocks], dtype=np.int64)
    ntask = tr.T * tc.T
    d = [to_dev(a if len(a) else np.zeros(1, np.int64), device)
         for a in (tr_u.ptr, tr_u.ent, tc_u.ptr, tc_u.ent, tr_u.tri, tc_u.tri)]
    cum = np.cumsum(ntask)
    cap = int(min(int(cum[-1]), max(_MAX_TASKS, int(ntask.max()))))
    U = empty(9 * max(cap, 1), device)
    pp = torch.empty(max(cap, 1), dtype=torch.int32, device=device)
    q = None if colloc else _Queue(cap, device)
    nsing = torch.zeros(1, dtype=torch.int32, device=device)
    i = 0
    while i < len(blocks):
        # consecutive blocks up to _MAX_TASKS pairs per device batch
        start_cum = int(cum[i - 1]) if i else 0
        j = max(int(np.searchsorted(cum, start_cum + _MAX_TASKS, side="right")), i + 1)
        sel = np.arange(i, j)
        live = sel[ntask[sel] > 0]
        n = int(ntask[sel].sum())
        base = np.r_[0, np.cumsum(ntask[sel])][:-1]
        desc = np.stack([tr.dof_off[sel], nr[sel], tc.dof_off[sel], nc[sel], offs[sel], base, tc.T[sel]], 1)
        blk = np.stack([base[ntask[sel] > 0], tc.T[live], tr.toff[live], tc.toff[live]], 1)
        d_desc = to_dev(np.ascontiguousarray(desc, np.int64), device)
        with torch.cuda.device(device):
            st = stream_handle()
            if n:
                d_blk = to_dev(np.ascontiguousarray(blk, np.int64), device)
                if colloc:
                    _native.call("gc_col_pairs_blocks", dmesh.geom_of(kind), ptr(dmesh.verts),
                                 crules.w.ctypes.data, crules.b.ctypes.data, len(crules.sw),
                                 crules.sw.ctypes.data, crules.sp.ctypes.data, n, len(blk), ptr(d_blk),
                                 ptr(d[4]), ptr(d[5]), ptr(U), ptr(pp), ptr(nsing), st)
                else:
                    _native.call("gc_lin_pairs_blocks", dmesh.geom_of(kind), rules.w.ctypes.data,
                                 rules.b.ctypes.data, n, len(blk), ptr(d_blk), ptr(d[4]), ptr(d[5]), ptr(U),
                                 ptr(pp), q.struct, ptr(q.flags), st)
                    c = (_native.c_i64 * 4)()
                    _flush(dmesh, kind, rules, q, U, c, st)
                    q.check()
                    for k in (1, 2, 3):
                        totals[k] += int(c[k])
            _native.call("gc_lin_gather", len(desc), ptr(d_desc), ptr(d[0]), ptr(d[1]), ptr(d[2]), ptr(d[3]),
                         ptr(U), ptr(pp), ptr(out), st)
        totals[0] += n
        i = j
    if colloc:
        s_ = int(nsing.item())
        totals[0] -= s_
        totals[1] += s_
    else:
        totals[0] -= sum(totals[1:])
    return totals


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
    t = _assemble(dmesh, kind, mesh, blocks, out, device, crules=rules)
    return t[:2]
