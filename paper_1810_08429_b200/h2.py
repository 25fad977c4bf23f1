"""H2 matrix-vector products on the device, storage accounting, solvers.

Mirror of ``greencross/h2.py``.  ``mvm`` / ``mvm_t`` (``h2.py:63-100``) keep
the reference's signature (host vectors in external ordering).  A product
is one replay of a CUDA graph built once per matrix and direction
(:class:`PanelPlan`): the external -> tree gather, the forward transform
(tiers of composed transfers, ``tiers.py``), the coupling panels bucketed by
row-cluster height on their own streams, the backward transform, the leaf
rows and the near field, all ``k_panelmv`` launches over contiguous
row-major panels (``csrc/h2mv.cu``), then the tree -> external scatter.
``mvm_t`` runs the same plan on the transposed operator (:func:`transposed`:
bases and trees swapped, blocks transposed once on the device).

``storage_report`` (``h2.py:110-134``) counts the same bytes the reference
does.  ``spectral_error_estimate``, ``cg_solve`` and ``cgnr_solve``
(``h2.py:144-253``) keep every vector and scalar in device memory
(``csrc/krylov.cu``); an operator from :func:`as_operator` applies its plans
to device vectors directly, any other closure is called on host copies.
"""

import threading
from collections import namedtuple

import numpy as np

from . import _native
from .device import ptr, stream_handle, to_dev, torch
from .errors import ConfigError, StateError

__all__ = ["mvm", "mvm_t", "as_operator", "storage_report", "storage_csv_rows",
           "spectral_error_estimate", "cg_solve", "cgnr_solve", "CGResult", "PanelPlan",
           "plan", "transposed", "mvm_device"]

_LOCKS_GUARD = threading.Lock()


def _plan_lock(d):
    with _LOCKS_GUARD:
        lk = getattr(d, "_plan_lock", None)
        if lk is None:
            lk = d._plan_lock = threading.Lock()
        return lk


def plan(h, trans=False):
    """Cached, captured product plan of ``h`` (``trans``: of its transpose),
    built on the operator's device."""
    d = h.dev
    key = "T" if trans else "N"
    with _plan_lock(d):
        if key not in d.plans:
            with torch.cuda.device(d.device):
                p = PanelPlan(transposed(h) if trans else h)
                p.capture()
            d.plans[key] = p
    return d.plans[key]


def _storage_order(d, kind, blocks):
    """``blocks`` (coupling "c" / near-field "n" block indices) in storage
    order - rows contiguous, as build_h2 laid the blocks out."""
    order = getattr(d, kind + "_order", None)
    if order is None:
        return blocks[np.argsort(getattr(d, kind + "_off")[blocks], kind="stable")]
    keep = np.zeros(len(order), bool)
    keep[blocks] = True
    return order[keep[order]]


def _check_dim(x, n):
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (n,):
        raise ConfigError("vector of length %d, operator wants %d" % (x.size, n))
    return x


def mvm_device(h, x_dev, y_dev=None, trans=False):
    """y = H x (H^T x) for float64 device vectors in external order, ordered
    on the current stream."""
    p = plan(h, trans)
    if y_dev is None:
        y_dev = torch.empty(p.n_out, dtype=torch.float64, device=p.dev)
    with torch.cuda.device(p.dev):
        p.run(x_dev, y_dev)
    return y_dev


def mvm(h, x):
    """y = H x, external ordering in and out (``h2.py:63-80``): the host
    vector is staged in pinned memory that the graph's gather kernel reads
    over the host link; the scatter kernel writes a pinned result."""
    nr, nc = h.shape
    return plan(h).apply_host(_check_dim(x, nc))


def mvm_t(h, x):
    """y = H^T x (``h2.py:83-100``), the same plan form on the transposed
    operator."""
    nr, nc = h.shape
    return plan(h, True).apply_host(_check_dim(x, nr))


class H2Operator:
    """``as_operator(h)`` (``h2.py:103-107``): callable ``apply(x, trans=False)``
    on host vectors; the device solvers recognise it and apply the plans to
    device vectors without host copies."""

    def __init__(self, h):
        self.h = h

    def __call__(self, x, trans=False):
        return mvm_t(self.h, x) if trans else mvm(self.h, x)

    def apply_device(self, x_dev, y_dev, trans=False):
        mvm_device(self.h, x_dev, y_dev, trans)


def as_operator(h):
    return H2Operator(h)


# --------------------------------------------------------------------------
# storage accounting

def storage_report(h):
    """Bytes per category at 8 bytes per real (``h2.py:110-134``)."""
    if isinstance(h, (int, np.integer)):
        n = int(h)
        return {"dense": 8 * n * n, "total": 8 * n * n}
    leaf_bases = transfers = index_bytes = 0
    for basis in (h.row_basis, h.col_basis):
        s = basis.store
        mat = s.materialized
        flat = s.tree.flat
        index_bytes += 8 * int(s.rank[mat].sum())
        leaf = mat & flat.is_leaf
        leaf_bases += 8 * int((s.rows[leaf] * s.rank[leaf]).sum())
        par = np.maximum(flat.parent, 0)
        nonroot = mat & (flat.parent >= 0) & mat[par]
        transfers += 8 * int((s.rank[nonroot] * s.rank[par[nonroot]]).sum())
    d = h.dev
    couplings = 8 * int((d.c_nr * d.c_nc).sum())
    nearfield = 8 * int((d.n_nr * d.n_nc).sum())
    nr, nc = h.shape
    return {"leaf_bases": leaf_bases, "transfers": transfers, "couplings": couplings,
            "nearfield": nearfield, "total": leaf_bases + transfers + couplings + nearfield,
            "index_bytes": index_bytes, "dense": 8 * nr * nc}


def storage_csv_rows(report):
    keys = ("leaf_bases", "transfers", "couplings", "nearfield", "total", "index_bytes", "dense")
    return [(k, report[k]) for k in keys if k in report]


# --------------------------------------------------------------------------
# transposed operator (mvm_t)

class _TransposedH2:
    """H^T as an H2 matrix for the flow plan: trees and bases swapped, every
    coupling / near-field block transposed and regrouped by its new row
    cluster (one gc_block_transpose over each store, built on first use)."""

    def __init__(self, h):
        from .gca import DeviceH2, _grouped_offsets
        if hasattr(h, "settle"):
            h.settle()
        d = h.dev
        dev = d.device
        if d.row_range is not None:
            raise ConfigError("mvm_t of a block-row shard: use the full operator")
        self.row_tree, self.col_tree = h.col_tree, h.row_tree
        self.row_basis, self.col_basis = h.col_basis, h.row_basis
        self.shape = (h.shape[1], h.shape[0])
        t = DeviceH2(dev)
        t.row_range = None
        t.perm_r, t.perm_c = d.perm_c, d.perm_r

        def regroup(rows, cols, nr, nc, off, src):
            # new block b = old block transposed: (nc x nr) stored as the
            # transpose of the new (nr' = nc) x (nc' = nr) block -> nr x nc
            new_off = _grouped_offsets(cols, nr * nc)
            dst = torch.empty(max(int((nr * nc).sum()), 1) + 4, dtype=torch.float64, device=dev)
            live = (nr * nc) > 0
            if live.any():
                # stored old block: nc x nr row-major at off; new: nr x nc row-major
                desc = np.stack([off, nr, nc, nr, new_off], 1)[live]
                _native.call("gc_block_transpose", int(live.sum()), ptr(to_dev(desc, dev)), ptr(src),
                             ptr(dst), _stream_ptr())
            return dst[:max(int((nr * nc).sum()), 1)], new_off

        with torch.cuda.device(dev):
            t.coup, t.c_off = regroup(d.c_rows, d.c_cols, d.c_nr, d.c_nc, d.c_off, d.coup)
            t.near, t.n_off = regroup(d.n_rows, d.n_cols, d.n_nr, d.n_nc, d.n_off, d.near)
        t.c_rows, t.c_cols, t.c_nr, t.c_nc = d.c_cols, d.c_rows, d.c_nc, d.c_nr
        t.n_rows, t.n_cols, t.n_nr, t.n_nc = d.n_cols, d.n_rows, d.n_nc, d.n_nr
        self.dev = t


def transposed(h):
    return _TransposedH2(h)


def _stream_ptr(stream=None):
    import ctypes
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


# --------------------------------------------------------------------------
# panel plan: the non-transposed product (the benchmarked hot path)

_ITEM_ELEMS = 65536          # <= 512 KB of matrix data per bulk work item (rows capped at 1024)
_ITEM_MAX_ROWS = 1024        # PAN_MAX_ROWS in csrc/h2mv.cu
_BULK_ITEMS_PER_SM = 1       # bulk items per SM per phase (4 -> 1: C2 product -3 %, sweeps/r02_bulk_items_per_sm.txt)
_PAIR_MAX_ELEMS = 12288      # k_panel_pair (two small panels per CTA): panel size cap (8192 -> 12288: cube L7 -4.6 %, L8 -1.4 %; sweeps/r02_pair_max_elems.txt)
_RING_MIN_BYTES = 16 << 30   # bulk phases this large stream through k_panel_ring (with one bulk item per SM: L7 -2.3 %, L8 -0.8 % without it, L9 +0.6 %; sweeps/r02_ring_threshold.txt)
_PAIR_BULK_MAX_BYTES = 32 << 20    # small operators: bulk phases paired like the tier phases
_SMALL_OPERATOR_BYTES = 128 << 20
_MERGE_MIN_BYTES = 1 << 30   # coupling row heights with the same producer / consumer merge into one launch


class _Phase:
    __slots__ = ("name", "height", "items", "xidx", "red", "arrivals", "nitems", "nred", "A0", "A1",
                 "in0", "in1", "out", "scratch", "bytes", "in_elems", "out_elems", "pair", "ring", "acc",
                 "_h_items", "_h_xidx", "_h_red", "_n_arrivals", "_n_scratch")   # staged tables (_flush_tables)


class _Node:
    """One step of the product DAG: a panel phase or a callable (gather,
    zero, scatter, a collective), run on ``stream`` after ``deps``;
    ``native`` = (kind, args) of the same step for the C++ executor
    (csrc/plan.cu node kinds 1-4)."""
    __slots__ = ("name", "phase", "fn", "stream", "deps", "launches", "priority", "native")

    def __init__(self, name, stream, deps=(), phase=None, fn=None, priority=0, native=None, launches=None):
        self.name, self.stream, self.deps, self.phase, self.fn = name, stream, list(deps), phase, fn
        self.launches = (1 if phase is not None else 0) if launches is None else launches
        self.priority = priority
        self.native = native


class PanelPlan:
    """mvm as a DAG of ``gc_panelmv`` phases over contiguous panels.

    The four phases of h2.py:63-80 are cut by tree height: forward levels
    (bottom-up) and backward levels (top-down) form the latency-bound
    "chain" on a high-priority stream (programmatic dependent launches: a
    level's prologue overlaps its predecessor's drain); the coupling panels
    are bucketed by the height of their row cluster and each bucket runs on
    its own stream as soon as the forward transform has produced every
    x-hat it reads, so the bandwidth-bound bulk (deep buckets, near field)
    streams from HBM while the chain climbs the tree.  A backward level
    waits only for the buckets that write the y-hat entries it reads or adds
    into.  Coupling overwrites y-hat before any backward contribution is
    added, so the summation order - and the result, bit for bit - does not
    depend on the schedule.  ``capture()`` records the DAG into one CUDA
    graph with static input/output buffers; ``run(..., phase_events=...)``
    executes it serially on the current stream (for per-phase timing).
    """

    def __init__(self, h, tiers="auto", xt_map=None, xt_len=None, bulk="auto", col_local=None):
        import time
        t0 = time.perf_counter()
        self.timing = {}
        self._bulk = bulk
        # a small operator (<= _SMALL_OPERATOR_BYTES of blocks) is latency-
        # bound throughout: its bulk phases of <= _PAIR_BULK_MAX_BYTES run one
        # item per panel, two panels per CTA.  Measured (profiles/sweeps/
        # r02_pair_bulk*.txt): sphere L4 eps 1e-4 (18 MB) 23.5 -> 18.6 us,
        # L5 eps 1e-4 (80 MB) 48 -> 37 us; L5 eps 1e-6 (166 MB) 52 -> 66 us,
        # neutral to slower from L6 on - hence the operator bound
        blocks = 8 * (h.dev.coup.numel() + h.dev.near.numel())
        self._pair_bulk = _PAIR_BULK_MAX_BYTES if blocks <= _SMALL_OPERATOR_BYTES else 0
        d = h.dev
        dev = d.device
        self.dev = dev
        self.lock = threading.Lock()
        self._dev_index = torch.device(dev).index
        if self._dev_index is None:
            self._dev_index = torch.cuda.current_device()
        self._pin_x_np = None
        # x_t positions of the tree-ordered input (a shard: its padded
        # all-gather layout, parallel.ShardPlan)
        self._xmap = None if xt_map is None else np.asarray(xt_map, np.int64)
        rs, cs = h.row_basis.store, h.col_basis.store
        rf, cf = h.row_tree.flat, h.col_tree.flat
        self.n_in, self.n_out = cf.stop[0], rf.stop[0]
        self.perm_in, self.perm_out = d.perm_c, d.perm_r
        self.iperm_in, self.iperm_out = _inverse_perm(self.perm_in), _inverse_perm(self.perm_out)
        f64 = dict(dtype=torch.float64, device=dev)
        self.x = torch.zeros(self.n_in, **f64)
        self.y = torch.zeros(self.n_out, **f64)
        self.xt = torch.zeros(self.n_in if xt_len is None else xt_len, **f64)
        # y (tree order, near-field part) | x-hat
        self._obuf = torch.zeros(self.n_out + max(cs.coef_size, 1), **f64)
        self.yt, self.xhat = self._obuf[:self.n_out], self._obuf[self.n_out:]
        self._keep = []
        self._t64, self._t32, self._staged = [], [], []      # tables of the phases (_flush_tables)
        self.tiers_pending = False
        ny = max(rs.coef_size, 1)
        # y-hat | y-hat from the tiers above | leaf-basis part of y (summed
        # in the scatter): one buffer, zeroed by one memset per product
        self._ybuf = torch.zeros(2 * ny + self.n_out, **f64)
        self.yhat, self.yhat_t, self.yt2 = self._ybuf[:ny], self._ybuf[ny:2 * ny], self._ybuf[2 * ny:]
        # col_local = (lo, hi): a shard (parallel.ShardPlan) whose own columns
        # are the tree positions [lo, hi) - blocks with local columns run
        # before the x / x-hat all-gathers, the others after them, adding
        # onto the same outputs
        self._col_local = col_local
        nloc = (np.ones(len(d.n_cols), bool) if col_local is None else
                (cf.start[d.n_cols] >= col_local[0]) & (cf.stop[d.n_cols] <= col_local[1]))
        # near field: one panel per row leaf
        near = self._near_phase(h, np.flatnonzero(nloc), 0)
        self._near_remote = None
        if col_local is not None and not nloc.all():
            has_local = np.zeros(len(rf.start), bool)
            has_local[d.n_rows[nloc]] = True
            self._near_remote = self._near_phase(h, np.flatnonzero(~nloc), has_local, ordered=True)
        self.tiers = None
        t1 = time.perf_counter()
        tiered = self._tiered(h, tiers) if tiers != "off" else None
        if tiered is None:
            fwd, bwd, leafp = self._level_phases(h)
            parts = [(leafp, None)]
        else:
            fwd, bwd, parts = tiered
        parts = [(P, hs) for P, hs in parts if P is not None and P.nitems]
        t1b = time.perf_counter()
        cloc = (np.ones(len(d.c_cols), bool) if col_local is None else
                (cf.start[d.c_cols] >= col_local[0]) & (cf.stop[d.c_cols] <= col_local[1]))
        cpl = self._coupling_phases(h, fwd, bwd, cloc, 0)
        self._cpl_remote = []
        if col_local is not None and not cloc.all():
            has_local = np.zeros(len(rf.start), bool)
            has_local[d.c_rows[cloc & (d.c_nr > 0) & (d.c_nc > 0)]] = True
            self._cpl_remote = self._coupling_phases(h, fwd, bwd, ~cloc, has_local, ordered=True)
        self._fwd, self._cpl, self._bwd, self._near, self._leafparts = fwd, cpl, bwd, near, parts
        self.phases = [P for P in [near, self._near_remote] + fwd + [c for c, _, _ in cpl + self._cpl_remote]
                       + [b for b, _ in bwd] + [p for p, _ in parts] if P is not None and P.nitems > 0]
        self._flush_tables()
        # the chain gets the highest stream priority so its CTAs are
        # scheduled ahead of the queued bulk (coupling buckets, near field)
        self.streams = {"chain": torch.cuda.Stream(device=dev, priority=-8)}
        self._bulk_priority = 0
        least, greatest = _native.ctypes.c_int32(0), _native.ctypes.c_int32(0)
        _native.call("gc_priority_range", _native.ctypes.byref(least), _native.ctypes.byref(greatest))
        self._prio = (least.value, greatest.value)
        self.trace = {}                    # id(phase) -> [2] int64 (profiling only)
        self.nodes = self._build_nodes()
        self.graph = None
        t2 = time.perf_counter()
        # the device assembly ran under this host work; its queue flags and
        # statistics settle now (an error surfaces before the plan is used)
        if hasattr(h, "settle"):
            h.settle()
        t3 = time.perf_counter()
        self.timing.update(near_phase_s=t1 - t0, transforms_s=t1b - t1, coupling_phases_s=t2 - t1b,
                           settle_s=t3 - t2)

    def _near_phase(self, h, blocks, acc_rows, ordered=False):
        """Near-field phase over the near blocks ``blocks``: one panel per
        row leaf; ``acc_rows`` (scalar or per row cluster) marks the rows
        whose panel adds onto y_t (written by an earlier near phase)."""
        d = h.dev
        rf, cf = h.row_tree.flat, h.col_tree.flat
        order = _storage_order(d, "n", blocks)                # rows contiguous
        sn = d.n_rows[order]
        cuts = np.flatnonzero(np.r_[True, sn[1:] != sn[:-1]]) if len(sn) else np.zeros(0, np.int64)
        K = np.add.reduceat(d.n_nc[order], cuts) if len(sn) else np.zeros(0, np.int64)
        rows = (self._xpos(cf.start[d.n_cols[order]]), d.n_nc[order])
        acc = np.asarray(acc_rows)[sn[cuts]].astype(np.int64) if np.ndim(acc_rows) else acc_rows
        panels = (d.n_off[order[cuts]], K, d.n_nr[order[cuts]], rows, rf.start[sn[cuts]], acc)
        return self._phase("nearfield", 0, panels, d.near, None, self.xt, None, self.yt, ordered=ordered)

    def _coupling_phases(self, h, fwd, bwd, mask, acc_rows, ordered=False):
        """Coupling phases over the blocks ``mask`` selects: one panel per
        row cluster.  Row clusters are grouped by (the forward phase
        producing every x-hat they read, the backward phase consuming their
        y-hat): one launch per group - e.g. all the deep buckets that only
        the leaf rows read - so a launch is as long as the dependencies
        allow.  ``acc_rows`` (scalar or per row cluster): panels that add
        onto y-hat written by an earlier coupling phase."""
        d = h.dev
        rs, cs = h.row_basis.store, h.col_basis.store
        rf, cf = h.row_tree.flat, h.col_tree.flat
        cpl = []
        live = mask & (d.c_nr > 0) & (d.c_nc > 0)
        order = _storage_order(d, "c", np.flatnonzero(live))
        if not order.size:
            return cpl
        sn = d.c_rows[order]
        cuts = np.flatnonzero(np.r_[True, sn[1:] != sn[:-1]])
        # panel inputs: the x-hat slots of the blocks' column clusters, in
        # block order - one index range per block, expanded on the device
        bstart, blen = cs.coef_off[d.c_cols[order]], d.c_nc[order]
        K = np.add.reduceat(blen, cuts)
        nblk = np.diff(np.r_[cuts, len(order)])
        colh = np.maximum.reduceat(cf.height[d.c_cols[order]], cuts)
        rowh = rf.height[sn[cuts]]
        acc = (np.asarray(acc_rows)[sn[cuts]].astype(np.int64) if np.ndim(acc_rows)
               else np.full(len(cuts), int(acc_rows), np.int64))
        # src: the first forward phase (ascending heights) covering the
        # panel's highest column cluster; dst: the first backward phase
        # (top down) whose heights include the row cluster's
        fwd_h = np.array([P.height for P in fwd if P.nitems], np.int64)
        src = np.searchsorted(fwd_h, colh, side="left")
        tab = np.full(int(rowh.max()) + 1, len(bwd), np.int64)
        for k in reversed(range(len(bwd))):
            P, hs = bwd[k]
            if P.nitems:
                hh = np.array([v for v in hs if 0 <= v < len(tab)], np.int64)
                tab[hh] = k
        dst = tab[rowh]
        # merge only into launches of >= _MERGE_MIN_BYTES: smaller groups stay
        # one launch per row height (measured: C4 -1.5 %, C2 +10 % merged)
        pair_key = src * (len(bwd) + 1) + dst
        gbytes = np.bincount(pair_key, weights=8.0 * (K * d.c_nr[order[cuts]]))
        grp = np.stack([src, dst, np.where(gbytes[pair_key] >= _MERGE_MIN_BYTES, -1, rowh)], 1).astype(np.int64)
        # one int64 code per group, groups in (consumer top down, producer,
        # height) order; members by a stable sort of the codes
        hcol = grp[:, 2] + 1                                   # -1 (merged) -> 0
        code = (len(bwd) - grp[:, 1]) * (len(fwd) + 2) * (int(hcol.max()) + 1) + grp[:, 0] * (int(hcol.max()) + 1) + hcol
        codes, inv = np.unique(code, return_inverse=True)
        members = np.argsort(inv, kind="stable")
        bounds = np.searchsorted(inv[members], np.arange(len(codes) + 1))
        for gi in range(len(codes)):
            sel = members[bounds[gi]:bounds[gi + 1]]
            bsel = _ranges_np(cuts[sel], nblk[sel])
            panels = (d.c_off[order[cuts[sel]]], K[sel], d.c_nr[order[cuts[sel]]],
                      (bstart[bsel], blen[bsel]), rs.coef_off[sn[cuts[sel]]], acc[sel])
            P = self._phase("coupling", int(rowh[sel].max()), panels, d.coup, None, self.xhat, None,
                            self.yhat, ordered=ordered)
            cpl.append((P, int(colh[sel].max()), set(rowh[sel].tolist())))
        return cpl

    def _xpos(self, p):
        """x_t buffer position of tree position p (index ranges never
        straddle a shard: they are leaf clusters)."""
        return p if self._xmap is None else self._xmap[np.asarray(p, np.int64)]

    def _level_phases(self, h):
        """The nested-basis recursion of h2.py:19-52 level by level: forward
        transform by height (bottom up), backward transform top down with
        the bucket heights each level waits for, and the leaf basis rows."""
        d = h.dev
        rs, cs = h.row_basis.store, h.col_basis.store
        rf, cf = h.row_tree.flat, h.col_tree.flat
        size_r = rf.stop - rf.start
        # forward transform (column basis), by height
        fwd = []
        mat = cs.materialized & (cs.rank > 0)
        for h_ in np.unique(cf.height[mat]):
            ids = np.flatnonzero(mat & (cf.height == h_))
            leaf = h_ == 0
            K = cs.rows[ids]
            base = self._xpos(cf.start[ids]) if leaf else cs.coef_off[cf.left[ids]]
            panels = (cs.v_off[ids], K, cs.rank[ids], (base, K), cs.coef_off[ids], 0)
            fwd.append(self._phase("forward", int(h_), panels, cs.V, None,
                                   self.xt if leaf else self.xhat, None, self.xhat, transform=True))
        # backward transform (row basis), top down
        bwd = []
        matb = rs.materialized & (rs.rank > 0) & ~rf.is_leaf
        for h_ in sorted(np.unique(rf.height[matb]), reverse=True):
            ids = np.flatnonzero(matb & (rf.height == h_))
            K = rs.rank[ids]
            panels = (rs.v_off[ids], K, rs.rows[ids], (rs.coef_off[ids], K), rs.coef_off[rf.left[ids]], 1)
            P = self._phase("backward", int(h_), panels, rs.transposed_V(), None, self.yhat, None, self.yhat,
                            transform=True)
            kids = np.r_[rf.left[ids], rf.right[ids]]
            bwd.append((P, set(rf.height[kids].tolist()) | {int(h_)}))
        # leaf basis: yt[leaf] += V yhat
        leafp = None
        leaves = np.flatnonzero(rf.is_leaf & rs.materialized & (rs.rank > 0))
        if d.row_range is not None:
            leaves = leaves[(rf.start[leaves] >= d.row_range[0]) & (rf.stop[leaves] <= d.row_range[1])]
        if leaves.size:
            K = rs.rank[leaves]
            panels = (rs.v_off[leaves], K, size_r[leaves], (rs.coef_off[leaves], K), rf.start[leaves], 1)
            # into yt2 (overwritten): the leaf basis need not wait for the near field
            panels = panels[:5] + (0,)
            leafp = self._phase("leafbasis", 0, panels, rs.transposed_V(), None, self.yhat, None, self.yt2,
                                transform=True)
        return fwd, bwd, leafp

    def _tiered(self, h, bounds):
        """Replace the level-by-level transforms by tiers (tiers.py): one
        launch per tier and direction, on the chain.  The lowest tier's
        backward writes the leaf rows of y (yt2) directly.  Returns (forward
        phases, backward (phase, bucket heights) top down, leaf parts
        (phase, bucket heights or None = all)).  Measured and rejected:
        the lowest tier split into one launch per height on parallel
        streams (forward) and per ancestor height accumulating as its
        bucket completes (backward) - 165 us against 136 us at sphere L6:
        the 4 x 2048 small leaf panels queue behind the bulk."""
        from . import tiers as T_
        rs, cs = h.row_basis.store, h.col_basis.store
        rf, cf = h.row_tree.flat, h.col_tree.flat
        d = h.dev
        explicit = None if bounds == "auto" else list(bounds)
        cb = T_.choose_tiers(cs, cf, bounds=explicit, max_rows=_ITEM_MAX_ROWS)
        # the tier choice depends on the tree, the live nodes and the ranks
        # only: a symmetric operator's row store gets the column store's
        same = (rf is cf and np.array_equal(rs.rank, cs.rank) and np.array_equal(rs.rows, cs.rows)
                and np.array_equal(rs.materialized, cs.materialized))
        rb = cb if (rs is cs or same) else T_.choose_tiers(rs, rf, bounds=explicit, max_rows=_ITEM_MAX_ROWS)
        if not cb or not rb:
            return None
        ct = T_.StoreTiers(cs, cf, cb, self.dev)
        rt = ct if (rs is cs and rb == cb) else T_.StoreTiers(rs, rf, rb, self.dev)
        groups, MT = rt.transposed(self.dev)
        if rt is not ct:
            rt.M = None                                  # only the transposed blocks are used
        self.tiers = dict(col=cb, row=rb, fwd_elems=ct.elems, bwd_elems=int(MT.numel()))
        self._keep.extend([ct.M, MT])
        self.tiers_pending = True
        nfwd = []
        for t in ct.tiers:
            u, f, w, nodes = t["u"], t["f"], t["w"], t["nodes"]
            low = t["lo"] < 0
            starts = self._xpos(cf.start[f]) if low else cs.coef_off[f]
            panels = (t["moff"][nodes], t["m"][nodes], cs.rank[nodes], (starts, w), cs.coef_off[nodes], 0)
            nfwd.append(self._phase("forward", t["hi"], panels, ct.M, None, self.xt if low else self.xhat,
                                    None, self.xhat, transform=True))
        nbwd, parts = [], []
        for t, g in reversed(list(zip(rt.tiers, groups))):
            first, uu, ff, ww, dst = g["first"], g["u"], g["f"], g["w"], g["dst"]
            if not first.size:
                continue
            cnt = np.diff(np.r_[first, len(ff)])
            elems = ff[first]
            low = t["lo"] < 0
            keep = np.ones(len(elems), bool)
            if low and d.row_range is not None:
                keep = (rf.start[elems] >= d.row_range[0]) & (rf.stop[elems] <= d.row_range[1])
            K = np.add.reduceat(rs.rank[uu], first)
            sel = np.repeat(keep, cnt)
            panels = (dst[first][keep], K[keep], ww[first][keep], (rs.coef_off[uu][sel], rs.rank[uu][sel]),
                      (rf.start[elems] if low else rs.coef_off[elems])[keep], 0)
            P = self._phase("leafbasis" if low else "backward", t["hi"], panels, MT, None, self.yhat,
                            self.yhat_t, self.yt2 if low else self.yhat_t, sum_inputs=True, transform=True)
            if low:
                parts.append((P, None))
            else:
                nbwd.append((P, set(range(t["lo"] + 1, t["hi"] + 1))))
        self.tiers_pending = False
        return nfwd, nbwd, parts

    # -- DAG -----------------------------------------------------------------
    def _split_height(self):
        """S = the lowest height whose coupling buckets together hold <= 20%
        of the coupling bytes.  Buckets at height >= S are small and gate
        the top of the backward chain: they get the chain's priority.  The
        deep buckets below S are the bulk: lower priority, and the higher
        the bucket the sooner the backward chain needs it, so the higher its
        priority."""
        if not self._cpl:
            return 0
        by_h = sorted(((P.height, P.bytes) for P, _, _ in self._cpl), reverse=True)
        total = sum(b for _, b in by_h)
        acc, S = 0, by_h[0][0] + 1
        for h_, b in by_h:
            if acc + b > 0.2 * total:
                break
            acc += b
            S = h_
        return S

    def _build_nodes(self, gather=True, after_gather=(), before_coupling=None, scatter=True):
        """Nodes in a valid serial order (a topological order of the DAG).
        ``gather`` / ``scatter``: True for the external-order gather of x /
        scatter of y, or a custom _Node; ``after_gather``: chain nodes
        before the forward transform (the sharded x all-gather);
        ``before_coupling``: a chain node every coupling launch waits for
        (the sharded x-hat all-gather)."""
        st = stream_handle
        nodes = []

        def add(n):
            nodes.append(n)
            return len(nodes) - 1

        S = self._split_height()
        least, greatest = self._prio
        levels = least - greatest
        def dl(*xs):
            return [x for x in xs if x is not None]

        # y-hat | y-hat from above | leaf rows: zeroed per product only when
        # a phase accumulates into its output (the level-by-level backward
        # transform); with tiers every output has one direct writer, and the
        # entries nobody writes stay zero from the allocation
        z = None
        if any(P.acc for P in self.phases):
            z = add(_Node("zero", "chain", fn=lambda: self._ybuf.zero_(),
                          native=(1, [self._ybuf.data_ptr(), 8 * self._ybuf.numel()])))
        if gather is True:
            gather = _Node("gather", "chain", fn=lambda: _native.call(
                "gc_gather_inv", ptr(self.x), ptr(self.iperm_in), self.n_in, ptr(self.xt), st()),
                native=(2, [self.x.data_ptr(), self.iperm_in.data_ptr(), self.n_in, self.xt.data_ptr()]),
                launches=1)
        # a shard with local-first blocks: its collectives run on their own
        # stream, the local near field and the forward transform start from
        # the own slice, the remote blocks follow the all-gathers
        split = self._col_local is not None
        g = z
        if gather:
            gather.deps = dl(z)
            g = add(gather)
        g_own = g
        for n in after_gather:
            n.deps = dl(g)
            if split:
                n.stream = "comm"
            g = add(n)
        g_x = g
        first = g_own if split else g_x
        last = first
        fwd_done = []                                   # (max height covered, node)
        near = add(_Node("nearfield", "near", dl(first), phase=self._near)) if self._near.nitems else None
        for P in self._fwd:
            if P.nitems:
                last = add(_Node("forward", "chain", dl(last), phase=P, priority=greatest))
                fwd_done.append((P.height, last))
        gate = None
        if before_coupling is not None:
            before_coupling.deps = dl(last, g_x if split else None)
            if split:
                before_coupling.stream = "comm"
            gate = add(before_coupling)
        bucket = {}                                     # row height -> coupling nodes

        def prio_of(P):
            if P.height >= S or levels < 2:
                return greatest
            pr = least - 1 - int(round(P.height * (levels - 2) / max(S - 1, 1)))
            return min(least - 1, max(greatest + 1, pr))

        for P, colh, heights in sorted(self._cpl, key=lambda c: c[0].height):
            if gate is not None and not split:
                dep = [gate]
            else:
                dep = [next((k for hh, k in fwd_done if hh >= colh), last)]
            k = add(_Node("coupling", "c%d" % P.height, dl(*dep, z), phase=P, priority=prio_of(P)))
            for hh in heights:
                bucket.setdefault(hh, []).append(k)
        for P, colh, heights in sorted(self._cpl_remote, key=lambda c: c[0].height):
            # after the x-hat all-gather and after the local phases that
            # wrote the rows it adds onto
            local = sorted({k for hh in heights for k in bucket.get(hh, [])})
            k = add(_Node("coupling", "c%d" % P.height, dl(gate, z) + local, phase=P, priority=prio_of(P)))
            for hh in heights:
                bucket.setdefault(hh, []).append(k)
        allb = sorted({k for ks in bucket.values() for k in ks})
        prev = gate if (gate is not None and not split) else last
        for P, hs in self._bwd:
            if P.nitems:
                need = sorted({k for x in hs for k in bucket.get(x, [])})
                prev = add(_Node("backward", "chain", dl(prev) + need, phase=P, priority=greatest))
        for P, hs in self._leafparts:
            need = allb if hs is None else sorted({k for x in hs for k in bucket.get(x, [])})
            prev = add(_Node("leafbasis", "chain", dl(prev) + need, phase=P, priority=greatest))
        if self._near_remote is not None and self._near_remote.nitems:
            near = add(_Node("nearfield", "near", dl(g_x, near), phase=self._near_remote))
        tail = dl(prev) + allb
        if near is not None:
            tail = tail + [near]
        if scatter is True:
            scatter = _Node("scatter", "chain", fn=lambda: _native.call(
                "gc_scatter2_inv", ptr(self.yt), ptr(self.yt2), ptr(self.iperm_out), self.n_out, ptr(self.y),
                st()), native=(3, [self.yt.data_ptr(), self.yt2.data_ptr(), self.iperm_out.data_ptr(), self.n_out,
                                   self.y.data_ptr()]), launches=1)
        if scatter:
            scatter.deps = tail
            add(scatter)
        else:
            add(_Node("join", "chain", tail, fn=lambda: None))
        return nodes

    def _stream(self, key):
        s = self.streams.get(key)
        if s is None:
            s = self.streams[key] = torch.cuda.Stream(device=self.dev, priority=self._bulk_priority)
        return s

    def _exec(self, nodes, serial=False, phase_events=None, phase="coupling"):
        main = torch.cuda.current_stream()
        if serial:
            st = stream_handle()
            first = lastn = None
            for i, n in enumerate(nodes):
                if n.name == phase:
                    first = i if first is None else first
                    lastn = i
            for i, n in enumerate(nodes):
                if phase_events is not None and i == first:
                    phase_events[0].record(main)
                if n.phase is not None:
                    self._launch(n.phase, st, n.stream == "chain", n.priority)
                else:
                    n.fn()
                if phase_events is not None and i == lastn:
                    phase_events[1].record(main)
            return
        fork = torch.cuda.Event()
        fork.record(main)
        events = [None] * len(nodes)
        used = set()
        for i, n in enumerate(nodes):
            s = self._stream(n.stream)
            if n.stream not in used:
                s.wait_event(fork)
                used.add(n.stream)
            for dep in n.deps:
                if nodes[dep].stream != n.stream:
                    s.wait_event(events[dep])
            with torch.cuda.stream(s):
                if n.phase is not None:
                    self._launch(n.phase, stream_handle(), n.stream == "chain", n.priority)
                else:
                    n.fn()
                ev = torch.cuda.Event()
                ev.record(s)
            events[i] = ev
        for key in used:                       # rejoin every forked stream
            last = max(i for i, n in enumerate(nodes) if n.stream == key)
            main.wait_event(events[last])

    # -- phases --------------------------------------------------------------
    def _phase(self, name, height, panels, A0, A1, in0, in1, out, transform=False, sum_inputs=False,
               ordered=False):
        """Work items of one phase.  panels = (a_off, K, T, rows, out_off,
        accumulate): panel p is the K x T row-major block at A[a_off] whose
        row k multiplies in[idx] (rows = (starts, lengths) index ranges,
        expanded on the device, or an explicit index array).  Transform
        phases get one item per panel (split only past the row cap: they are
        latency-bound, and a split panel costs a second pass over L2 for its
        reduction); bulk phases are cut into items of <= _ITEM_ELEMS
        elements, about _BULK_ITEMS_PER_SM per SM per phase (fewer, larger
        items: fewer split-panel reductions; the concurrent phases fill
        the SMs).  A panel split over
        several items writes partial sums to scratch and its last item adds
        them in item order."""
        a_off, K, T, rows, out_off, accumulate = panels
        a_off = np.asarray(a_off, np.int64)
        K = np.asarray(K, np.int64)
        T = np.asarray(T, np.int64)
        out_off = np.asarray(out_off, np.int64)
        n = len(a_off)
        elems = int((K * T).sum())
        ring = bool(not transform and n and int(T.max()) <= 256
                    and (self._bulk == "ring" or (self._bulk == "auto" and 8 * elems >= _RING_MIN_BYTES)))
        # small bulk phases (a few MB: the latency-bound products of small
        # operators) get one item per panel, paired like the tier phases
        small_bulk = bool(not transform and n and 8 * elems <= self._pair_bulk)
        if transform or small_bulk:
            target = 1 << 40
        else:
            target = max(256, min(_ITEM_ELEMS, elems // (148 * _BULK_ITEMS_PER_SM) + 1))
        rpi = np.minimum(_ITEM_MAX_ROWS, np.maximum(1, -(-target // np.maximum(T, 1))))  # rows/item
        # at most 8 items per panel: the last item of a split panel sums the
        # partials serially, so deep splits of small phases cost latency
        rpi = np.maximum(rpi, np.minimum(_ITEM_MAX_ROWS, -(-K // 8)))
        nit = np.maximum(1, -(-K // rpi))
        segs = rows if isinstance(rows, tuple) else None      # (starts, lengths) of index ranges
        xidx = None if segs is not None else (np.asarray(rows).astype(np.int32) if n else np.zeros(1, np.int32))
        xoff = _offsets_np(K)
        item_panel = np.repeat(np.arange(n), nit)
        item_idx_in_panel = _ranges_np(np.zeros(n, np.int64), nit)
        item_k = item_idx_in_panel * rpi[item_panel]
        item_rows = np.minimum(rpi[item_panel], K[item_panel] - item_k)
        multi = nit > 1
        scr_off = _offsets_np(np.where(multi, nit * T, 0))
        slot = np.cumsum(multi) - 1                  # reduction slot of each split panel
        direct = ~multi[item_panel]
        out_col = np.where(direct, out_off[item_panel],
                           scr_off[item_panel] + item_idx_in_panel * T[item_panel])
        acc = np.broadcast_to(np.asarray(accumulate, np.int64), (n,))      # per panel
        mode = np.where(direct, 4 | (8 * acc[item_panel]), 0) | (32 if sum_inputs else 0)
        items = np.stack([a_off[item_panel] + item_k * T[item_panel], xoff[item_panel] + item_k,
                          out_col, T[item_panel], item_rows, mode,
                          np.where(direct, -1, slot[item_panel]), np.zeros_like(mode)], 1).reshape(-1, 8)
        red = np.stack([out_off[multi], T[multi], scr_off[multi], nit[multi], acc[multi]], 1)
        P = _Phase()
        P.name, P.height = name, height
        # some item adds into an output that no earlier phase of the same
        # product wrote (``ordered``: the phase only adds onto outputs its
        # dependencies wrote) - the product then needs its memset
        P.acc = bool(n and acc.any() and not ordered)
        # two whole small panels per CTA (k_panel_pair) in the tier phases
        # whose items all fit: half the CTAs, half the waves of round trips
        P.pair = bool(((transform and self.tiers_pending) or small_bulk) and n and bool(np.all(direct))
                      and int(T.max()) <= 128
                      and int(item_rows.max()) <= 512
                      and int((item_rows * T[item_panel]).max()) <= _PAIR_MAX_ELEMS)
        if P.pair:   # pair equal-sized panels, largest first
            items = items[np.argsort(-(items[:, 3] * items[:, 4]), kind="stable")]
        # large bulk phases stream through the TMA ring kernel (k_panel_ring)
        P.ring = ring
        # the device tables of every phase go up together (_flush_tables)
        P._h_items = self._stage(self._t64, items)
        if segs is not None:
            st_, ln_ = np.asarray(segs[0], np.int64), np.asarray(segs[1], np.int64)
            P._h_xidx = ("ranges", st_, ln_, int(ln_.sum()))
        else:
            P._h_xidx = ("explicit", self._stage(self._t32, xidx))
        P.nitems, P.nred = len(items), int(multi.sum())
        P._h_red = self._stage(self._t64, red) if P.nred else None
        P._n_arrivals = max(P.nred, 1)
        P._n_scratch = max(int((np.where(multi, nit * T, 0)).sum()), 1)
        P.items = P.xidx = P.red = P.arrivals = P.scratch = None
        self._staged.append(P)
        P.A0, P.A1, P.in0, P.in1, P.out = A0, A1, in0, in1, out
        P.scratch = torch.zeros(max(int((np.where(multi, nit * T, 0)).sum()), 1),
                                dtype=torch.float64, device=self.dev)
        P.bytes = 8 * elems
        P.in_elems, P.out_elems = int(K.sum()), int(T.sum())
        return P

    @staticmethod
    def _stage(parts, a):
        """Queue a host table for the plan's single upload; returns its
        (element offset, length), segments 16-byte aligned."""
        a = np.ascontiguousarray(a).ravel()
        off = sum(len(x) for x in parts)
        parts.append(a)
        pad = (-len(a)) % 4
        if pad:
            parts.append(np.zeros(pad, a.dtype))
        return off, len(a)

    def _flush_tables(self):
        """One upload per element type for the tables of every phase, one
        launch expanding all index ranges, one zeroed buffer each for the
        split-panel arrivals and partial sums."""
        staged, self._staged = self._staged, []
        if not staged:
            return
        d64 = to_dev(np.concatenate(self._t64) if self._t64 else np.zeros(4, np.int64), self.dev)
        d32 = to_dev(np.concatenate(self._t32) if self._t32 else np.zeros(4, np.int32), self.dev)
        self._t64, self._t32 = [], []
        rng = [P for P in staged if P._h_xidx[0] == "ranges"]
        sizes = [P._h_xidx[3] + (-P._h_xidx[3]) % 4 for P in rng]
        xbuf = torch.empty(max(sum(sizes), 4), dtype=torch.int32, device=self.dev)
        arr = torch.zeros(sum(P._n_arrivals + (-P._n_arrivals) % 4 for P in staged), dtype=torch.int32,
                          device=self.dev)
        scr = torch.zeros(sum(P._n_scratch + (-P._n_scratch) % 4 for P in staged), dtype=torch.float64,
                          device=self.dev)
        self._keep.extend([d64, d32, xbuf, arr, scr])
        base = 0
        starts, lens, outs = [], [], []
        for P, sz in zip(rng, sizes):
            _, st_, ln_, total = P._h_xidx
            P.xidx = xbuf[base:base + max(total, 1)]
            starts.append(st_)
            lens.append(ln_)
            outs.append(base + _offsets_np(ln_))
            base += sz
        if rng and sum(len(x) for x in starts):
            tab = to_dev(np.concatenate(starts + lens + outs), self.dev)
            m = sum(len(x) for x in starts)
            with torch.cuda.device(self.dev):
                _native.call("gc_expand_ranges", m, ptr(tab[:m]), ptr(tab[m:2 * m]), ptr(tab[2 * m:]),
                             ptr(xbuf), stream_handle())
        oa = os_ = 0
        for P in staged:
            o, n = P._h_items
            P.items = d64[o:o + n]
            if P._h_xidx[0] == "explicit":
                o, n = P._h_xidx[1]
                P.xidx = d32[o:o + n]
            if P._h_red is not None:
                o, n = P._h_red
                P.red = d64[o:o + n]
            P.arrivals = arr[oa:oa + P._n_arrivals]
            P.scratch = scr[os_:os_ + P._n_scratch]
            oa += P._n_arrivals + (-P._n_arrivals) % 4
            os_ += P._n_scratch + (-P._n_scratch) % 4
            del P._h_items, P._h_xidx, P._h_red

    def _launch(self, P, stream, chain=False, priority=0):
        mode = (1 if chain else 0) | (16 if P.pair else 0) | (32 if P.ring else 0)
        _native.call("gc_panelmv", P.nitems, ptr(P.items), ptr(P.xidx), ptr(P.A0), ptr(P.A1),
                     ptr(P.in0), ptr(P.in1), ptr(P.out), ptr(P.scratch), P.nred, ptr(P.red),
                     ptr(P.arrivals), mode, int(priority), ptr(self.trace.get(id(P))), stream)

    def _body(self, phase_events=None, phase="coupling"):
        self._exec(self.nodes, serial=phase_events is not None, phase_events=phase_events, phase=phase)

    def _native_table(self):
        """The DAG as gc_plan_create's node table (csrc/plan.cu), or None
        when a node is a Python callable (the sharded plan's collectives)."""
        skip = {i for i, n in enumerate(self.nodes) if n.name == "join"}
        remap, rows, deps, streams = {}, [], [], {"chain": 0}
        for i, n in enumerate(self.nodes):
            if i in skip:
                continue
            sidx = streams.setdefault(n.stream, len(streams))
            a = [0] * 12
            if n.phase is not None:
                P = n.phase
                kind = 0
                chain = (1 if n.stream == "chain" else 0) | (16 if P.pair else 0) | (32 if P.ring else 0)
                a = [P.items.data_ptr(), P.nitems, P.xidx.data_ptr(), P.A0.data_ptr(),
                     P.A1.data_ptr() if P.A1 is not None else 0, P.in0.data_ptr(),
                     P.in1.data_ptr() if P.in1 is not None else 0, P.out.data_ptr(), P.scratch.data_ptr(),
                     P.nred, P.red.data_ptr() if P.red is not None else 0, P.arrivals.data_ptr()]
            elif n.native is not None:
                kind, chain = n.native[0], 0
                a[:len(n.native[1])] = n.native[1]
            else:
                return None
            d = [remap[j] for j in n.deps if j not in skip]
            rows.append([kind, sidx, n.priority, chain, len(d), len(deps)] + a)
            deps.extend(d)
            remap[i] = len(rows) - 1
        least, greatest = self._prio
        prio = np.array([greatest if k == "chain" else least for k in streams], np.int32)
        return (np.array(rows, np.int64).reshape(-1, 18), np.array(deps or [0], np.int64), len(deps), prio)

    def capture(self):
        """Record the product into a CUDA graph: the C++ executor
        (csrc/plan.cu: its own streams, events and graph); a DAG with Python
        steps (the sharded plan's collectives) is captured through torch.
        A failed capture raises."""
        import time
        t0 = time.perf_counter()
        # phase timelines (self.trace, diagnostics) need the Python launches
        tab = self._native_table() if not self.trace else None
        if tab is not None:
            self._body()                         # warm-up (module loads) outside the capture
            torch.cuda.synchronize(self.dev)
            self.timing["warmup_s"] = time.perf_counter() - t0
            rows, deps, ndeps, prio = tab
            h = _native.ctypes.c_void_p(0)
            _native.call("gc_plan_create", len(rows), rows.ctypes.data, ndeps, deps.ctypes.data, len(prio),
                         prio.ctypes.data, _native.ctypes.byref(h))
            self.graph = _NativeGraph(h)
            self.timing["capture_s"] = time.perf_counter() - t0
            return self.graph
        s = torch.cuda.Stream(device=self.dev)
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            self._body()                   # warm-up outside capture
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize(self.dev)
        # capture_begin/end on a side stream directly: torch.cuda.graph()
        # would empty the caching allocator first (and the assembly's next
        # allocations would pay cudaMalloc again)
        g = torch.cuda.CUDAGraph(keep_graph=True)
        with torch.cuda.stream(s):
            g.capture_begin()
            try:
                self._body()
            finally:
                g.capture_end()
        g.instantiate()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize(self.dev)
        self.graph = g
        # the gather / scatter nodes read self.x / write self.y until run()
        # re-points them at the caller's buffers (gc_graph_retarget)
        self._captured = [self.x.data_ptr(), self.y.data_ptr()]
        self._bound = list(self._captured)
        return g

    def bind(self, x_dev, y_dev):
        """Point the captured graph's input gather at x_dev and its output
        scatter at y_dev (contiguous float64 vectors of this plan's sizes,
        device or pinned host; they must stay alive until the replays that
        use them ran)."""
        if isinstance(self.graph, _NativeGraph):
            self.graph.bind(x_dev, y_dev)
            return True
        if self.graph is None:
            return False
        want = [x_dev.data_ptr(), y_dev.data_ptr()]
        for slot, (kernel, arg) in enumerate(((2, 0), (3, 4))):
            if want[slot] == self._bound[slot]:
                continue
            cnt = _native.ctypes.c_int32(0)
            _native.call("gc_graph_retarget", _native.ctypes.c_void_p(self.graph.raw_cuda_graph()),
                         _native.ctypes.c_void_p(self.graph.raw_cuda_graph_exec()), kernel, arg,
                         _native.ctypes.c_void_p(self._captured[slot]), _native.ctypes.c_void_p(want[slot]),
                         _native.ctypes.byref(cnt))
            if cnt.value != 1:
                raise StateError("product graph: %d gather/scatter nodes re-pointed (expected 1)" % cnt.value)
            self._bound[slot] = want[slot]
        return True

    def _direct_ok(self, x_dev, y_dev):
        return (self.graph is not None and x_dev.is_contiguous() and y_dev.is_contiguous()
                and x_dev.dtype == torch.float64 and y_dev.dtype == torch.float64
                and x_dev.device == self.x.device and y_dev.device == self.y.device
                and x_dev.numel() == self.n_in and y_dev.numel() == self.n_out
                and x_dev.data_ptr() != y_dev.data_ptr())

    def run(self, x_dev, y_dev, phase_events=None, phase="coupling", serial=False):
        """y_dev = H x_dev (device vectors, external ordering) on the current
        stream; one product at a time per plan (the plan's buffers are
        shared).  With ``phase_events`` (or ``serial``) every node runs in
        order on the current stream and the events bracket the named
        phase's kernels."""
        with self.lock:
            if phase_events is None and not serial and self._direct_ok(x_dev, y_dev):
                self.bind(x_dev, y_dev)              # graph reads x_dev, writes y_dev: no copies
                self.graph.replay()
                return
            self.x.copy_(x_dev, non_blocking=True)
            if phase_events is None and not serial and self.graph is not None:
                self.bind(self.x, self.y)
                self.graph.replay()
            else:
                self._exec(self.nodes, serial=serial or phase_events is not None,
                           phase_events=phase_events, phase=phase)
            y_dev.copy_(self.y, non_blocking=True)

    def apply_host(self, x):
        """Host vector in, host vector out; thread-safe (one product at a
        time per plan).  The input is staged in the plan's pinned buffer,
        which the graph's gather kernel reads over the host link; the
        scatter kernel writes a fresh pinned array (torch's pinned block
        cache) that is returned without a copy."""
        with self.lock:
            g = self.graph
            if isinstance(g, _NativeGraph) and torch._C._cuda_getDevice() == self._dev_index:
                # the e2e hot path: staging copy, graph and sync in one C call
                if self._pin_x_np is None:
                    self._pin_x = torch.empty(self.n_in, dtype=torch.float64, pin_memory=True)
                    self._pin_x_np = self._pin_x.numpy()
                x = np.ascontiguousarray(x, dtype=np.float64)
                y = torch.empty(self.n_out, dtype=torch.float64, pin_memory=True)
                px, py = self._pin_x.data_ptr(), y.data_ptr()
                # the raw current stream (the torch.cuda.Stream wrapper costs ~2 us per call)
                _native.check(g._run_host(g.handle, x.ctypes.data, px, self.n_in, py,
                                          torch._C._cuda_getCurrentRawStream(self._dev_index)))
                g._x, g._y = px, py
                return y.numpy()
            with torch.cuda.device(self.dev):
                if self._pin_x_np is None:
                    self._pin_x = torch.empty(self.n_in, dtype=torch.float64, pin_memory=True)
                    self._pin_x_np = self._pin_x.numpy()
                np.copyto(self._pin_x_np, x)
                y = torch.empty(self.n_out, dtype=torch.float64, pin_memory=True)
                if self.graph is not None and self.bind(self._pin_x, y):
                    self.graph.replay()
                else:
                    self.x.copy_(self._pin_x, non_blocking=True)
                    self._body()
                    y.copy_(self.y, non_blocking=True)
                torch.cuda.current_stream().synchronize()
                return y.numpy()

    @property
    def num_kernels(self):
        """Own kernels per product (the y-hat memset not counted)."""
        return sum(n.launches for n in self.nodes)


class _NativeGraph:
    """The product graph owned by the C++ executor (gc_plan_*): replay()
    launches it on the current stream with the last bound x / y."""

    def __init__(self, handle):
        self.handle = handle
        self._x = self._y = 0
        self._run = _native.load().gc_plan_run        # bound once: this is on the e2e path
        self._run_host = _native.load().gc_plan_run_host

    def bind(self, x, y):
        self._x, self._y = x.data_ptr(), y.data_ptr()

    def replay(self):
        _native.check(self._run(self.handle, self._x, self._y, torch.cuda.current_stream().cuda_stream))

    def __del__(self):
        try:
            _native.load().gc_plan_destroy(self.handle)
        except Exception:        # pragma: no cover - interpreter shutdown
            pass


def _offsets_np(sizes):
    sizes = np.asarray(sizes, dtype=np.int64)
    return np.cumsum(sizes) - sizes


def _inverse_perm(perm):
    inv = torch.empty_like(perm)
    inv[perm] = torch.arange(perm.numel(), dtype=perm.dtype, device=perm.device)
    return inv


def _ranges_np(starts, lengths):
    lengths = np.asarray(lengths, dtype=np.int64)
    total = int(lengths.sum())
    if total == 0:
        return np.zeros(0, dtype=np.int64)
    heads = np.cumsum(lengths) - lengths
    return np.arange(total, dtype=np.int64) + np.repeat(np.asarray(starts, np.int64) - heads, lengths)


# --------------------------------------------------------------------------
# device solvers (h2.py:144-253): vectors and scalars stay in HBM

CGResult = namedtuple("CGResult", "x residuals converged")


class _DevOp:
    """apply(x_dev, y_dev, trans) for an H2Operator (flow plans) or any
    host closure (x copied to the host and back)."""

    def __init__(self, op, n, dev):
        self.op, self.n, self.dev = op, n, dev

    def __call__(self, x, y, trans=False):
        if isinstance(self.op, H2Operator):
            self.op.apply_device(x, y, trans)
        else:
            r = np.asarray(self.op(x.cpu().numpy(), trans) if trans else self.op(x.cpu().numpy()),
                           dtype=np.float64)
            y.copy_(torch.from_numpy(r))


class _Vec:
    """Device BLAS-1 on float64 vectors through csrc/krylov.cu."""

    def __init__(self, n, dev):
        self.n, self.dev = n, dev
        self.partial = torch.empty(int(_native.load().gc_krylov_partials()), dtype=torch.float64, device=dev)

    def dot(self, a, b, out):
        _native.call("gc_dot", self.n, ptr(a), ptr(b), ptr(self.partial), ptr(out), _stream_ptr())



def _device_of(op):
    if isinstance(op, H2Operator):
        return op.h.dev.device
    return torch.device("cuda", torch.cuda.current_device())


def cg_solve(apply, b, tol=1e-8, max_iter=500):
    """Conjugate gradients on an SPD operator (``h2.py:190-219``) with every
    vector and scalar in HBM (``gc_cg_*``); per iteration one product and a
    16-byte read of (r.r, stop flag).  Returns a :class:`CGResult` with host
    arrays."""
    from .device import require_device
    dev = require_device(_device_of(apply))
    b = np.asarray(b, dtype=np.float64)
    n = b.size
    op = _DevOp(apply, n, dev)
    with torch.cuda.device(dev):
        b_d = torch.from_numpy(b.copy()).to(dev)
        x = torch.zeros_like(b_d)
        r = b_d.clone()
        p = b_d.clone()
        q = torch.empty_like(b_d)
        s = torch.zeros(8, dtype=torch.float64, device=dev)
        v = _Vec(n, dev)
        v.dot(b_d, b_d, s)
        bnorm = float(np.sqrt(s[0].item()))
        hist = [bnorm]
        if bnorm == 0.0:
            return CGResult(x.cpu().numpy(), np.asarray(hist), True)
        for _ in range(max_iter):
            if hist[-1] <= tol * bnorm:
                break
            op(p, q)
            _native.call("gc_cg_pq", n, ptr(p), ptr(q), ptr(v.partial), ptr(s), _stream_ptr())
            _native.call("gc_cg_update", n, ptr(x), ptr(r), ptr(p), ptr(q), ptr(v.partial), ptr(s),
                         _stream_ptr())
            host = s[[0, 5]].cpu().numpy()
            if host[1] != 0.0:
                break
            hist.append(float(np.sqrt(host[0])))
        return CGResult(x.cpu().numpy(), np.asarray(hist), bool(hist[-1] <= tol * bnorm))


def cgnr_solve(apply, b, tol=1e-8, max_iter=500):
    """CG on the normal equations (``h2.py:222-253``); the history is the
    true residual ||b - A x||.  Device-resident like :func:`cg_solve`: per
    iteration A p, A^T r and the fused updates of ``gc_cgnr_*``."""
    from .device import require_device
    dev = require_device(_device_of(apply))
    b = np.asarray(b, dtype=np.float64)
    n = b.size
    op = _DevOp(apply, n, dev)
    with torch.cuda.device(dev):
        b_d = torch.from_numpy(b.copy()).to(dev)
        x = torch.zeros_like(b_d)
        r = b_d.clone()
        sv = torch.empty_like(b_d)
        q = torch.empty_like(b_d)
        # s: [0] ss, [1] q.q, [2] r.r, [3] b.b, [4] new ss, [5] stop flag
        s = torch.zeros(8, dtype=torch.float64, device=dev)
        v = _Vec(n, dev)
        op(r, sv, True)
        p = sv.clone()
        v.dot(sv, sv, s[0:])
        v.dot(r, r, s[2:])
        v.dot(b_d, b_d, s[3:])
        host = s.cpu().numpy()
        bnorm = float(np.sqrt(host[3]))
        hist = [float(np.sqrt(host[2]))]
        if bnorm == 0.0:
            return CGResult(x.cpu().numpy(), np.asarray(hist), True)
        ss0 = host[0]
        for _ in range(max_iter):
            if hist[-1] <= tol * bnorm or ss0 == 0.0:
                break
            op(p, q)
            # q.q; stop if zero; alpha = ss / q.q; x += alpha p; r -= alpha q; r.r
            _native.call("gc_cgnr_step", n, ptr(x), ptr(r), ptr(p), ptr(q), ptr(v.partial), ptr(s),
                         _stream_ptr())
            host = s[[2, 5]].cpu().numpy()
            if host[1] != 0.0:
                break
            hist.append(float(np.sqrt(host[0])))
            op(r, sv, True)
            # ss_new = s.s; p = s + (ss_new / ss) p; ss = ss_new
            _native.call("gc_cgnr_dir", n, ptr(sv), ptr(p), ptr(v.partial), ptr(s), _stream_ptr())
            ss0 = float(s[0].item())
        return CGResult(x.cpu().numpy(), np.asarray(hist), bool(hist[-1] <= tol * bnorm))


def spectral_error_estimate(apply_ref, apply_approx, n, iters=100, seed=0):
    """Power-iteration estimate of ||ref - approx||_2 and of its ratio to
    ||ref||_2 (``h2.py:144-184``): z <- E^T (E z) / ||.|| on device vectors
    (the start vector is the reference's seeded N(0,1) draw); both
    operators take (x, trans=False)."""
    if iters < 1:
        raise ConfigError("iters must be positive")
    from .device import require_device
    dev = require_device(_device_of(apply_approx if isinstance(apply_approx, H2Operator) else apply_ref))
    with torch.cuda.device(dev):
        ref = _DevOp(apply_ref, n, dev)
        app = _DevOp(apply_approx, n, dev)
        v = _Vec(n, dev)

        def power(diff):
            z0 = np.random.default_rng(seed).standard_normal(n)
            if np.linalg.norm(z0) == 0.0:
                z0 = np.random.default_rng(seed + 1).standard_normal(n)
                if np.linalg.norm(z0) == 0.0:
                    raise ConfigError("degenerate start vector")
            z = torch.from_numpy(z0).to(dev)
            w = torch.empty_like(z)
            w2 = torch.empty_like(z)
            s = torch.zeros(8, dtype=torch.float64, device=dev)
            v.dot(z, z, s)
            _native.call("gc_scale_inv_norm", n, ptr(z), ptr(s), _stream_ptr())    # z /= sqrt(s[0])
            est = 0.0
            for _ in range(iters):
                ref(z, w)
                if diff:
                    app(z, w2)
                    _native.call("gc_axpy_neg", n, ptr(w2), ptr(w), _stream_ptr())    # w -= w2
                v.dot(w, w, s)
                est = float(np.sqrt(s[0].item()))
                if est == 0.0:
                    return 0.0
                ref(w, z, True)
                if diff:
                    app(w, w2, True)
                    _native.call("gc_axpy_neg", n, ptr(w2), ptr(z), _stream_ptr())
                v.dot(z, z, s)
                if s[0].item() == 0.0:
                    return est
                _native.call("gc_scale_inv_norm", n, ptr(z), ptr(s), _stream_ptr())
            return est

        err = power(True)
        nref = power(False)
    if nref == 0.0:
        return err, (0.0 if err == 0.0 else np.inf)
    return err, err / nref
