"""H2 matrix-vector products on the device, storage accounting, solvers.

Mirror of ``greencross/h2.py``.  ``mvm`` / ``mvm_t`` (``h2.py:63-100``) keep
the reference's signature (host vectors in external ordering) and run as a
fixed sequence of ``gc_segmv`` launches over level-wise batches:

  gather x[perm] -> forward transform (leaves, then one launch per tree
  height) -> coupling (one launch, segment = row cluster) -> backward
  transform (one launch per height, top down) -> leaf basis + near-field
  (one launch, segment = row leaf) -> scatter y[perm].

The launch sequence is captured once into a CUDA graph per matrix and
direction and replayed.  ``storage_report`` (``h2.py:110-134``) counts the
same bytes the reference does; ``spectral_error_estimate``, ``cg_solve``
and ``cgnr_solve`` are host consumers of the device matvec.
"""

import os
from collections import namedtuple

import numpy as np

from . import _native
from .device import empty, ptr, stream_handle, to_dev, torch
from .errors import ConfigError, StateError

__all__ = ["mvm", "mvm_t", "as_operator", "storage_report", "storage_csv_rows",
           "spectral_error_estimate", "cg_solve", "cgnr_solve", "CGResult", "MatvecPlan"]


class _Launch:
    __slots__ = ("seg", "blk", "nseg", "A0", "A1", "in0", "in1", "out", "acc", "maxT", "name")


class MatvecPlan:
    """Device descriptors and buffers for one product direction."""

    def __init__(self, h, trans=False):
        d = h.dev
        dev = d.device
        self.dev = dev
        self.trans = trans
        rs = h.row_basis.store
        cs = h.col_basis.store
        rf, cf = h.row_tree.flat, h.col_tree.flat
        if trans:
            # H^T: forward on the row basis, backward on the column basis
            fwd, bwd, ftree, btree_ = rs, cs, rf, cf
        else:
            fwd, bwd, ftree, btree_ = cs, rs, cf, rf
        self.n_in = ftree.stop[0]
        self.n_out = btree_.stop[0]
        self.perm_in = d.perm_r if trans else d.perm_c
        self.perm_out = d.perm_c if trans else d.perm_r
        self.xt = torch.zeros(self.n_in, dtype=torch.float64, device=dev)
        self.yt = torch.zeros(self.n_out, dtype=torch.float64, device=dev)
        self.xhat = torch.zeros(max(fwd.coef_size, 1), dtype=torch.float64, device=dev)
        self.yhat = torch.zeros(max(bwd.coef_size, 1), dtype=torch.float64, device=dev)
        self.launches = []
        size_f = ftree.stop - ftree.start
        size_b = btree_.stop - btree_.start
        fwdA = fwd.VT if trans else fwd.V
        bwdA = bwd.V if trans else bwd.VT

        # ---- forward transform
        mat = fwd.materialized & (fwd.rank > 0)
        for h_ in np.unique(ftree.height[mat]):
            ids = np.flatnonzero(mat & (ftree.height == h_))
            T = fwd.rank[ids]
            leaf = ftree.is_leaf[ids]
            K = fwd.rows[ids]                       # leaf: size, internal: sum child ranks
            first_child = np.where(leaf, 0, ftree.left[ids])
            in_off = np.where(leaf, ftree.start[ids], fwd.coef_off[np.maximum(first_child, 0)])
            if trans:   # stored V^T (r x R): element (k, t) at t*R + k
                lda, ts = np.ones_like(T), K
            else:       # stored V (R x r): element (k, t) at k*r + t
                lda, ts = T, np.ones_like(T)
            # leaves read the permuted input vector, internal nodes x-hat
            for is_leaf in (True, False):
                sel = leaf == is_leaf
                if not sel.any():
                    continue
                n = int(sel.sum())
                seg = np.stack([fwd.coef_off[ids[sel]], T[sel], np.arange(n), np.arange(1, n + 1)], 1)
                blk = np.stack([fwd.v_off[ids[sel]], K[sel], lda[sel], in_off[sel],
                                np.zeros(n, np.int64), ts[sel]], 1)
                self._add(seg, blk, fwdA, None, self.xt if is_leaf else self.xhat, None,
                          self.xhat, 0, "forward")

        # ---- coupling
        c_off = d.c_off
        if trans:
            seg_node, in_node = d.c_cols, d.c_rows
            T_all, K_all = d.c_nc, d.c_nr
            lda_all, ts_all = np.ones_like(T_all), d.c_nr
        else:
            seg_node, in_node = d.c_rows, d.c_cols
            T_all, K_all = d.c_nr, d.c_nc
            lda_all, ts_all = d.c_nr, np.ones_like(T_all)
        live = (T_all > 0) & (K_all > 0)
        order = np.flatnonzero(live)[np.argsort(seg_node[live], kind="stable")]
        if order.size:
            sn = seg_node[order]
            cuts = np.flatnonzero(np.r_[True, sn[1:] != sn[:-1]])
            ends = np.r_[cuts[1:], len(order)]
            seg = np.stack([bwd.coef_off[sn[cuts]], T_all[order][cuts], cuts, ends], 1)
            blk = np.stack([c_off[order], K_all[order], lda_all[order],
                            fwd.coef_off[in_node[order]], np.zeros(len(order), np.int64),
                            ts_all[order]], 1)
            self._add(seg, blk, d.coup, None, self.xhat, None, self.yhat, 0, "coupling")

        # ---- backward transform, top down
        matb = bwd.materialized & (bwd.rank > 0) & ~btree_.is_leaf
        for h_ in sorted(np.unique(btree_.height[matb]), reverse=True):
            ids = np.flatnonzero(matb & (btree_.height == h_))
            T = bwd.rows[ids]                       # sum of child ranks
            K = bwd.rank[ids]
            out_off = bwd.coef_off[btree_.left[ids]]
            if trans:   # V-hat (R x r) row-major: element (k, t) at t*r + k
                lda, ts = np.ones_like(T), K
            else:       # V-hat^T (r x R): element (k, t) at k*R + t
                lda, ts = T, np.ones_like(T)
            n = len(ids)
            seg = np.stack([out_off, T, np.arange(n), np.arange(1, n + 1)], 1)
            blk = np.stack([bwd.v_off[ids], K, lda, bwd.coef_off[ids], np.zeros(n, np.int64), ts], 1)
            self._add(seg, blk, bwdA, None, self.yhat, None, self.yhat, 1, "backward")

        # ---- leaf basis + near field, one segment per output leaf
        if trans:
            n_seg, n_in = d.n_cols, d.n_rows
            nT, nK = d.n_nc, d.n_nr
            nlda, nts = np.ones_like(nT), d.n_nr
            in_tree = rf
        else:
            n_seg, n_in = d.n_rows, d.n_cols
            nT, nK = d.n_nr, d.n_nc
            nlda, nts = d.n_nr, np.ones_like(nT)
            in_tree = cf
        leaves = np.flatnonzero(btree_.is_leaf)
        if d.row_range is not None and not trans:
            leaves = leaves[(btree_.start[leaves] >= d.row_range[0])
                            & (btree_.stop[leaves] <= d.row_range[1])]
        has_basis = bwd.materialized[leaves] & (bwd.rank[leaves] > 0)
        # rows of the block table: near blocks (sel 0) and leaf-basis blocks (sel 3)
        bl_seg = np.concatenate([n_seg, leaves[has_basis]])
        bl = np.concatenate([
            np.stack([d.n_off, nK, nlda, in_tree.start[n_in], np.zeros(len(n_seg), np.int64), nts], 1),
            np.stack([bwd.v_off[leaves[has_basis]], bwd.rank[leaves[has_basis]],
                      np.ones(int(has_basis.sum()), np.int64) if trans else size_b[leaves[has_basis]],
                      bwd.coef_off[leaves[has_basis]], np.full(int(has_basis.sum()), 3, np.int64),
                      bwd.rank[leaves[has_basis]] if trans else np.ones(int(has_basis.sum()), np.int64)], 1)
        ]).reshape(-1, 6)
        order = np.argsort(bl_seg, kind="stable")
        bl_seg, bl = bl_seg[order], bl[order]
        # segments: every output leaf (blocks may be empty -> writes zeros)
        first = np.searchsorted(bl_seg, leaves, side="left")
        last = np.searchsorted(bl_seg, leaves, side="right")
        seg = np.stack([btree_.start[leaves], size_b[leaves], first, last], 1)
        leafA = bwd.V if trans else bwd.VT
        self._add(seg, bl, d.near, leafA, self.xt, self.yhat, self.yt, 0, "leaf_near")

    def _add(self, seg, blk, A0, A1, in0, in1, out, acc, name):
        if len(seg) == 0:
            return
        L = _Launch()
        L.seg = to_dev(np.ascontiguousarray(seg, dtype=np.int64), self.dev)
        L.blk = to_dev(np.ascontiguousarray(blk, dtype=np.int64).reshape(-1, 6), self.dev) \
            if len(blk) else torch.zeros(6, dtype=torch.int64, device=self.dev)
        L.nseg = len(seg)
        L.A0, L.A1, L.in0, L.in1, L.out, L.acc = A0, A1, in0, in1, out, acc
        L.maxT = int(np.max(seg[:, 1]))
        L.name = name
        self.launches.append(L)

    def run(self, x_dev, y_dev, phase_events=None, phase="coupling"):
        """y_dev = H x_dev (or H^T) for device vectors in external order.
        ``phase_events=(start, end)`` records CUDA events around the launch
        named ``phase`` (bench roofline timing on the launching stream)."""
        stream = stream_handle()
        _native.call("gc_gather", ptr(x_dev), ptr(self.perm_in), self.n_in, ptr(self.xt), stream)
        self.yhat.zero_()
        for L in self.launches:
            timed = phase_events is not None and L.name == phase
            if timed:
                phase_events[0].record()
            _native.call("gc_segmv", L.nseg, ptr(L.seg), ptr(L.blk), ptr(L.A0), ptr(L.A1),
                         ptr(L.in0), ptr(L.in1), ptr(L.out), L.acc, L.maxT, stream)
            if timed:
                phase_events[1].record()
        _native.call("gc_scatter", ptr(self.yt), ptr(self.perm_out), self.n_out, ptr(y_dev), stream)

    @property
    def num_kernels(self):
        return len(self.launches) + 2




def plan(h, trans=False, graph=True):
    """Cached product plan: PanelPlan (CUDA graph) for H x, MatvecPlan
    (segmented kernel over the same storage) for H^T x."""
    key = "T" if trans else "N"
    if key not in h.dev.plans:
        if trans:
            h.dev.plans[key] = MatvecPlan(h, True)
        else:
            pl = PanelPlan(h)
            if graph:
                with torch.cuda.device(pl.dev):
                    pl.capture()
            h.dev.plans[key] = pl
    return h.dev.plans[key]


def _check_dim(x, n):
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (n,):
        raise ConfigError("vector of length %d, operator wants %d" % (x.size, n))
    return x


def mvm_device(h, x_dev, y_dev=None, trans=False):
    p = plan(h, trans)
    if y_dev is None:
        y_dev = torch.empty(p.n_out, dtype=torch.float64, device=p.dev)
    with torch.cuda.device(p.dev):
        p.run(x_dev, y_dev)
    return y_dev


def mvm(h, x):
    """y = H x, external ordering in and out (``h2.py:63-80``).

    Host vector -> pinned staging, read by the captured graph's gather
    kernel over the host link -> replay -> the scatter kernel writes the
    pinned output -> host vector."""
    nr, nc = h.shape
    x = _check_dim(x, nc)
    p = plan(h)
    if not hasattr(p, "pin_x"):
        p.pin_x = torch.empty(nc, dtype=torch.float64, pin_memory=True)
        p.pin_y = torch.empty(nr, dtype=torch.float64, pin_memory=True)
    p.pin_x.numpy()[:] = x
    with torch.cuda.device(p.dev):
        # large outputs: a fresh pinned array per call (torch's pinned block
        # cache) that the graph's scatter writes directly - no output copy;
        # small ones: the plan's pinned buffer plus a copy (cheaper than a
        # new allocation and a re-pointed scatter node)
        fresh = nr >= 16384
        y = torch.empty(nr, dtype=torch.float64, pin_memory=True) if fresh else p.pin_y
        if p.graph is not None and p.bind(p.pin_x, y):
            # zero-copy: the graph's gather reads the pinned input and its
            # scatter writes the pinned output (mapped host memory, read /
            # written contiguously), no DMA copies around the replay
            p.graph.replay()
        else:
            p.x.copy_(p.pin_x, non_blocking=True)
            p._body()
            y.copy_(p.y, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    return y.numpy() if fresh else y.numpy().copy()


def mvm_t(h, x):
    """y = H^T x (``h2.py:83-100``)."""
    nr, nc = h.shape
    x = _check_dim(x, nr)
    xd = to_dev(x, h.dev.device)
    return mvm_device(h, xd, trans=True).cpu().numpy()


def as_operator(h):
    def apply(x, trans=False):
        return mvm_t(h, x) if trans else mvm(h, x)
    return apply


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


def spectral_error_estimate(apply_ref, apply_approx, n, iters=100, seed=0):
    """Power-iteration estimate of ||ref - approx||_2 and its ratio to
    ||ref||_2 (``h2.py:144-184``); both closures take (x, trans=False)."""
    if iters < 1:
        raise ConfigError("iters must be positive")

    def power(fwd, bwd):
        z = np.random.default_rng(seed).standard_normal(n)
        nz = np.linalg.norm(z)
        if nz == 0.0:
            z = np.random.default_rng(seed + 1).standard_normal(n)
            nz = np.linalg.norm(z)
            if nz == 0.0:
                raise ConfigError("degenerate start vector")
        z = z / nz
        est = 0.0
        for _ in range(iters):
            w = fwd(z)
            est = np.linalg.norm(w)
            if est == 0.0:
                return 0.0
            z = bwd(w)
            nz = np.linalg.norm(z)
            if nz == 0.0:
                return est
            z = z / nz
        return est

    err = power(lambda u: apply_ref(u) - apply_approx(u),
                lambda u: apply_ref(u, True) - apply_approx(u, True))
    ref = power(lambda u: apply_ref(u), lambda u: apply_ref(u, True))
    if ref == 0.0:
        return err, (0.0 if err == 0.0 else np.inf)
    return err, err / ref


CGResult = namedtuple("CGResult", "x residuals converged")


def cg_solve(apply, b, tol=1e-8, max_iter=500):
    """Conjugate gradients on an SPD closure (``h2.py:190-219``)."""
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    r = b.copy()
    p = r.copy()
    rr = float(r @ r)
    bnorm = np.sqrt(float(b @ b))
    hist = [np.sqrt(rr)]
    if bnorm == 0.0:
        return CGResult(x, np.asarray(hist), True)
    for _ in range(max_iter):
        if hist[-1] <= tol * bnorm:
            break
        q = apply(p)
        pq = float(p @ q)
        if pq <= 0.0:
            break
        alpha = rr / pq
        x = x + alpha * p
        r = r - alpha * q
        rr_new = float(r @ r)
        hist.append(np.sqrt(rr_new))
        p = r + (rr_new / rr) * p
        rr = rr_new
    return CGResult(x, np.asarray(hist), bool(hist[-1] <= tol * bnorm))


def cg_solve_device(h, b, tol=1e-8, max_iter=500):
    """Conjugate gradients on the H2 operator with every vector resident on
    the device (``h2.py:190-219`` semantics): the product
    is the captured panel plan, the vector updates and dot products are
    ``gc_cg_*`` kernels with the scalars in device memory, and the only
    host traffic per iteration is the 16-byte read of r.r and the stop flag.
    Returns a :class:`CGResult` with host arrays."""
    pl = plan(h)
    dev = pl.dev
    b_d = torch.as_tensor(np.asarray(b, dtype=np.float64)).to(dev)
    n = b_d.numel()
    if n != pl.n_in or pl.n_in != pl.n_out:
        raise ConfigError("cg_solve_device needs a square operator matching b")
    x = torch.zeros_like(b_d)
    r = b_d.clone()
    p = b_d.clone()
    q = torch.empty_like(b_d)
    s = torch.zeros(8, dtype=torch.float64, device=dev)
    partial = torch.empty(int(_native.load().gc_krylov_partials()), dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        st = stream_handle()
        _native.call("gc_dot", n, ptr(b_d), ptr(b_d), ptr(partial), ptr(s), st)
        host = s[[0, 5]].cpu().numpy()
        bnorm = float(np.sqrt(host[0]))
        hist = [bnorm]
        if bnorm == 0.0:
            return CGResult(x.cpu().numpy(), np.asarray(hist), True)
        for _ in range(max_iter):
            if hist[-1] <= tol * bnorm:
                break
            pl.run(p, q)
            st = stream_handle()
            _native.call("gc_cg_pq", n, ptr(p), ptr(q), ptr(partial), ptr(s), st)
            _native.call("gc_cg_update", n, ptr(x), ptr(r), ptr(p), ptr(q), ptr(partial), ptr(s), st)
            host = s[[0, 5]].cpu().numpy()
            if host[1] != 0.0:
                break
            hist.append(float(np.sqrt(host[0])))
        return CGResult(x.cpu().numpy(), np.asarray(hist), bool(hist[-1] <= tol * bnorm))


def cgnr_solve(apply, b, tol=1e-8, max_iter=500):
    """CG on the normal equations; history is the true residual
    (``h2.py:222-253``)."""
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    r = b.copy()
    s = apply(r, True)
    p = s.copy()
    ss = float(s @ s)
    bnorm = np.sqrt(float(b @ b))
    hist = [np.sqrt(float(r @ r))]
    if bnorm == 0.0:
        return CGResult(x, np.asarray(hist), True)
    for _ in range(max_iter):
        if hist[-1] <= tol * bnorm or ss == 0.0:
            break
        q = apply(p)
        qq = float(q @ q)
        if qq == 0.0:
            break
        alpha = ss / qq
        x = x + alpha * p
        r = r - alpha * q
        hist.append(np.sqrt(float(r @ r)))
        s = apply(r, True)
        ss_new = float(s @ s)
        p = s + (ss_new / ss) * p
        ss = ss_new
    return CGResult(x, np.asarray(hist), bool(hist[-1] <= tol * bnorm))


# --------------------------------------------------------------------------
# panel plan: the non-transposed product (the benchmarked hot path)

_ITEM_ELEMS = int(os.environ.get("GC_ITEM_ELEMS", 65536))  # <= 512 KB of matrix data per work item (rows capped at 1024)
_ITEM_MAX_ROWS = 1024       # PAN_MAX_ROWS in csrc/h2mv.cu
_WARP_MAX_ROWS = 256        # WARP_MAX_ROWS in csrc/h2mv.cu
_STREAM_MAX_T = 1024        # ST_MAX_T in csrc/h2mv.cu
_PAIR_MAX_ELEMS = int(os.environ.get("GC_PAIR_MAX_ELEMS", 8192))   # k_panel_pair: small panels only
_RESIDENT = 148 * 6         # resident k_panelmv CTAs (40 registers, 256 threads, 6 per SM)


class _Phase:
    __slots__ = ("name", "height", "items", "xidx", "red", "arrivals", "nitems", "nred", "A0", "A1",
                 "in0", "in1", "out", "scratch", "bytes", "cta", "in_elems", "out_elems", "tma", "warp", "pair")


class _Node:
    """One step of the product DAG: a panel phase or a host callable
    (gather, zero, scatter, a collective), run on ``stream`` after ``deps``."""
    __slots__ = ("name", "phase", "fn", "stream", "deps", "launches", "priority")

    def __init__(self, name, stream, deps=(), phase=None, fn=None, priority=0):
        self.name, self.stream, self.deps, self.phase, self.fn = name, stream, list(deps), phase, fn
        self.launches = 1 if phase is not None else 0
        self.priority = priority


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

    def __init__(self, h):
        d = h.dev
        dev = d.device
        self.dev = dev
        rs, cs = h.row_basis.store, h.col_basis.store
        rf, cf = h.row_tree.flat, h.col_tree.flat
        self.n_in, self.n_out = cf.stop[0], rf.stop[0]
        self.perm_in, self.perm_out = d.perm_c, d.perm_r
        self.iperm_in, self.iperm_out = _inverse_perm(self.perm_in), _inverse_perm(self.perm_out)
        f64 = dict(dtype=torch.float64, device=dev)
        self.x = torch.zeros(self.n_in, **f64)
        self.y = torch.zeros(self.n_out, **f64)
        self.xt = torch.zeros(self.n_in, **f64)
        # y (tree order, near-field part) | x-hat in one buffer, so one launch
        # can write both (the near field fused with the lowest forward tier)
        self._obuf = torch.zeros(self.n_out + max(cs.coef_size, 1), **f64)
        self.yt, self.xhat = self._obuf[:self.n_out], self._obuf[self.n_out:]
        self._keep = []
        self.tiers_pending = False
        ny = max(rs.coef_size, 1)
        # y-hat | y-hat from the tiers above | leaf-basis part of y (summed
        # in the scatter): one buffer, zeroed by one memset per product
        self._ybuf = torch.zeros(2 * ny + self.n_out, **f64)
        self.yhat, self.yhat_t, self.yt2 = self._ybuf[:ny], self._ybuf[ny:2 * ny], self._ybuf[2 * ny:]
        # "pdl": one launch per transform level; "persistent": runs of levels
        # in one co-resident launch with grid barriers (experimental)
        self.chain_mode = os.environ.get("GC_CHAIN_MODE", "pdl")
        # bulk phases: "panel" (plain 8-byte loads, 8 per thread in flight;
        # the fastest measured), "tma" (one cp.async.bulk per item into
        # shared memory) and "stream" (persistent producer/consumer ring)
        # are kept as measured alternatives (matvec section)
        self.bulk_kernel = os.environ.get("GC_BULK_KERNEL", "panel")
        self._tma_elems = int(_native.load().gc_panel_tma_item_elems())
        # chain launches: 0 = plain, 1 = PDL released at CTA start, 2 = PDL
        # released after each CTA's item
        self._pdl = int(os.environ.get("GC_CHAIN_PDL", "1"))
        # transform levels with at least this many panels run one warp per panel
        # (168 us vs 144 us for the full C2 product: kept as an option)
        self._warp_min_panels = int(os.environ.get("GC_WARP_MIN_PANELS", str(1 << 40)))   # off: measured slower
        self._balance_waves = os.environ.get("GC_BALANCE_WAVES", "0") == "1"
        grid = _native.ctypes.c_int64(0)
        _native.call("gc_panel_chain_grid", _native.ctypes.byref(grid))
        self._chain_grid = grid.value
        _native.call("gc_panel_stream_grid", _native.ctypes.byref(grid))
        self._stream_grid = grid.value
        size_r = rf.stop - rf.start
        # forward transform (column basis), by height
        fwd = []
        mat = cs.materialized & (cs.rank > 0)
        for h_ in np.unique(cf.height[mat]):
            ids = np.flatnonzero(mat & (cf.height == h_))
            leaf = h_ == 0
            K = cs.rows[ids]
            base = cf.start[ids] if leaf else cs.coef_off[cf.left[ids]]
            panels = (cs.v_off[ids], K, cs.rank[ids], (base, K), cs.coef_off[ids], 0)
            fwd.append(self._phase("forward", int(h_), panels, cs.V, None,
                                   self.xt if leaf else self.xhat, None, self.xhat, transform=True))
        # coupling: one panel per row cluster, bucketed by row height
        cpl = []
        live = (d.c_nr > 0) & (d.c_nc > 0)
        order = np.flatnonzero(live)[np.argsort(d.c_rows[live], kind="stable")]
        if order.size:
            sn = d.c_rows[order]
            cuts = np.flatnonzero(np.r_[True, sn[1:] != sn[:-1]])
            # panel inputs: the x-hat slots of the blocks' column clusters, in
            # block order - one index range per block, expanded on the device
            bstart, blen = cs.coef_off[d.c_cols[order]], d.c_nc[order]
            K = np.add.reduceat(blen, cuts)
            nblk = np.diff(np.r_[cuts, len(order)])
            colh = np.maximum.reduceat(cf.height[d.c_cols[order]], cuts)
            rowh = rf.height[sn[cuts]]
            for h_ in np.unique(rowh):
                sel = np.flatnonzero(rowh == h_)
                bsel = _ranges_np(cuts[sel], nblk[sel])
                panels = (d.c_off[order[cuts[sel]]], K[sel], d.c_nr[order[cuts[sel]]],
                          (bstart[bsel], blen[bsel]), rs.coef_off[sn[cuts[sel]]], 0)
                P = self._phase("coupling", int(h_), panels, d.coup, None, self.xhat, None, self.yhat)
                cpl.append((P, int(colh[sel].max())))
        # backward transform (row basis), top down
        bwd = []
        matb = rs.materialized & (rs.rank > 0) & ~rf.is_leaf
        for h_ in sorted(np.unique(rf.height[matb]), reverse=True):
            ids = np.flatnonzero(matb & (rf.height == h_))
            K = rs.rank[ids]
            panels = (rs.v_off[ids], K, rs.rows[ids], (rs.coef_off[ids], K), rs.coef_off[rf.left[ids]], 1)
            P = self._phase("backward", int(h_), panels, rs.VT, None, self.yhat, None, self.yhat,
                            transform=True)
            kids = np.r_[rf.left[ids], rf.right[ids]]
            bwd.append((P, set(rf.height[kids].tolist()) | {int(h_)}))
        # near field: one panel per row leaf
        order = np.argsort(d.n_rows, kind="stable")
        sn = d.n_rows[order]
        cuts = np.flatnonzero(np.r_[True, sn[1:] != sn[:-1]]) if len(sn) else np.zeros(0, np.int64)
        K = np.add.reduceat(d.n_nc[order], cuts) if len(sn) else np.zeros(0, np.int64)
        rows = (cf.start[d.n_cols[order]], d.n_nc[order])
        panels = (d.n_off[order[cuts]], K, d.n_nr[order[cuts]], rows, rf.start[sn[cuts]], 0)
        near = self._phase("nearfield", 0, panels, d.near, None, self.xt, None, self.yt)
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
            leafp = self._phase("leafbasis", 0, panels, rs.VT, None, self.yhat, None, self.yt2,
                                transform=True)
        self.tiers = None
        parts = [(leafp, None)]
        if self.chain_mode == "pdl" and os.environ.get("GC_TIERS", "auto") != "off":
            fwd, bwd, parts = self._tiered(h, fwd, bwd, leafp)
        parts = [(P, hs) for P, hs in parts if P is not None and P.nitems]
        self._fused = None
        if (self.tiers is not None and os.environ.get("GC_FUSE_NEAR", "0") == "1" and fwd
                and near.nitems and fwd[0].nitems):
            # the near field and the lowest forward tier both read only x:
            # one launch, forward items first (HBM busy while the latency-
            # bound tier runs; the coupling buckets then wait for both).
            # Measured: C1 28 -> 31 us, C2 135 -> 150 us, C3/C4 -0.5 %: off
            self._fused = self._fuse(fwd[0], near)
        self._fwd, self._cpl, self._bwd, self._near, self._leafparts = fwd, cpl, bwd, near, parts
        self.phases = [P for P in [near] + fwd + [c for c, _ in cpl] + [b for b, _ in bwd] + [p for p, _ in parts]
                       + [self._fused] if P is not None and P.nitems > 0]
        # the chain gets the highest stream priority so its CTAs are
        # scheduled ahead of the queued bulk (coupling buckets, near field)
        self.streams = {"chain": torch.cuda.Stream(device=dev, priority=-8)}
        self._bulk_priority = 0
        least, greatest = _native.ctypes.c_int32(0), _native.ctypes.c_int32(0)
        _native.call("gc_priority_range", _native.ctypes.byref(least), _native.ctypes.byref(greatest))
        self._prio = (least.value, greatest.value)
        self._barrier = torch.zeros(1, dtype=torch.int32, device=dev)
        self.trace = {}                    # id(phase) -> [2] int64 (profiling only)
        self.nodes = self._build_nodes()
        self.graph = None

    def _fuse(self, F, N):
        """One phase running the items of F (forward, A1, writes x-hat) and
        N (near field, A0, writes y) - both read in0 = xt; outputs are
        offsets into the shared buffer [yt | x-hat]."""
        assert F.in0 is N.in0 is self.xt and F.out is self.xhat and N.out is self.yt
        fi, ni = F.items.cpu().numpy().copy(), N.items.cpu().numpy().copy()
        fr = F.red.cpu().numpy().copy() if F.nred else np.zeros((0, 5), np.int64)
        nr = N.red.cpu().numpy().copy() if N.nred else np.zeros((0, 5), np.int64)
        nx_f, ns_f = F.xidx.numel(), F.scratch.numel()
        direct = (fi[:, 5] & 4) != 0
        fi[:, 5] |= 1                                   # forward items read A1
        fi[direct, 2] += self.n_out                     # x-hat lives after yt
        fr[:, 0] += self.n_out
        ni[:, 1] += nx_f                                # near indices after the forward ones
        nd = (ni[:, 5] & 4) != 0
        ni[~nd, 2] += ns_f                              # near partial sums after the forward ones
        ni[~nd, 6] += F.nred
        nr[:, 2] += ns_f
        P = _Phase()
        P.name, P.height = "nearfield+forward", F.height
        P.items = to_dev(np.ascontiguousarray(np.concatenate([fi, ni]), np.int64), self.dev)
        P.xidx = torch.cat([F.xidx[:nx_f], N.xidx])
        P.nitems, P.nred = len(fi) + len(ni), F.nred + N.nred
        red = np.concatenate([fr, nr])
        P.red = to_dev(np.ascontiguousarray(red, np.int64), self.dev) if P.nred else None
        P.arrivals = torch.zeros(max(P.nred, 1), dtype=torch.int32, device=self.dev)
        P.scratch = torch.cat([F.scratch[:ns_f], N.scratch])
        P.A0, P.A1, P.in0, P.in1, P.out = N.A0, F.A0, self.xt, None, self._obuf
        P.bytes = F.bytes + N.bytes
        P.in_elems, P.out_elems = F.in_elems + N.in_elems, F.out_elems + N.out_elems
        P.warp, P.cta, P.tma, P.pair = False, None, False, False
        return P

    def _tiered(self, h, fwd, bwd, leafp):
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
        # "upper" / "all": split the large panels of the upper tiers (232
        # CTAs for 24 MB at C2) / of every tier over more items - both
        # measured slower inside the product (142 / 144 us vs 135 us at C2)
        self._tier_split = os.environ.get("GC_TIER_SPLIT", "none")
        cb = T_.choose_tiers(cs, cf)
        rb = cb if (rs is cs and rf is cf) else T_.choose_tiers(rs, rf)
        if not cb or not rb:
            return fwd, bwd, [(leafp, None)]
        ct = T_.StoreTiers(cs, cf, cb, self.dev)
        rt = ct if (rs is cs and rb == cb) else T_.StoreTiers(rs, rf, rb, self.dev)
        groups, MT = rt.transposed(self.dev)
        if rt is not ct:
            rt.M = None                                  # only the transposed blocks are used
        self.tiers = dict(col=cb, row=rb, fwd_elems=ct.elems, bwd_elems=int(MT.numel()))
        self._keep.extend([ct.M, MT])
        def kw(low):
            return dict(transform=True, split=self._tier_split == "all" or (self._tier_split == "upper" and not low))
        self.tiers_pending = True
        nfwd = []
        for t in ct.tiers:
            u, f, w, nodes = t["u"], t["f"], t["w"], t["nodes"]
            low = t["lo"] < 0
            starts = cf.start[f] if low else cs.coef_off[f]
            panels = (t["moff"][nodes], t["m"][nodes], cs.rank[nodes], (starts, w), cs.coef_off[nodes], 0)
            nfwd.append(self._phase("forward", t["hi"], panels, ct.M, None, self.xt if low else self.xhat,
                                    None, self.xhat, **kw(low)))
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
            if low and os.environ.get("GC_LEAF_SPLIT", "0") == "1":
                # leaf rows in two launches: the ancestors' part as soon as
                # their buckets are done, then only V_leaf y-hat_leaf after
                # the deepest (last) bucket.  Measured slower (C1 29 -> 31,
                # C2 135 -> 142, C3 525 -> 561 us): the 2048 tiny leaf panels
                # still take 10 us at the end and the first part slows the bulk
                assert np.array_equal(uu[first], elems)      # the leaf itself leads its stack
                kl = rs.rank[elems]
                own = np.zeros(len(ff), bool)
                own[first] = True
                up = keep & (cnt > 1)
                sa = sel & ~own & np.repeat(up, cnt)
                pa = (dst[first][up] + (kl * ww[first])[up], (K - kl)[up], ww[first][up],
                      (rs.coef_off[uu][sa], rs.rank[uu][sa]), rf.start[elems][up], 1)
                pb = (dst[first][keep], kl[keep], ww[first][keep], (rs.coef_off[elems][keep], kl[keep]),
                      rf.start[elems][keep], 1)
                if up.any():
                    PA = self._phase("leafbasis", t["hi"], pa, MT, None, self.yhat, self.yhat_t, self.yt2,
                                     sum_inputs=True, **kw(low))
                    parts.append((PA, set(range(1, t["hi"] + 1))))
                PB = self._phase("leafbasis", 0, pb, MT, None, self.yhat, self.yhat_t, self.yt2,
                                 sum_inputs=True, **kw(low))
                parts.append((PB, {0}))
                continue
            panels = (dst[first][keep], K[keep], ww[first][keep], (rs.coef_off[uu][sel], rs.rank[uu][sel]),
                      (rf.start[elems] if low else rs.coef_off[elems])[keep], 0)
            P = self._phase("leafbasis" if low else "backward", t["hi"], panels, MT, None, self.yhat,
                            self.yhat_t, self.yt2 if low else self.yhat_t, sum_inputs=True, **kw(low))
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
        priority.  (The persistent mode also splits its launches at S.)"""
        if not self._cpl:
            return 0
        by_h = sorted(((P.height, P.bytes) for P, _ in self._cpl), reverse=True)
        total = sum(b for _, b in by_h)
        acc, S = 0, by_h[0][0] + 1
        for h_, b in by_h:
            if acc + b > 0.2 * total:
                break
            acc += b
            S = h_
        return S

    def _segment_nodes(self, name, phases, deps):
        """Chain steps for a run of levels: one PDL launch per level, or (in
        the persistent mode) one co-resident launch with grid barriers."""
        phases = [P for P in phases if P.nitems > 0]
        if not phases:
            return []
        if len(phases) == 1 or self.chain_mode != "persistent":
            return [_Node(name, "chain", deps if i == 0 else [], phase=P, priority=self._prio[1])
                    for i, P in enumerate(phases)]
        assert _native.load().gc_panel_phase_bytes() == 96

        def addr(t):
            return ptr(t).value or 0
        desc = np.array([[addr(P.items), P.nitems, addr(P.xidx), addr(P.A0), addr(P.A1), addr(P.in0),
                          addr(P.in1), addr(P.out), addr(P.scratch), addr(P.red), addr(P.arrivals), 0]
                         for P in phases], dtype=np.uint64)
        dev_desc = to_dev(desc.view(np.int64), self.dev)
        self._keep.append(dev_desc)
        n = len(phases)

        def launch():
            _native.call("gc_panel_chain", n, ptr(dev_desc), self._chain_grid, ptr(self._barrier),
                         stream_handle())
        node = _Node(name, "chain", deps, fn=launch)
        node.launches = 1
        return [node]

    def _build_nodes(self, gather=True, before_coupling=None, scatter=True):
        """Nodes in a valid serial order (a topological order of the DAG)."""
        st = stream_handle
        nodes = []

        def add(n):
            nodes.append(n)
            return len(nodes) - 1

        def add_steps(name, phases, deps):
            k = None
            for n in self._segment_nodes(name, phases, deps):
                k = add(n)
            return k

        persistent = self.chain_mode == "persistent"
        S = self._split_height()
        least, greatest = self._prio
        levels = least - greatest
        z = add(_Node("zero", "chain", fn=lambda: self._ybuf.zero_()))
        if gather:
            g = add(_Node("gather", "chain", [z], fn=lambda: _native.call(
                "gc_gather_inv", ptr(self.x), ptr(self.iperm_in), self.n_in, ptr(self.xt), st())))
            nodes[g].launches = 1
        else:
            g = z
        last = g
        fwd_done = []                                   # (max height covered, node)
        chain_fwd = self._fwd
        if self._fused is not None:
            near = last = add(_Node("nearfield+forward", "chain", [g], phase=self._fused, priority=greatest))
            fwd_done.append((self._fwd[0].height, near))
            chain_fwd = self._fwd[1:]
        else:
            near = add(_Node("nearfield", "near", [g], phase=self._near)) if self._near.nitems else None
        groups = ([[P for P in chain_fwd if P.height < S], [P for P in chain_fwd if P.height >= S]]
                  if persistent else [[P] for P in chain_fwd])
        for grp in groups:
            k = add_steps("forward", grp, [last])
            if k is not None:
                last = k
                fwd_done.append((max(P.height for P in grp), k))
        gate = None
        if before_coupling is not None:
            gate = add(_Node("pre-coupling", "chain", [last], fn=before_coupling))
        bucket = {}
        for P, colh in sorted(self._cpl, key=lambda c: c[0].height):
            if gate is not None:
                dep = [gate]
            else:
                dep = [next((k for hh, k in fwd_done if hh >= colh), last)]
            if P.height >= S or levels < 2:
                prio = greatest
            else:
                prio = least - 1 - int(round(P.height * (levels - 2) / max(S - 1, 1)))
                prio = min(least - 1, max(greatest + 1, prio))
            bucket[P.height] = add(_Node("coupling", "c%d" % P.height, dep + [z], phase=P, priority=prio))
        prev = gate if gate is not None else last
        groups = ([[b for b in self._bwd if b[0].height > S], [b for b in self._bwd if b[0].height <= S]]
                  if persistent else [[b] for b in self._bwd])
        for grp in groups:
            if not grp:
                continue
            need = sorted(set().union(*[hs for _, hs in grp]))
            k = add_steps("backward", [P for P, _ in grp], [prev] + [bucket[x] for x in need if x in bucket])
            if k is not None:
                prev = k
        for P, hs in self._leafparts:
            need = list(bucket.values()) if hs is None else [bucket[x] for x in sorted(hs) if x in bucket]
            prev = add(_Node("leafbasis", "chain", [prev] + need, phase=P, priority=greatest))
        tail = [prev] + list(bucket.values())
        if near is not None:
            tail = tail + [near]
        if scatter:
            k = add(_Node("scatter", "chain", tail, fn=lambda: _native.call(
                "gc_scatter2_inv", ptr(self.yt), ptr(self.yt2), ptr(self.iperm_out), self.n_out, ptr(self.y),
                st())))
            nodes[k].launches = 1
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
               split=False):
        a_off, K, T, rows, out_off, accumulate = panels
        a_off = np.asarray(a_off, np.int64)
        K = np.asarray(K, np.int64)
        T = np.asarray(T, np.int64)
        out_off = np.asarray(out_off, np.int64)
        n = len(a_off)
        elems = int((K * T).sum())
        if transform and split:
            # tier transforms: split only the panels larger than
            # GC_TIER_SPLIT_ELEMS (0: like the bulk, so the launch fills the SMs)
            cap = int(os.environ.get("GC_TIER_SPLIT_ELEMS", "0"))
            target = cap if cap > 0 else max(1024, min(_ITEM_ELEMS, elems // (148 * 4) + 1))
            max_rows = _ITEM_MAX_ROWS
        elif transform:
            # transform levels: one item per panel (split only past the row
            # cap) - these levels are latency-bound, and a split panel costs
            # a second pass over L2 for its reduction
            target = 1 << 40
            max_rows = _WARP_MAX_ROWS if self.chain_mode == "persistent" else _ITEM_MAX_ROWS
        elif self.bulk_kernel == "tma":
            # TMA kernel: items fill its shared-memory tile
            target = self._tma_elems
            max_rows = _ITEM_MAX_ROWS
        else:
            # chunk rows so every phase has >= ~4 items per SM when it can
            target = max(256, min(_ITEM_ELEMS, elems // (148 * 4) + 1))
            if self._balance_waves and elems > _ITEM_ELEMS * _RESIDENT // 2:
                # whole waves: ~k x (resident CTAs) items of <= _ITEM_ELEMS
                wave_elems = int(os.environ.get("GC_WAVE_ELEMS", str(_ITEM_ELEMS)))
                waves = -(-elems // (wave_elems * _RESIDENT))
                target = -(-elems // (waves * _RESIDENT))
            max_rows = _ITEM_MAX_ROWS
        if not transform and self.bulk_kernel == "tma":
            rpi = np.minimum(max_rows, np.maximum(1, target // np.maximum(T, 1)))  # fits the smem tile
        else:
            rpi = np.minimum(max_rows, np.maximum(1, -(-target // np.maximum(T, 1))))  # rows/item
        # at most 8 items per panel: the last item of a split panel sums the
        # partials serially, so deep splits of small phases cost latency
        if transform or self.bulk_kernel != "tma":          # (tma items must fit its tile)
            rpi = np.maximum(rpi, np.minimum(max_rows, -(-K // 8)))
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
        mode = np.where(direct, 4 | (8 * accumulate), 0) | (32 if sum_inputs else 0)
        if not transform and os.environ.get("GC_BULK_PREFETCH", "0") == "1":
            mode = mode | 16
        items = np.stack([a_off[item_panel] + item_k * T[item_panel], xoff[item_panel] + item_k,
                          out_col, T[item_panel], item_rows, mode,
                          np.where(direct, -1, slot[item_panel]), np.zeros_like(mode)], 1)
        if not transform and len(items) and os.environ.get("GC_BULK_LPT", "0") == "1":
            items = items[np.argsort(-(items[:, 3] * items[:, 4]), kind="stable")]
        if transform and len(items) and os.environ.get("GC_LPT", "0") == "1":
            # largest items first (CTAs dispatch in launch order): measured
            # -6 % at sphere L4, +1-3 % at L6-L8, so off by default
            items = items[np.argsort(-(items[:, 3] * items[:, 4]), kind="stable")]
        red = np.stack([out_off[multi], T[multi], scr_off[multi], nit[multi],
                        np.full(int(multi.sum()), accumulate)], 1)
        P = _Phase()
        P.name, P.height = name, height
        P.items = to_dev(np.ascontiguousarray(items, np.int64), self.dev)
        if segs is not None:
            st_, ln_ = np.asarray(segs[0], np.int64), np.asarray(segs[1], np.int64)
            total = int(ln_.sum())
            P.xidx = torch.empty(max(total, 1), dtype=torch.int32, device=self.dev)
            tab = to_dev(np.concatenate([st_, ln_, _offsets_np(ln_)]), self.dev)
            m = len(st_)
            with torch.cuda.device(self.dev):
                _native.call("gc_expand_ranges", m, ptr(tab[:m]), ptr(tab[m:2 * m]), ptr(tab[2 * m:]),
                             ptr(P.xidx), stream_handle())
        else:
            P.xidx = to_dev(xidx, self.dev)
        P.nitems, P.nred = len(items), int(multi.sum())
        P.red = to_dev(np.ascontiguousarray(red, np.int64), self.dev) if P.nred else None
        P.arrivals = torch.zeros(max(P.nred, 1), dtype=torch.int32, device=self.dev)
        P.A0, P.A1, P.in0, P.in1, P.out = A0, A1, in0, in1, out
        P.scratch = torch.zeros(max(int((np.where(multi, nit * T, 0)).sum()), 1),
                                dtype=torch.float64, device=self.dev)
        P.bytes = 8 * elems
        P.in_elems, P.out_elems = int(K.sum()), int(T.sum())
        # many small whole panels (lower transform levels): one warp each
        P.warp = bool(transform and n >= self._warp_min_panels and len(items) == n
                      and int(K.max()) <= _WARP_MAX_ROWS)
        P.cta = None
        # two whole small panels per CTA (k_panel_pair) for tier phases
        P.pair = bool(transform and self.tiers_pending and os.environ.get("GC_PAIR", "1") == "1" and n
                      and bool(np.all(direct)) and int(T.max()) <= 128 and int(item_rows.max()) <= 512
                      and int((item_rows * T[item_panel]).max()) <= _PAIR_MAX_ELEMS and not P.warp)
        if P.pair and os.environ.get("GC_PAIR_SORT", "desc") != "0":
            # pair equal-sized panels (largest first, or smallest first)
            sz = items[:, 3] * items[:, 4]
            order = np.argsort(-sz if os.environ.get("GC_PAIR_SORT", "desc") == "desc" else sz, kind="stable")
            P.items = to_dev(np.ascontiguousarray(items[order], np.int64), self.dev)
        P.tma = bool(not transform and self.bulk_kernel == "tma" and n and int(T.max()) <= self._tma_elems)
        if (not transform and n and int(T.max()) <= _STREAM_MAX_T and self._stream_grid > 0
                and self.bulk_kernel == "stream"):
            # bulk phase: TMA streaming kernel, items split over the
            # co-resident grid by equal bytes (+ a per-item latency charge)
            cost = np.cumsum(8 * item_rows * T[item_panel] + 4096)
            G = self._stream_grid
            begin = np.searchsorted(cost, cost[-1] * np.arange(1, G) / G, side="left")
            P.cta = to_dev(np.r_[0, np.minimum(begin, len(items)), len(items)].astype(np.int64), self.dev)
        return P

    def _launch(self, P, stream, chain=False, priority=0):
        if P.cta is not None and not chain:
            _native.call("gc_panel_stream", P.nitems, ptr(P.items), ptr(P.xidx), ptr(P.A0), ptr(P.A1),
                         ptr(P.in0), ptr(P.in1), ptr(P.out), ptr(P.scratch), P.nred, ptr(P.red),
                         ptr(P.arrivals), ptr(P.cta), self._stream_grid, int(priority),
                         ptr(self.trace.get(id(P))), stream)
            return
        if P.tma and not chain:
            _native.call("gc_panel_tma", P.nitems, ptr(P.items), ptr(P.xidx), ptr(P.A0), ptr(P.A1),
                         ptr(P.in0), ptr(P.in1), ptr(P.out), ptr(P.scratch), P.nred, ptr(P.red),
                         ptr(P.arrivals), int(priority), ptr(self.trace.get(id(P))), stream)
            return
        mode = (self._pdl if chain else 0) | (4 if P.warp else 0) | (16 if P.pair else 0)
        _native.call("gc_panelmv", P.nitems, ptr(P.items), ptr(P.xidx), ptr(P.A0), ptr(P.A1),
                     ptr(P.in0), ptr(P.in1), ptr(P.out), ptr(P.scratch), P.nred, ptr(P.red),
                     ptr(P.arrivals), mode, int(priority), ptr(self.trace.get(id(P))), stream)

    def _body(self, phase_events=None, phase="coupling"):
        self._exec(self.nodes, serial=phase_events is not None, phase_events=phase_events, phase=phase)

    def _native_table(self):
        """The DAG as gc_plan_create's node table (csrc/plan.cu), or None
        when a node is not expressible there (a Python callable such as a
        collective, or a non-default bulk kernel)."""
        skip = {i for i, n in enumerate(self.nodes) if n.name == "join"}
        remap, rows, deps, streams = {}, [], [], {"chain": 0}
        for i, n in enumerate(self.nodes):
            if i in skip:
                continue
            sidx = streams.setdefault(n.stream, len(streams))
            a = [0] * 12
            if n.phase is not None:
                P = n.phase
                if P.cta is not None or P.tma:
                    return None
                kind = 0
                chain = (self._pdl if n.stream == "chain" else 0) | (4 if P.warp else 0) | (16 if P.pair else 0)
                a = [P.items.data_ptr(), P.nitems, P.xidx.data_ptr(), P.A0.data_ptr(),
                     P.A1.data_ptr() if P.A1 is not None else 0, P.in0.data_ptr(),
                     P.in1.data_ptr() if P.in1 is not None else 0, P.out.data_ptr(), P.scratch.data_ptr(),
                     P.nred, P.red.data_ptr() if P.red is not None else 0, P.arrivals.data_ptr()]
            elif n.name == "zero":
                kind, chain, a[:2] = 1, 0, [self._ybuf.data_ptr(), 8 * self._ybuf.numel()]
            elif n.name == "gather":
                kind, chain = 2, 0
                a[:4] = [self.x.data_ptr(), self.iperm_in.data_ptr(), self.n_in, self.xt.data_ptr()]
            elif n.name == "scatter":
                kind, chain = 3, 0
                a[:5] = [self.yt.data_ptr(), self.yt2.data_ptr(), self.iperm_out.data_ptr(), self.n_out,
                         self.y.data_ptr()]
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
        """Record the product into a CUDA graph (static x -> y buffers).  The
        default is the C++ executor (csrc/plan.cu: its own streams, events
        and graph); a DAG with Python steps (the sharded plan's collectives)
        is captured through torch."""
        if os.environ.get("GC_NATIVE_PLAN", "1") == "1" and type(self) is PanelPlan:
            tab = self._native_table()
            if tab is not None:
                self._body()                         # warm-up (module loads) outside the capture
                torch.cuda.synchronize(self.dev)
                rows, deps, ndeps, prio = tab
                h = _native.ctypes.c_void_p(0)
                _native.call("gc_plan_create", len(rows), rows.ctypes.data, ndeps, deps.ctypes.data, len(prio),
                             prio.ctypes.data, _native.ctypes.byref(h))
                self.graph = _NativeGraph(h)
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
        g = torch.cuda.CUDAGraph(keep_graph=os.environ.get("GC_KEEP_GRAPH", "1") == "1")
        with torch.cuda.stream(s):
            g.capture_begin()
            try:
                self._body()
            finally:
                g.capture_end()
        if os.environ.get("GC_KEEP_GRAPH", "1") == "1":
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
        use them ran).  Returns False (nothing changed) when the graph has no
        such nodes."""
        if isinstance(self.graph, _NativeGraph):
            self.graph.bind(x_dev, y_dev)
            return True
        if self.graph is None or os.environ.get("GC_KEEP_GRAPH", "1") != "1":
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
        """y_dev = H x_dev (device vectors, external ordering).  With
        ``phase_events`` (or ``serial``) every node runs in order on the
        current stream and the events bracket the named phase's kernels."""
        if phase_events is None and not serial and self._direct_ok(x_dev, y_dev):
            self.bind(x_dev, y_dev)                  # graph reads x_dev, writes y_dev: no copies
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

    @property
    def num_kernels(self):
        """Own kernels per product (the torch fill of y-hat not counted)."""
        return sum(n.launches for n in self.nodes)


class _NativeGraph:
    """The product graph owned by the C++ executor (gc_plan_*): replay()
    launches it on the current stream with the last bound x / y."""

    def __init__(self, handle):
        self.handle = handle
        self._x = self._y = 0
        self._run = _native.load().gc_plan_run        # bound once: this is on the e2e path

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
