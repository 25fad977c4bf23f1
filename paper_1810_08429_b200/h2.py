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

from collections import namedtuple

import numpy as np

from . import _native
from .device import empty, ptr, stream_handle, to_dev, torch
from .errors import ConfigError

__all__ = ["mvm", "mvm_t", "as_operator", "storage_report", "storage_csv_rows",
           "spectral_error_estimate", "cg_solve", "cgnr_solve", "CGResult", "MatvecPlan"]


class _Launch:
    __slots__ = ("seg", "blk", "nseg", "A0", "A1", "in0", "in1", "out", "acc", "maxT")


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
                          self.xhat, 0)

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
            self._add(seg, blk, d.coup, None, self.xhat, None, self.yhat, 0)

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
            self._add(seg, blk, bwdA, None, self.yhat, None, self.yhat, 1)

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
        self._add(seg, bl, d.near, leafA, self.xt, self.yhat, self.yt, 0)

    def _add(self, seg, blk, A0, A1, in0, in1, out, acc):
        if len(seg) == 0:
            return
        L = _Launch()
        L.seg = to_dev(np.ascontiguousarray(seg, dtype=np.int64), self.dev)
        L.blk = to_dev(np.ascontiguousarray(blk, dtype=np.int64).reshape(-1, 6), self.dev) \
            if len(blk) else torch.zeros(6, dtype=torch.int64, device=self.dev)
        L.nseg = len(seg)
        L.A0, L.A1, L.in0, L.in1, L.out, L.acc = A0, A1, in0, in1, out, acc
        L.maxT = int(np.max(seg[:, 1]))
        self.launches.append(L)

    def run(self, x_dev, y_dev):
        """y_dev = H x_dev (or H^T) for device vectors in external order."""
        stream = stream_handle()
        _native.call("gc_gather", ptr(x_dev), ptr(self.perm_in), self.n_in, ptr(self.xt), stream)
        self.yhat.zero_()
        for L in self.launches:
            _native.call("gc_segmv", L.nseg, ptr(L.seg), ptr(L.blk), ptr(L.A0), ptr(L.A1),
                         ptr(L.in0), ptr(L.in1), ptr(L.out), L.acc, L.maxT, stream)
        _native.call("gc_scatter", ptr(self.yt), ptr(self.perm_out), self.n_out, ptr(y_dev), stream)

    @property
    def num_kernels(self):
        return len(self.launches) + 2


def plan(h, trans=False):
    key = "T" if trans else "N"
    if key not in h.dev.plans:
        h.dev.plans[key] = MatvecPlan(h, trans)
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
    """y = H x, external ordering in and out (``h2.py:63-80``)."""
    nr, nc = h.shape
    x = _check_dim(x, nc)
    xd = to_dev(x, h.dev.device)
    return mvm_device(h, xd).cpu().numpy()


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
