"""GCA-H2 construction on the device: nested cluster bases and H2 assembly.

Host-side mirror of the hot-path part of ``greencross/gca.py``:
``aca_interpolation`` (``:41-79``), ``BasisNode`` / ``ClusterBasis``
(``:92-146``), ``coupling_marks`` (``:149-159``), ``build_cluster_basis``
(``:162-220``), ``expand_basis`` (``:223-227``), ``H2Matrix`` and
``build_h2`` (``:230-312``).

The reference builds bases by recursion (one factor + one ACA per node).
Here the materialised forest is processed level-synchronously by height
(SPEC.md:500-501): one ``gc_green_box_rules`` + ``gc_green_factor`` +
``gc_aca`` launch per level over every node of that level; the next
level's row lists (the children's pivots) are gathered on the device
(``csrc/bases.cu``) and the host reads only each level's row totals.  ``build_h2`` assembles every coupling and near-field
block with two ``gc_assemble_blocks`` launches plus the singular flush;
values stay in HBM in the matvec layout (``h2.py``) and reach the host only
through the lazy ``.values`` / ``.v`` / ``.transfer`` views.
"""

import threading
import time
import weakref
from collections import namedtuple
from collections.abc import Sequence

import numpy as np

from . import _native
from .assembly import device_block_assembly, resolve_counts
from .device import (DeviceMesh, DeviceRules, SingularQueue, check_mesh, empty, padded_copy,
                     padded_empty, ptr, require_device, stream_handle, to_dev, torch)
from .errors import ConfigError, GeometryError
from .quadrature import _gauss01

__all__ = ["Interpolation", "aca_interpolation", "BasisNode", "ClusterBasis",
           "build_cluster_basis", "expand_basis", "CouplingBlock", "NearfieldBlock",
           "H2Matrix", "build_h2", "coupling_marks"]

Interpolation = namedtuple("Interpolation", "pivots v")
CouplingBlock = namedtuple("CouplingBlock", "row col values")
NearfieldBlock = namedtuple("NearfieldBlock", "row col values")


def _offsets(sizes):
    sizes = np.asarray(sizes, dtype=np.int64)
    return np.cumsum(sizes) - sizes


def _grouped_offsets(keys, sizes, with_order=False):
    """Offsets that store items with equal key contiguously (keys ascending,
    original order inside a key); ``with_order``: also the storage order
    (the item indices by ascending offset)."""
    order = np.argsort(keys, kind="stable")
    off = np.empty(len(keys), dtype=np.int64)
    off[order] = _offsets(np.asarray(sizes, dtype=np.int64)[order])
    return (off, order) if with_order else off


# --------------------------------------------------------------------------
# ACA on one matrix (API parity with gca.aca_interpolation)

def aca_interpolation(a, eps, max_rank=None, device=None):
    """Full-pivot cross approximation of a thin matrix on the device
    (``gca.py:41-79``).  ``v[pivots] == I`` exactly."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    n, w = a.shape
    dev = require_device(device)
    limit = min(n, w if max_rank is None else int(max_rank))
    fac = to_dev(a.ravel(), dev)
    cap = max(n * max(limit, 0), 1)
    v = empty(cap, dev)
    u = empty(cap, dev)
    piv = torch.zeros(max(limit, 1), dtype=torch.int64, device=dev)
    rank = torch.zeros(1, dtype=torch.int64, device=dev)
    desc = to_dev(np.array([[0, n, 0, 0]], dtype=np.int64), dev)
    mr = limit if max_rank is not None else 0
    if max_rank is not None and limit <= 0:
        return Interpolation(np.zeros(0, dtype=np.intp), np.zeros((n, 0)))
    with torch.cuda.device(dev):
        _native.call("gc_aca", 1, ptr(desc), w, float(eps), mr, ptr(fac), ptr(piv), ptr(rank),
                     ptr(v), ptr(u), n, stream_handle())
    r = int(rank.item())
    pivots = piv.cpu().numpy()[:r].astype(np.intp)
    if r == 0:
        return Interpolation(pivots, np.zeros((n, 0)))
    return Interpolation(pivots, v[:n * r].cpu().numpy().reshape(n, r))


# --------------------------------------------------------------------------
# nested bases

class BasisNode:
    """Per-cluster basis content (``gca.py:92-121``): leaves carry ``v``
    (size x rank), every non-root node its ``transfer`` (rank x parent
    rank); ``pivots`` are global dof indices.  ``v`` and ``transfer`` are
    host views of the device store, copied on first access."""

    __slots__ = ("cluster", "pivots", "_children", "_kids", "_store", "_slot", "_v", "_transfer")

    def __init__(self, cluster, pivots, children, store, slot, kids=None):
        self.cluster = cluster
        self.pivots = pivots
        self._children = children
        self._kids = kids              # lazy: slot -> children tuple
        self._store, self._slot = store, slot
        self._v = None
        self._transfer = None

    @property
    def children(self):
        if self._children is None:
            self._children = self._kids(self._slot)
        return self._children

    @children.setter
    def children(self, value):
        self._children = value

    @property
    def rank(self):
        return len(self.pivots)

    @property
    def v(self):
        if self._v is None and not self.children and self._store is not None:
            self._v = self._store.host_matrix(self.cluster.index)
        return self._v

    @v.setter
    def v(self, value):
        self._v = value

    @property
    def transfer(self):
        if self._transfer is None and self._store is not None:
            self._transfer = self._store.host_transfer(self.cluster.index)
        return self._transfer

    @transfer.setter
    def transfer(self, value):
        self._transfer = value

    def nodes(self):
        out = [self]
        for c in self.children:
            out.extend(c.nodes())
        return out

    def __repr__(self):
        return "BasisNode(#%d, rank %d)" % (self.cluster.index, self.rank)


class ClusterBasis:
    """Nested basis over a (possibly partial) cluster tree (``gca.py:124-146``).

    Built from a device store, the per-node Python objects are created on
    first access (a C2 basis has ~4,000 nodes; the product never needs
    them)."""

    def __init__(self, roots, by_index, store=None):
        self._roots = roots
        self._root_ids = None
        self._by_index = by_index
        self.store = store

    @classmethod
    def lazy(cls, store, flat, root_ids):
        b = cls(None, {}, store)
        b._root_ids = [int(r) for r in root_ids]
        b._flat = flat
        return b

    def _get(self, i):
        bn = self._by_index.get(i)
        if bn is None:
            st, flat = self.store, self._flat
            o_, r_ = st.piv_off[i], st.rank[i]
            bn = BasisNode(flat.node(i), st.pivots_host[o_:o_ + r_], None, st, i, self._kids_of)
            self._by_index[i] = bn
        return bn

    def _kids_of(self, i):
        flat = self._flat
        if flat.is_leaf[i]:
            return ()
        return (self._get(int(flat.left[i])), self._get(int(flat.right[i])))

    @property
    def roots(self):
        if self._roots is None:
            self._roots = [self._get(r) for r in self._root_ids]
        return self._roots

    @roots.setter
    def roots(self, value):
        self._roots = value

    @property
    def root(self):
        if len(self.roots) != 1:
            raise ConfigError("basis is a forest, not a single tree")
        return self.roots[0]

    def node(self, cluster):
        i = cluster.index if hasattr(cluster, "index") else int(cluster)
        if self._root_ids is not None:
            if not self.store.available[i] or not self.store.materialized[i]:
                raise KeyError(i)
            return self._get(i)
        return self._by_index[i]

    def nodes(self):
        return [bn for r in self.roots for bn in r.nodes()]


class DeviceBasis:
    """Device store of one nested basis, indexed by cluster-tree node id.

    Arrays (length = number of tree nodes, -1 / 0 where not materialised):
    ``rank, rows (R = factor rows), piv_off, v_off, coef_off, height``.
    Tensors: ``pivots`` (compact global pivot ids), ``V`` (R x rank
    row-major per node at ``v_off``: leaf V or internal V-hat whose row
    blocks are the children's transfers), ``VT`` (the transposes, lazily,
    :meth:`transposed_V`).
    """

    def __init__(self, tree, side, device):
        self.tree = tree
        self.flat = tree.flat
        self.side = side
        self.device = device
        n = len(self.flat)
        self.materialized = np.zeros(n, dtype=bool)
        self.available = self.materialized     # nodes whose pivots are known (sharding)
        self.rank = np.zeros(n, dtype=np.int64)
        self.rows = np.zeros(n, dtype=np.int64)
        self.piv_off = np.full(n, -1, dtype=np.int64)
        self.v_off = np.full(n, -1, dtype=np.int64)
        self.coef_off = np.full(n, -1, dtype=np.int64)
        self.child_row = np.zeros(n, dtype=np.int64)   # row offset inside parent's V-hat
        self.pivots_host = None
        self.pivots = None
        self.V = None
        self.VT = None
        self.coef_size = 0
        self._host_V = None
        self.timing = {}

    def transposed_V(self):
        """``VT``: every node's R x rank block transposed (rank x R row-major
        at the same offset), built on first use (the level-by-level
        backward transform reads it; the tiered plan does not)."""
        if self.VT is None:
            ids = np.flatnonzero(self.materialized & (self.rank > 0))
            self.VT = padded_empty(self.V.numel(), self.device).zero_()
            if ids.size:
                tdesc = to_dev(np.stack([self.v_off[ids], self.rows[ids], self.rank[ids]], 1), self.device)
                with torch.cuda.device(self.device):
                    _native.call("gc_batched_transpose", len(ids), ptr(tdesc), ptr(self.V), ptr(self.VT),
                                 stream_handle())
        return self.VT

    def host_V(self):
        if self._host_V is None:
            self._host_V = self.V.cpu().numpy()
        return self._host_V

    def host_matrix(self, i):
        o, R, r = self.v_off[i], self.rows[i], self.rank[i]
        return self.host_V()[o:o + R * r].reshape(R, r)

    def host_transfer(self, i):
        p = self.flat.parent[i]
        if p < 0 or not self.materialized[p]:
            return None
        vhat = self.host_matrix(p)
        o = self.child_row[i]
        return vhat[o:o + self.rank[i]]


def coef_layout(flat, roots, rank, base=0):
    """Coefficient offsets of a basis forest: roots first, then breadth
    first with the two children of every node adjacent, so the input of a
    parent's V-hat^T product is one contiguous slice.  Returns (offsets for
    every tree node, -1 where absent; total size).  One generation of the
    BFS queue at a time (the queue order: roots, then each generation's
    children in the order of their parents)."""
    off = np.full(len(flat), -1, dtype=np.int64)
    rank = np.asarray(rank, dtype=np.int64)
    cur = np.asarray([int(r) for r in roots], dtype=np.int64)
    pos = base
    while cur.size:
        r = rank[cur]
        off[cur] = pos + np.cumsum(r) - r
        pos += int(r.sum())
        inner = cur[~flat.is_leaf[cur]]
        cur = np.stack([flat.left[inner], flat.right[inner]], 1).ravel()
    return off, int(pos - base)


def _coef_layout_queue(flat, roots, rank, base=0):
    """The same layout with an explicit FIFO queue (reference order; kept
    for the host test that pins the vectorised form to it)."""
    off = np.full(len(flat), -1, dtype=np.int64)
    pos = base
    queue = [int(r) for r in roots]
    for r in queue:
        off[r] = pos
        pos += int(rank[r])
    k = 0
    while k < len(queue):
        i = queue[k]
        k += 1
        if not flat.is_leaf[i]:
            for c in (int(flat.left[i]), int(flat.right[i])):
                off[c] = pos
                pos += int(rank[c])
                queue.append(c)
    return off, int(pos - base)


def coupling_marks(btree):
    """Row and column cluster indices of admissible leaves (``gca.py:149-159``)."""
    r, c = coupling_mark_arrays(btree)
    return set(r.tolist()), set(c.tolist())


def coupling_mark_arrays(btree):
    """``coupling_marks`` as two sorted unique index arrays (the pipeline's
    form: no Python sets of 10^5 clusters)."""
    fb = btree.flat
    ids = btree._leaf_ids(0)
    n = max(len(fb.row_tree), len(fb.col_tree))
    return (np.flatnonzero(np.bincount(fb.row[ids], minlength=n)),
            np.flatnonzero(np.bincount(fb.col[ids], minlength=n)))


def _materialize(flat, marks):
    n = len(flat)
    if marks is None:
        mat = np.zeros(n, dtype=bool)
        mat[0] = True
    else:
        mat = np.zeros(n, dtype=bool)
        idx = (np.asarray(marks, dtype=np.int64) if isinstance(marks, np.ndarray)
               else np.fromiter((int(i) for i in marks), dtype=np.int64))
        if idx.size:
            mat[idx] = True
    marked = mat.copy()
    order = np.argsort(flat.depth, kind="stable")
    for d in range(1, int(flat.depth.max()) + 1 if n else 0):
        ids = order[flat.depth[order] == d]
        mat[ids] |= mat[flat.parent[ids]]
    roots = np.flatnonzero(marked & ~np.where(flat.parent >= 0, mat[np.maximum(flat.parent, 0)], False))
    roots = roots[mat[roots]]
    return mat, roots


def build_cluster_basis(tree, mesh, basis, m, delta_factor=0.5, eps=1e-4, side="row",
                        orders=(3, 5), marks=None, device=None, row_range=None):
    """Nested interpolation basis built bottom-up, level-synchronously on
    the device (``gca.py:162-220``).  ``row_range=(lo, hi)`` keeps only the
    nodes inside that range of tree positions (one GPU's subtree when the
    operator is sharded by block rows, ``parallel.py``); node results do
    not depend on the restriction."""
    if side not in ("row", "col"):
        raise ConfigError("side must be 'row' or 'col', got %r" % (side,))
    if basis == "collocation" and side == "col":
        raise ConfigError("column factors integrate a Galerkin basis")
    return build_cluster_bases(tree, mesh, basis, m, delta_factor, eps, [(side, marks)],
                               orders, device, row_range)[0]


class _Side:
    """Per-basis state while several bases are built in shared launches."""

    def __init__(self, tree, side, marks, row_range, dev, basis="constant"):
        flat = tree.flat
        self.side = side
        self.basis = basis
        self.store = DeviceBasis(tree, side, dev)
        mat, roots = _materialize(flat, marks)
        if row_range is not None:
            inside = (flat.start >= row_range[0]) & (flat.stop <= row_range[1])
            crossing = mat & ~inside & (flat.start < row_range[1]) & (flat.stop > row_range[0])
            if np.any(crossing & np.isin(np.arange(len(flat)), roots)):
                raise ConfigError("a basis root straddles the shard boundary; shard at a "
                                  "coarser tree level")
            mat = mat & inside
            roots = roots[inside[roots]]
        self.mat, self.roots = mat, roots
        self.store.materialized = mat
        self.store.available = mat.copy()
        self.v_parts = []        # (level tensor, start, stop)
        self.v_base = 0


def _bases_levels_device(S, flat, heights, dmesh, m, K, W, eps, delta_factor, dev, stream, d_g01, d_w01):
    """The level loop of :func:`build_cluster_bases` with its bookkeeping on
    the device (``csrc/bases.cu``): per height the factor rows R (leaf size
    or the children's ranks), their scans, the row lists, the factor and ACA
    launches and the local -> global pivot map, with one 4 + sides integer
    read per level (the row totals that size the buffers and the ACA's
    shared memory).  Ranks, pivots and offsets come back once at the end."""
    nf = len(flat)
    levels, lo = [], 0
    for h in heights:
        segs = []
        for k, s in enumerate(S):
            ids = np.flatnonzero(s.mat & (flat.height == h))
            if ids.size:
                segs.append((k, ids))
        nn = sum(len(i) for _, i in segs)
        if nn:
            levels.append((lo, nn, segs))
            lo += nn
    T = lo
    if T == 0:
        return 0.0, 0.0
    all_ids = np.concatenate([i for _, _, segs in levels for _, i in segs])
    bounds = [np.r_[np.cumsum([0] + [len(i) for _, i in segs])] for _, _, segs in levels]
    b_off = _offsets(np.array([len(b) for b in bounds]))
    diam = flat.diam[all_ids]
    perm_dev = getattr(flat, "_perm_dev", None)
    if perm_dev is not None and perm_dev.device != dev:
        perm_dev = None
    ints = to_dev(np.concatenate([flat.left, flat.right, flat.start, flat.stop, all_ids, np.concatenate(bounds)]
                                 + ([] if perm_dev is not None else [flat.perm])), dev)
    d_left, d_right, d_start, d_stop = (ints[i * nf:(i + 1) * nf] for i in range(4))
    d_nodes = ints[4 * nf:4 * nf + T]
    d_bounds = ints[4 * nf + T:4 * nf + T + int(b_off[-1] + len(bounds[-1]))]
    if perm_dev is None:
        perm_dev = ints[4 * nf + T + len(d_bounds):]
    box = np.concatenate([flat.lower[all_ids], flat.upper[all_ids], (delta_factor * diam)[:, None],
                          diam[:, None]], axis=1)
    dbl = to_dev(np.concatenate([box.ravel(), diam]), dev)
    d_box, d_diam = dbl[:8 * T], dbl[8 * T:]
    # per side on the device: rank | piv_off | rows | v_off | cursor | pivots
    side_buf = []
    for s in S:
        cap = int(np.minimum((flat.stop - flat.start)[s.mat], W).sum()) if s.mat.any() else 0
        b = torch.zeros(4 * nf + 1 + max(cap, 1), dtype=torch.int64, device=dev)
        b[nf:2 * nf].fill_(-1)
        b[3 * nf:4 * nf].fill_(-1)
        side_buf.append(b)
    # level scratch: R, limit, vcap, their offsets (6 T), descriptors (9 T),
    # the per-level totals (4 + bounds) and the post scan's rank offsets
    n_tot = sum(4 + len(b) for b in bounds)
    scr = torch.empty(15 * T + n_tot + max(nn for _, nn, _ in levels), dtype=torch.int64, device=dev)
    tb = _native.ctypes.c_int64(0)
    _native.call("gc_bases_scan_bytes", max(nn for _, nn, _ in levels), _native.ctypes.byref(tb))
    temp = torch.empty(max(tb.value, 1), dtype=torch.uint8, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    P = scr.data_ptr()
    p_left, p_right, p_start, p_stop = (t.data_ptr() for t in (d_left, d_right, d_start, d_stop))
    cols = [P + 8 * c * T for c in range(15)]         # R lim vcap roff ploff voff fdesc(5) adesc(4)
    t_factor = t_aca = 0.0
    tot_base = 15 * T
    rk_off = P + 8 * (15 * T + n_tot)
    side_code = [0 if s.side == "row" else 1 for s in S]
    with torch.cuda.device(dev):
        for li, (lo, nn, segs) in enumerate(levels):
            R, lim, vcap, roff, ploff, voff = (c + 8 * lo for c in cols[:6])
            fdesc, adesc = cols[6] + 40 * lo, cols[6] + 40 * T + 32 * lo
            tot = tot_base + sum(4 + len(b) for b in bounds[:li])
            pos = [int(v) for v in bounds[li]]
            for j, (k, ids) in enumerate(segs):
                sb = side_buf[k].data_ptr()
                _native.call("gc_bases_R", len(ids), d_nodes.data_ptr() + 8 * (lo + pos[j]), p_left, p_right, p_start,
                             p_stop, sb, int(pos[j]), W, R, lim, vcap, sb + 16 * nf, stream)
            _native.call("gc_bases_scan", nn, R, lim, vcap, roff, ploff, voff, d_bounds.data_ptr() + 8 * int(b_off[li]),
                         len(pos), P + 8 * tot, ptr(temp), tb.value, stream)
            host = scr[tot:tot + 4 + len(pos)].cpu().numpy()      # the level's only sync
            r_max, n_rows, n_lim, n_v = (int(v) for v in host[:4])
            tf = time.perf_counter()
            rows = torch.empty(max(n_rows, 1), dtype=torch.int64, device=dev)
            for j, (k, ids) in enumerate(segs):
                sb = side_buf[k].data_ptr()
                _native.call("gc_bases_rows", len(ids), d_nodes.data_ptr() + 8 * (lo + pos[j]), p_left, p_right, p_start,
                             sb, sb + 8 * nf, sb + 8 * (4 * nf + 1), ptr(perm_dev), int(pos[j]), 0,
                             side_code[k], W, R, roff, ploff, voff, ptr(rows), fdesc, adesc, stream)
            z = empty(nn * K * 3, dev)
            sq = empty(nn * K, dev)
            nz = empty(nn * K * 3, dev)
            _native.call("gc_green_box_rules", m, ptr(d_g01), ptr(d_w01), nn, d_box.data_ptr() + 64 * lo,
                         ptr(z), ptr(sq), ptr(nz), stream)
            fac = empty(max(n_rows, 1) * 2 * K, dev)
            # one factor launch per run of sides with the same row kind
            # (collocation rows pair with linear columns)
            runs = []
            for j, (k, ids) in enumerate(segs):
                if runs and runs[-1][0] == S[k].basis:
                    runs[-1][2] = int(pos[j + 1])
                else:
                    runs.append([S[k].basis, int(pos[j]), int(pos[j + 1])])
            for b, p0, p1 in runs:
                _native.call("gc_green_factor", dmesh.geom_of("slp", b), -1, K, p1 - p0, fdesc + 40 * p0,
                             d_diam.data_ptr() + 8 * (lo + p0), ptr(z), ptr(sq), ptr(nz), ptr(rows), ptr(fac),
                             ptr(flags), stream)
            ta = time.perf_counter()
            t_factor += ta - tf
            V = torch.zeros(max(n_v, 1), dtype=torch.float64, device=dev)
            U = empty(max(n_v, 1), dev)
            small = torch.zeros(max(n_lim, 1) + nn, dtype=torch.int64, device=dev)
            d_piv, d_rank = small[:max(n_lim, 1)], small[max(n_lim, 1):]
            _native.call("gc_aca", nn, adesc, W, float(eps), 0, ptr(fac), ptr(d_piv), ptr(d_rank),
                         ptr(V), ptr(U), r_max, stream)
            for j, (k, ids) in enumerate(segs):
                s, sb = S[k], side_buf[k].data_ptr()
                v0, v1 = int(host[4 + j]), int(host[5 + j])
                _native.call("gc_bases_post", len(ids), d_nodes.data_ptr() + 8 * (lo + pos[j]), int(pos[j]),
                             ptr(d_rank), ptr(d_piv), ploff, ptr(rows), roff, voff, s.v_base, sb + 32 * nf,
                             sb, sb + 8 * nf, sb + 8 * (4 * nf + 1), sb + 24 * nf, rk_off, ptr(temp), tb.value,
                             stream)
                s.v_parts.append(V[v0:max(v1, v0)])
                s.v_base += v1 - v0
            t_aca += time.perf_counter() - ta
            del U, fac, z, sq, nz
    fl = flags.cpu()
    if int(fl[0]) & 1:
        raise GeometryError("expansion point touches the surface; enlarge delta or the cluster box")
    for s, b in zip(S, side_buf):
        st = s.store
        host = b[:4 * nf + 1].cpu().numpy()
        st.rank, st.piv_off, st.rows, st.v_off = (host[i * nf:(i + 1) * nf].copy() for i in range(4))
        cursor = int(host[4 * nf])
        st.pivots = b[4 * nf + 1:4 * nf + 1 + max(cursor, 1)]
        st.pivots_host = st.pivots[:cursor].cpu().numpy()
        inner = np.flatnonzero(s.mat & ~flat.is_leaf)
        st.child_row[flat.right[inner]] = st.rank[flat.left[inner]]
    return t_factor, t_aca


def build_cluster_bases(tree, mesh, basis, m, delta_factor, eps, sides, orders=(3, 5),
                        device=None, row_range=None):
    """Several nested bases of one cluster tree (row and column side of the
    H2 matrix) built together: per tree height one ``gc_green_box_rules``,
    one ``gc_green_factor`` (side per node) and one ``gc_aca`` launch over
    the nodes of every basis, with the row lists and the pivot bookkeeping
    on the device (:func:`_bases_levels_device`); ranks, pivots and the
    touch flags reach the host once, at the end.  ``sides`` is a list of (side, marks) or (side,
    marks, basis) - collocation rows pair a "collocation" row side with a
    "linear" column side.  Rows are triangles (constant basis) or vertices
    (linear basis, collocation points)."""
    for sd in sides:
        check_mesh(mesh, "slp", sd[2] if len(sd) > 2 else basis, linear_ok=True)
    if tree.index != 0:
        raise ConfigError("build_cluster_basis expects the root of a cluster tree")
    dev = require_device(device)
    t0 = time.perf_counter()
    flat = tree.flat
    dmesh = DeviceMesh.get(mesh, orders[0], dev)
    K = 6 * m * m
    W = 2 * K
    g01, w01 = _gauss01(m)
    d_g01, d_w01 = to_dev(g01, dev), to_dev(w01, dev)
    S = [_Side(tree, sd[0], sd[1], row_range, dev, sd[2] if len(sd) > 2 else basis) for sd in sides]
    heights = np.unique(np.concatenate([flat.height[s.mat] for s in S])) if S else []
    t_factor, t_aca = _bases_levels_device(S, flat, heights, dmesh, m, K, W, eps, delta_factor,
                                           dev, stream_handle(), d_g01, d_w01)
    out = []
    for s in S:
        st = s.store
        st.V = padded_copy(torch.cat(s.v_parts)) if s.v_parts else padded_empty(1, dev)
        if st.V.numel() == 0:
            st.V = padded_empty(1, dev).zero_()
        st.coef_off, st.coef_size = coef_layout(flat, s.roots, st.rank)
        st.timing = {"factor_s": t_factor, "aca_s": t_aca, "total_s": time.perf_counter() - t0,
                     "shared_with": len(S)}
        out.append(ClusterBasis.lazy(st, flat, s.roots))
    return out


def expand_basis(node):
    """Dense cluster-size x rank matrix realised by the nested basis."""
    if not node.children:
        return node.v
    return np.vstack([expand_basis(c) @ c.transfer for c in node.children])


# --------------------------------------------------------------------------
# H2 matrix

class _BlockList(Sequence):
    """Lazy list of coupling / near-field blocks backed by a device store
    (column-major per block); ``values`` are host arrays created on access."""

    def __init__(self, factory, rows, cols, nr, nc, off, store):
        self._factory = factory
        self._rows, self._cols = rows, cols
        self._nr, self._nc, self._off = nr, nc, off
        self._store = store
        self._host = None
        self._owner = None          # weakref to the H2Matrix (settle before reading)

    def __len__(self):
        return len(self._rows)

    def _host_store(self):
        if self._host is None:
            owner = self._owner() if self._owner is not None else None
            if owner is not None:
                owner.settle()
            self._host = self._store.cpu().numpy()
        return self._host

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        nr, nc, o = int(self._nr[i]), int(self._nc[i]), int(self._off[i])
        vals = self._host_store()[o:o + nr * nc].reshape(nc, nr).T
        return self._factory(self._tree_r.node(int(self._rows[i])),
                             self._tree_c.node(int(self._cols[i])), vals)

    def bind(self, row_flat, col_flat):
        self._tree_r, self._tree_c = row_flat, col_flat
        return self


class H2Matrix:
    """Compressed operator (``gca.py:234-259``) whose blocks live in HBM.

    ``dev`` holds the device stores and the matvec plans used by
    :mod:`h2`; ``coupling`` / ``nearfield`` are lazy host views.
    """

    def __init__(self, row_tree, col_tree, row_basis, col_basis, coupling, nearfield,
                 exec_stats=None, dev=None):
        self.row_tree = row_tree
        self.col_tree = col_tree
        self.row_basis = row_basis
        self.col_basis = col_basis
        self.coupling = coupling
        self.nearfield = nearfield
        self._exec_stats = exec_stats
        self._settle = None
        self._settle_lock = threading.Lock()
        self.dev = dev

    def settle(self):
        """Wait for the device assembly (build_h2 returns while its
        quadrature runs), check its queue flags and fix the executor
        statistics; idempotent and thread-safe.  Every reader of block data
        calls it."""
        if self._settle is not None:
            with self._settle_lock:
                if self._settle is not None:
                    self._exec_stats = self._settle()
                    self._settle = None
        return self

    @property
    def exec_stats(self):
        """Per-case executor statistics (``batchexec.py:211-213``)."""
        self.settle()
        return self._exec_stats

    @exec_stats.setter
    def exec_stats(self, value):
        self._settle = None
        self._exec_stats = value

    @property
    def shape(self):
        return (self.row_tree.size, self.col_tree.size)

    def __repr__(self):
        return "H2Matrix(%dx%d, %d coupling, %d nearfield)" % (
            self.shape + (len(self.coupling), len(self.nearfield)))


class DeviceH2:
    """Device-resident block data of an H2 matrix.

    coupling store: S (r_tau x r_sigma) column-major per block;
    near store: N (size_tau x size_sigma) column-major per block.
    Block metadata arrays are kept in reference (depth-first) order.
    """

    def __init__(self, device):
        self.device = device
        self.plans = {}


DEFAULT_CAPACITY = 4096        # the reference executor's list capacity (batchexec.py:27)


def _exec_stats(tasks, capacity, seconds):
    """Per-case executor statistics as the reference's BatchExecutor.stats()
    (``batchexec.py:211-213``): every case's tasks go through one list that
    is sealed whenever it reaches ``capacity`` and once more at finalize for
    a partial tail, so batches = ceil(tasks / capacity)
    (``batchexec.py:37-52, 154-166``).  ``wall_s``: the device time that
    evaluated the case (the reference: evaluator wall time summed over its
    batches)."""
    if capacity < 1:
        raise ConfigError("capacity must be >= 1")
    return [{"tasks": int(t), "batches": -(-int(t) // capacity), "wall_s": float(w), "case": k}
            for k, (t, w) in enumerate(zip(tasks, seconds))]


def _case_seconds(calls, rules):
    """Device seconds per pair case from device_block_assembly's events
    (``calls`` = [(events, counts)] per call): the block kernel evaluates
    the disjoint pairs (case 0), the singular flush cases 1-3, split by
    their quadrature points (tasks x points)."""
    sec = [0.0] * 4
    for (a, b, c), st in [(ev[0], st) for ev, st in calls if ev]:
        sec[0] += a.elapsed_time(b) * 1e-3
        w = [st[k] * rules.npts[k] for k in (1, 2, 3)]
        tot = float(sum(w))
        for k in (1, 2, 3):
            if tot > 0:
                sec[k] += b.elapsed_time(c) * 1e-3 * w[k - 1] / tot
    return sec


class _BlockTables:
    """Coupling and near-field block tables of one build_h2 call, built on
    the device (``gc_h2_blocks``): the assembly descriptors stay there, the
    host copies (row, col, nr, nc, off, order per kind) arrive on a side
    stream while the quadrature runs."""

    def __init__(self, shapes, c_desc, n_desc, host_buf, counts, done):
        self.shapes = shapes
        self.c_desc, self.n_desc = c_desc, n_desc
        self._buf, self._counts, self._done = host_buf, counts, done
        self._host = None

    def host(self):
        if self._host is None:
            self._done.synchronize()
            h = self._buf.numpy()
            nc_, nn_ = self._counts
            tc, tn = h[:6 * nc_].reshape(6, nc_), h[6 * nc_:6 * (nc_ + nn_)].reshape(6, nn_)
            self._host = tuple(tc), tuple(tn)
        return self._host


def _device_block_tables(btree, rf, cf, rstore, cstore, row_range, dev):
    """The block tables of :func:`build_h2` from the block tree's leaves
    (``csrc/h2blocks.cu``); one small read of the totals (counts, maxima,
    entries), which size the stores and the quadrature launches."""
    fb = btree.flat
    a, b = np.searchsorted(fb.leaf_key, [fb.key_lo[btree._id], fb.key_hi[btree._id]], side="left")
    nl = int(b - a)
    # the device block tree's node arrays (clustering._build_block_tree_device)
    # serve this one call; later calls upload the host arrays
    dv = getattr(fb, "_dev", None)
    fb._dev = None
    if dv is None or dv[0].device != dev:
        nn = len(fb.row)
        ints = to_dev(np.concatenate([fb.row, fb.col, fb.leaf_ids]).astype(np.int64), dev)
        dv = (ints[:nn], ints[nn:2 * nn], to_dev(fb.state.astype(np.int8), dev), ints[2 * nn:])
    node_row, node_col, node_state, leaf_ids = dv
    same = cf is rf
    parts = [rf.start, rf.stop, rstore.rank, rstore.piv_off]
    if not same:
        parts += [cf.start, cf.stop]
    parts += [cstore.rank, cstore.piv_off]
    tree_i = to_dev(np.concatenate(parts).astype(np.int64), dev)
    nr_, nc_ = len(rf.start), len(cf.start)
    r_start, r_stop, r_rank, r_poff = (tree_i[k * nr_:(k + 1) * nr_] for k in range(4))
    o = 4 * nr_
    if same:
        c_start, c_stop = r_start, r_stop
    else:
        c_start, c_stop = tree_i[o:o + nc_], tree_i[o + nc_:o + 2 * nc_]
        o += 2 * nc_
    c_rank, c_poff = tree_i[o:o + nc_], tree_i[o + nc_:o + 2 * nc_]
    ok = to_dev(np.concatenate([rstore.materialized, cstore.available]).astype(np.int8), dev)
    r_ok, c_ok = ok[:nr_], ok[nr_:]
    lo, hi = (-1, -1) if row_range is None else (int(row_range[0]), int(row_range[1]))
    key_bits = max(1, int(2 * nr_ + 2).bit_length())
    n = max(nl, 1)
    tb = _native.ctypes.c_int64(0)
    _native.call("gc_h2_blocks_bytes", n, _native.ctypes.byref(tb))
    temp = torch.empty(max(tb.value, 1), dtype=torch.uint8, device=dev)
    scratch = torch.empty(12 * n, dtype=torch.int64, device=dev)
    flags = torch.empty(2 * n, dtype=torch.int8, device=dev)
    tables = torch.empty(2, 11 * n, dtype=torch.int64, device=dev)       # table (6 n) | desc (5 n) per kind
    totals = torch.zeros(2, 8, dtype=torch.int64, device=dev)
    stream = stream_handle()
    with torch.cuda.device(dev):
        for kind in (0, 1):
            _native.call("gc_h2_blocks", nl, leaf_ids.data_ptr() + 8 * int(a), ptr(node_row), ptr(node_col),
                         ptr(node_state), ptr(r_start), ptr(r_stop), ptr(c_start), ptr(c_stop), ptr(r_rank),
                         ptr(r_poff), ptr(c_rank), ptr(c_poff), ptr(r_ok), ptr(c_ok), lo, hi, kind, key_bits,
                         ptr(tables[kind]), tables[kind].data_ptr() + 8 * 6 * n, totals[kind].data_ptr(),
                         ptr(scratch), ptr(flags), ptr(temp), tb.value, stream)
        tot = totals.cpu().numpy()                  # the only synchronisation
        if tot[0, 7]:
            raise ConfigError("coupling block without basis content; build the bases "
                              "with coupling_marks(btree)")
        counts = int(tot[0, 0]), int(tot[1, 0])
        host = torch.empty(max(6 * sum(counts), 1), dtype=torch.int64, pin_memory=True)
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            host[:6 * counts[0]].copy_(tables[0, :6 * counts[0]], non_blocking=True)
            host[6 * counts[0]:6 * sum(counts)].copy_(tables[1, :6 * counts[1]], non_blocking=True)
            done = torch.cuda.Event()
            done.record(side)
        # the tables stay referenced by the side stream's copy
        tables.record_stream(side)
    shapes = tuple((int(t[1]), int(t[2]), int(t[3]), int(t[4]), int(t[0])) for t in tot)
    c_desc = tables[0, 6 * n:6 * n + 5 * shapes[0][0]].view(-1, 5)
    n_desc = tables[1, 6 * n:6 * n + 5 * shapes[1][0]].view(-1, 5)
    return _BlockTables(shapes, c_desc, n_desc, host, counts, done)


def build_h2(btree, row_basis, col_basis, mesh, kind="slp", basis="constant",
             disc="galerkin", orders=(3, 5), capacity=None, threads=None, device=None,
             row_range=None):
    """Assemble the H2 matrix (``gca.py:282-312``) on the device.

    Admissible leaves get exact entries at pivot rows x pivot columns,
    inadmissible leaves dense blocks.  ``row_range=(lo, hi)`` restricts the
    assembly to block rows whose row cluster lies in tree positions
    [lo, hi) (block-row sharding across GPUs, SURVEY.md §8 e)."""
    if disc not in ("galerkin", "collocation"):
        raise ConfigError("unknown discretization %r" % (disc,))
    if disc == "collocation" and basis != "linear":
        raise ConfigError("collocation rows pair with the linear basis")
    check_mesh(mesh, kind, basis, linear_ok=True)
    dev = require_device(device)
    fb = btree.flat
    rf, cf = fb.row_tree, fb.col_tree
    rstore, cstore = row_basis.store, col_basis.store
    dmesh = DeviceMesh.get(mesh, orders[0], dev)
    rules = DeviceRules.get(orders[1], dev, kind)
    queue = SingularQueue.get(mesh, dev)
    t0 = time.perf_counter()
    # coupling blocks: pivot rows x pivot columns; near-field blocks: full
    # clusters.  Storage is grouped by row cluster: the blocks of one block
    # row form one contiguous (sum r_sigma) x r_tau panel for the matvec
    # (h2.PanelPlan); a block-row shard stores, inside each block row, the
    # blocks with local columns (its own tree positions) before the others,
    # so either subset is one contiguous sub-panel (the sharded product runs
    # them before / after its all-gathers, parallel.ShardPlan)
    tabs = _device_block_tables(btree, rf, cf, rstore, cstore, row_range, dev)
    c_shape, n_shape = tabs.shapes
    c_total, n_total = c_shape[3], n_shape[3]
    coup = padded_empty(max(c_total, 1), dev)
    near = padded_empty(max(n_total, 1), dev)
    perm_r = to_dev(rf.perm, dev)
    perm_c = perm_r if cf is rf else to_dev(cf.perm, dev)
    if basis == "linear":
        # vertex DOFs: every block is the scatter of its triangle pairs'
        # 3x3 integrals (linear.py); collocation rows are point evaluations
        from . import linear
        (cr, cc, c_nr, c_nc, c_off, c_order), (nr_r, nc_r, n_nr, n_nc, n_off, n_order) = tabs.host()
        keep = (c_nr > 0) & (c_nc > 0)
        rp, cp = rstore.pivots_host, cstore.pivots_host
        # (rows, cols, out_off, row key, col key): one triangle table per cluster
        cblocks = [(rp[rstore.piv_off[a]:rstore.piv_off[a] + nr], cp[cstore.piv_off[b]:cstore.piv_off[b] + nc], o,
                    int(a), int(b))
                   for a, b, nr, nc, o in zip(cr[keep], cc[keep], c_nr[keep], c_nc[keep], c_off[keep])]
        nblocks = [(rf.perm[rf.start[a]:rf.stop[a]], cf.perm[cf.start[b]:cf.stop[b]], o, int(a), int(b))
                   for a, b, o in zip(nr_r, nc_r, n_off)]
        if disc == "collocation":
            crules = linear.CollocationRules(*orders)
            s_c = linear.collocation_blocks(dmesh, kind, crules, mesh, cblocks, coup, dev)
            t1 = time.perf_counter()
            s_n = linear.collocation_blocks(dmesh, kind, crules, mesh, nblocks, near, dev)
            stats_c, stats_n = s_c + [0, 0], s_n + [0, 0]
        else:
            lrules = linear.LinearRules.get(orders[0], orders[1], dev)
            stats_c = linear.assemble_blocks(dmesh, kind, lrules, mesh, cblocks, coup, dev)
            t1 = time.perf_counter()
            stats_n = linear.assemble_blocks(dmesh, kind, lrules, mesh, nblocks, near, dev)
    else:
        # plane charts: no host synchronisation - the quadrature runs while
        # the caller continues (e.g. builds the matvec plan); the counts,
        # the queue flags and the timings settle on first use (H2Matrix.settle).
        # The descriptors were built on the device; the host copies of the
        # block tables arrive meanwhile on a side stream.
        ev_c, ev_n, pending = [], [], ([] if not dmesh.curved else None)
        stats_c = device_block_assembly(dmesh, rules, queue, rstore.pivots, cstore.pivots, None, coup,
                                        kind=kind, events=ev_c, pending=pending, d_desc=tabs.c_desc,
                                        shape=c_shape)
        t1 = time.perf_counter()
        # near-field blocks: full clusters
        stats_n = device_block_assembly(dmesh, rules, queue, perm_r, perm_c, None, near, kind=kind,
                                        events=ev_n, pending=pending, d_desc=tabs.n_desc, shape=n_shape)
        (cr, cc, c_nr, c_nc, c_off, c_order), (nr_r, nc_r, n_nr, n_nc, n_off, n_order) = tabs.host()
    d = DeviceH2(dev)
    d.coup, d.near = coup, near
    d.c_rows, d.c_cols, d.c_nr, d.c_nc, d.c_off = cr, cc, c_nr, c_nc, c_off
    d.n_rows, d.n_cols, d.n_nr, d.n_nc, d.n_off = nr_r, nc_r, n_nr, n_nc, n_off
    d.c_order, d.n_order = c_order, n_order            # block indices in storage order
    d.perm_r, d.perm_c = perm_r, perm_c
    d.row_range = row_range
    ncase = 2 if disc == "collocation" else 4                 # the reference's executor cases
    cap = DEFAULT_CAPACITY if capacity is None else int(capacity)

    def settle():
        torch.cuda.synchronize(dev)
        t2 = time.perf_counter()
        if basis != "linear":
            done = iter(resolve_counts(pending, queue) if pending else [])
            sc, sn = [next(done) if r is None else r for r in (stats_c, stats_n)]
            sec = _case_seconds([(ev_c, sc), (ev_n, sn)], rules)
            d.timing = {"coupling_s": sum(a.elapsed_time(c) for a, _, c in ev_c) * 1e-3,
                        "nearfield_s": sum(a.elapsed_time(c) for a, _, c in ev_n) * 1e-3}
        else:
            sc, sn = stats_c, stats_n
            sec = [t2 - t0] + [0.0] * (ncase - 1)
            d.timing = {"coupling_s": t1 - t0, "nearfield_s": t2 - t1}
        return _exec_stats([sc[k] + sn[k] for k in range(ncase)], cap, sec)

    if cap < 1:
        raise ConfigError("capacity must be >= 1")
    coupling = _BlockList(CouplingBlock, cr, cc, c_nr, c_nc, c_off, coup).bind(rf, cf)
    nearfield = _BlockList(NearfieldBlock, nr_r, nc_r, n_nr, n_nc, n_off, near).bind(rf, cf)
    hm = H2Matrix(rf.node(0), cf.node(0), row_basis, col_basis, coupling, nearfield, None, d)
    hm._settle = settle
    coupling._owner = nearfield._owner = weakref.ref(hm)
    if basis == "linear" or pending is None:
        hm.settle()                       # synchronous paths: settle now (errors surface here)
    return hm
