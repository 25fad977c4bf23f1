"""Cluster trees and admissibility block trees, built array-at-a-time.

Host-side mirror of ``greencross/clustering.py``.  The public objects keep
the reference's shapes (``BoundingBox`` ``:15-43``, ``admissible``
``:46-51``, ``ClusterTree`` ``:54-104``, ``BlockTree`` ``:170-212``) and the
results are bit-identical: same permutation, same boxes, same preorder
indices, same leaves in the same depth-first order.  The construction is
different: instead of one Python call per node the trees are grown one level
at a time over flat arrays (segmented min/max, one stable ``lexsort`` per
level, vectorised admissibility), which is what makes the host plan cheap
enough at 0.5-2 M triangles (SURVEY.md §8 f, rank 1).  The flat arrays
(``ClusterTree.flat`` and ``BlockTree.flat``) are what the device layout in
``gca.py`` is built from.
"""

import numpy as np

from .errors import ConfigError
from .geometry import control_points

ADMISSIBLE = "admissible"
INADMISSIBLE = "inadmissible"
SUBDIVIDED = "subdivided"


def _blas_norm(v):
    # 1-D numpy norm = sqrt(ddot(v, v)); the reference's rounding
    return float(np.linalg.norm(v))


_NORM_MODE = []


def blas_norms(v):
    """``np.linalg.norm(row)`` for every row of an (n,3) array, bit for bit,
    without n Python calls: the native host helper evaluates the rounding
    sequence that numpy's 1-D norm (OpenBLAS ddot) was found to use on this
    host, checked once against numpy on a probe set; if neither candidate
    reproduces numpy exactly the rows are normed one by one."""
    v = np.ascontiguousarray(v, dtype=np.float64).reshape(-1, 3)
    if not _NORM_MODE:
        rng = np.random.default_rng(7)
        probe = np.concatenate([rng.standard_normal((512, 3)),
                                rng.random((512, 3)) * np.array([1e-3, 1.0, 3.0])])
        want = np.array([float(np.linalg.norm(r)) for r in probe])
        mode = None
        for m in (0, 1):
            got = _native_norms(probe, m)
            if np.array_equal(got, want):
                mode = m
                break
        _NORM_MODE.append(mode)
    mode = _NORM_MODE[0]
    if mode is None:
        return np.array([float(np.linalg.norm(r)) for r in v])
    return _native_norms(v, mode)


def _native_norms(v, mode):
    """Row norms by the C-ABI's host routine (gc_host_norm3); the library
    is required (a load failure raises)."""
    from . import _native
    lib = _native.load()
    out = np.empty(len(v))
    if len(v):
        _native.check(lib.gc_host_norm3(v.ctypes.data, len(v), out.ctypes.data, mode))
    return out


class BoundingBox:
    """Axis-parallel box (``clustering.py:15-43``)."""

    __slots__ = ("lower", "upper")

    def __init__(self, lower, upper):
        self.lower = np.asarray(lower, dtype=float)
        self.upper = np.asarray(upper, dtype=float)
        if self.lower.shape != (3,) or self.upper.shape != (3,):
            raise ConfigError("bounding box corners must be 3-vectors")
        if np.any(self.lower > self.upper):
            raise ConfigError("bounding box has lower > upper")

    @classmethod
    def of_points(cls, points):
        p = np.asarray(points, dtype=float).reshape(-1, 3)
        return cls(p.min(axis=0), p.max(axis=0))

    def diameter(self):
        return _blas_norm(self.upper - self.lower)

    def distance(self, other):
        gap = np.maximum(0.0, np.maximum(self.lower - other.upper,
                                         other.lower - self.upper))
        return _blas_norm(gap)

    def __repr__(self):
        return "BoundingBox(%s, %s)" % (self.lower.tolist(), self.upper.tolist())


def admissible(tau, sigma, eta):
    """Standard admissibility max(diam) <= 2 eta dist (``clustering.py:46-51``)."""
    if eta <= 0:
        raise ConfigError("eta must be positive, got %r" % (eta,))
    return max(tau.diameter(), sigma.diameter()) <= 2.0 * eta * tau.distance(sigma)


class ClusterTree:
    """Node view of a flat cluster tree; ``perm[start:stop]`` are its dofs,
    ``index`` its preorder number."""

    __slots__ = ("perm", "start", "stop", "_box", "_children", "index", "flat")

    def __init__(self, flat, index):
        self.flat = flat
        self.perm = flat.perm
        self.index = index
        self.start = int(flat.start[index])
        self.stop = int(flat.stop[index])
        self._box = None
        self._children = None

    @property
    def box(self):
        if self._box is None:
            self._box = BoundingBox(self.flat.lower[self.index], self.flat.upper[self.index])
        return self._box

    @property
    def children(self):
        if self._children is None:
            f, i = self.flat, self.index
            self._children = () if f.left[i] < 0 else (f.node(int(f.left[i])), f.node(int(f.right[i])))
        return self._children

    @property
    def size(self):
        return self.stop - self.start

    @property
    def indices(self):
        return self.perm[self.start:self.stop]

    def is_leaf(self):
        return bool(self.flat.left[self.index] < 0)

    def nodes(self):
        """Subtree nodes in preorder."""
        return [self.flat.node(i) for i in range(self.index,
                                                 self.index + int(self.flat.count[self.index]))]

    def leaves(self):
        return [n for n in self.nodes() if n.is_leaf()]

    def depth(self):
        sub = slice(self.index, self.index + int(self.flat.count[self.index]))
        return int(self.flat.depth[sub].max() - self.flat.depth[self.index])

    def __repr__(self):
        return "ClusterTree(#%d, %d dofs, %s)" % (
            self.index, self.size, "leaf" if self.is_leaf() else "2 children")


class FlatClusterTree:
    """Preorder arrays of a binary cluster tree.

    ``start, stop, left, right (-1 for leaves), parent, depth, count
    (subtree size in nodes), lower, upper (N,3), diam`` plus ``perm``.
    ``diam`` is the reference's ``box.diameter()`` bit for bit.
    """

    def __init__(self, perm, start, stop, left, right, parent, depth, lower, upper):
        self.perm = perm
        self.start, self.stop = start, stop
        self.left, self.right, self.parent, self.depth = left, right, parent, depth
        self.lower, self.upper = lower, upper
        n = len(start)
        self.is_leaf = left < 0
        # subtree node counts and heights, one tree depth at a time (bottom up)
        self.count = np.ones(n, dtype=np.int64)
        h = np.zeros(n, dtype=np.int64)
        for d in range(int(depth.max()) if n else 0, 0, -1):
            ids = np.flatnonzero(depth == d)
            np.add.at(self.count, parent[ids], self.count[ids])
            np.maximum.at(h, parent[ids], h[ids] + 1)
        self.height = h
        self.diam = blas_norms(upper - lower)
        self._nodes = [None] * n

    def __len__(self):
        return len(self.start)

    def node(self, i):
        nd = self._nodes[i]
        if nd is None:
            nd = ClusterTree(self, i)
            self._nodes[i] = nd
        return nd


def _support_data(mesh, basis_kind):
    """Reference points and support bounds per dof (``clustering.py:107-128``)."""
    ctrl = control_points(mesh)
    lo, hi = ctrl[:, 0].copy(), ctrl[:, 0].copy()      # = ctrl.min/max(axis=1), exact, 3x faster
    for k in range(1, ctrl.shape[1]):
        np.minimum(lo, ctrl[:, k], out=lo)
        np.maximum(hi, ctrl[:, k], out=hi)
    if basis_kind == "constant":
        return mesh.centroids(), lo, hi
    stars = mesh.vertex_stars()
    sizes = np.array([len(s) for s in stars])
    if np.any(sizes == 0):
        raise ConfigError("mesh has isolated vertices")
    adj = np.concatenate(stars)
    first = np.concatenate(([0], np.cumsum(sizes)))[:-1]
    return (mesh.vertices.copy(), np.minimum.reduceat(lo[adj], first, axis=0),
            np.maximum.reduceat(hi[adj], first, axis=0))


def _subtree_counts(size, leaf_size, memo):
    if size not in memo:
        if size <= leaf_size:
            memo[size] = 1
        else:
            h = size // 2
            memo[size] = (1 + _subtree_counts(h, leaf_size, memo)
                          + _subtree_counts(size - h, leaf_size, memo))
    return memo[size]


def build_cluster_tree(mesh, basis_kind="constant", leaf_size=32, device=None):
    """Binary cluster tree: split at the positional median along the longest
    box axis, stable in the reference point coordinate
    (``clustering.py:131-162``).  Returns the root :class:`ClusterTree`.
    With ``device`` the per-depth box reductions, key sorts and permutations
    run on the GPU (``csrc/tree.cu``); the result is identical."""
    if basis_kind not in ("constant", "linear"):
        raise ConfigError("unknown basis kind %r" % (basis_kind,))
    if leaf_size < 1:
        raise ConfigError("leaf_size must be >= 1")
    if device is not None:
        return _build_cluster_tree_device(mesh, basis_kind, leaf_size, device)
    points, lo, hi = _support_data(mesh, basis_kind)
    n = len(points)
    memo = {}
    total = _subtree_counts(n, leaf_size, memo)
    start = np.zeros(total, dtype=np.int64)
    stop = np.zeros(total, dtype=np.int64)
    left = np.full(total, -1, dtype=np.int64)
    right = np.full(total, -1, dtype=np.int64)
    parent = np.full(total, -1, dtype=np.int64)
    depth = np.zeros(total, dtype=np.int64)
    lower = np.zeros((total, 3))
    upper = np.zeros((total, 3))
    perm = np.arange(n)
    # one padding row so that reduceat may address index n
    # lo/hi/points in current permutation order, plus one padding row so
    # that reduceat may address index n; permuted in place with perm
    # one (n+1, 9) array [lo | hi | point] permuted as a whole each level
    pack = np.concatenate([np.concatenate([lo, hi, points], axis=1),
                           np.concatenate([lo[:1], hi[:1], points[:1]], axis=1)])
    lo_p, hi_p, pts_p = pack[:, 0:3], pack[:, 3:6], pack[:, 6:9]

    # frontier of one tree depth: node ids with contiguous [start, stop)
    ids = np.array([0], dtype=np.int64)
    stop[0] = n
    d = 0
    while ids.size:
        s, e = start[ids], stop[ids]
        depth[ids] = d
        # boxes: segmented min/max over the current permutation (the
        # frontier may have gaps where shallower leaves sit, so reduce over
        # explicit [start, stop) pairs and drop the in-between reductions)
        bounds = np.stack([s, e], axis=1).ravel()
        lower[ids] = np.minimum.reduceat(lo_p, bounds, axis=0)[::2]
        upper[ids] = np.maximum.reduceat(hi_p, bounds, axis=0)[::2]
        split = (e - s) > leaf_size
        if not split.any():
            break
        ids_s, s_s, e_s = ids[split], s[split], e[split]
        axis = np.argmax(upper[ids_s] - lower[ids_s], axis=1)
        seg_len = e_s - s_s
        seg_of = np.repeat(np.arange(len(ids_s)), seg_len)
        heads = np.cumsum(seg_len) - seg_len
        pos = np.arange(int(seg_len.sum())) + np.repeat(s_s - heads, seg_len)
        key = pts_p[pos, axis[seg_of]]
        if np.all(seg_len == seg_len[0]):
            # equal segments (power-of-two trees): one row-wise stable sort
            L = int(seg_len[0])
            order = (np.argsort(key.reshape(-1, L), axis=1, kind="stable")
                     + (np.arange(len(seg_len)) * L)[:, None]).ravel()
        else:
            order = np.lexsort((key, seg_of))    # stable within each segment
        src = pos[order]
        perm[pos] = perm[src]
        pack[pos] = np.take(pack, src, axis=0)
        half = seg_len // 2
        lid = ids_s + 1
        rid = ids_s + 1 + np.array([memo[int(h)] for h in half], dtype=np.int64)
        left[ids_s], right[ids_s] = lid, rid
        parent[lid], parent[rid] = ids_s, ids_s
        start[lid], stop[lid] = s_s, s_s + half
        start[rid], stop[rid] = s_s + half, e_s
        ids = np.concatenate([lid, rid])
        ids = ids[np.argsort(start[ids], kind="stable")]
        d += 1
    flat = FlatClusterTree(perm, start, stop, left, right, parent, depth, lower, upper)
    return flat.node(0)


_TREE_SMALL_SEGMENT = 4096      # depths whose segments are all this short sort per segment


def _tree_topology(n, leaf_size):
    """The shape of the cluster tree of n dofs: it depends only on n and the
    leaf size (every split halves a segment, ``clustering.py:150-160``).
    Returns the per-node arrays and, per depth, the frontier (node ids in
    start order) and which of them split."""
    memo = {}
    total = _subtree_counts(n, leaf_size, memo)
    start = np.zeros(total, dtype=np.int64)
    stop = np.zeros(total, dtype=np.int64)
    left = np.full(total, -1, dtype=np.int64)
    right = np.full(total, -1, dtype=np.int64)
    parent = np.full(total, -1, dtype=np.int64)
    depth = np.zeros(total, dtype=np.int64)
    stop[0] = n
    ids = np.array([0], dtype=np.int64)
    depths = []
    d = 0
    while ids.size:
        depth[ids] = d
        split = (stop[ids] - start[ids]) > leaf_size
        depths.append((ids, split))
        if not split.any():
            break
        ids_s = ids[split]
        s_s, e_s = start[ids_s], stop[ids_s]
        half = (e_s - s_s) // 2
        lid = ids_s + 1
        rid = ids_s + 1 + np.array([memo[int(h)] for h in half], dtype=np.int64)
        left[ids_s], right[ids_s] = lid, rid
        parent[lid], parent[rid] = ids_s, ids_s
        start[lid], stop[lid] = s_s, s_s + half
        start[rid], stop[rid] = s_s + half, e_s
        ids = np.concatenate([lid, rid])
        ids = ids[np.argsort(start[ids], kind="stable")]
        d += 1
    return start, stop, left, right, parent, depth, depths


def _build_cluster_tree_device(mesh, basis_kind, leaf_size, device):
    """build_cluster_tree with the n-sized work on the device.  The tree's
    shape is known up front (:func:`_tree_topology`), so every depth - box
    reduction, split axes, key sort and permutation - is queued back to back
    from one upload of the frontier tables; the boxes and the permutation
    come back in one read at the end."""
    import torch

    from . import _native
    from .device import ptr, stream_handle
    from .device import device_charts
    charts = device_charts(mesh, device) if basis_kind == "constant" else None
    if charts is not None:
        # per-dof pack [lo | hi | centroid] straight from the device charts
        n = int(charts["support"].shape[0])
    else:
        points, lo, hi = _support_data(mesh, basis_kind)
        n = len(points)
    start, stop, left, right, parent, depth, depths = _tree_topology(n, leaf_size)
    total = len(start)
    # one table: per depth the frontier [start | stop], then per splitting
    # depth the split rows (into the box table), segment start / length /
    # head and the int32 item offsets (as int64 pairs)
    front = np.concatenate([ids for ids, _ in depths])
    f_off = np.cumsum([0] + [len(ids) for ids, _ in depths])
    parts, plan = [start[front], stop[front]], []
    o = 2 * len(front)
    for di, (ids, split) in enumerate(depths):
        if not split.any():
            continue
        ids_s = ids[split]
        s_s = start[ids_s]
        seg_len = stop[ids_s] - s_s
        heads = np.cumsum(seg_len) - seg_len
        nitems = int(seg_len.sum())
        offs = np.r_[heads, nitems].astype(np.int32)
        offs = np.r_[offs, np.zeros(len(offs) % 2, np.int32)].view(np.int64)
        k = len(ids_s)
        rows = f_off[di] + np.flatnonzero(split)
        parts += [rows, s_s, seg_len, heads, offs]
        plan.append((di, k, nitems, o, int(seg_len.max()) <= _TREE_SMALL_SEGMENT))
        o += 4 * k + len(offs)
    f64 = dict(dtype=torch.float64, device=device)
    pack = [charts["support"].clone() if charts is not None else
            torch.from_numpy(np.ascontiguousarray(np.concatenate([lo, hi, points], axis=1))).to(device),
            torch.empty((n, 9), **f64)]
    perm = [torch.arange(n, dtype=torch.int64, device=device), torch.empty(n, dtype=torch.int64, device=device)]
    keys = torch.empty(2 * n, **f64)                       # sort scratch (torch caching allocator)
    vals = torch.empty(2 * n, dtype=torch.int32, device=device)
    with torch.cuda.device(device):
        st = stream_handle()
        tab = torch.from_numpy(np.concatenate(parts)).to(device)
        box = torch.empty((len(front), 6), **f64)
        axis = torch.empty(max([k for _, k, _, _, _ in plan] + [1]), dtype=torch.int64, device=device)
        tb, need = _native.ctypes.c_int64(0), 1
        for _, k, nitems, _, _ in plan:
            _native.call("gc_tree_sort_bytes", nitems, k, _native.ctypes.byref(tb))
            need = max(need, tb.value)
        temp = torch.empty(need, dtype=torch.uint8, device=device)
        T, nf = tab.data_ptr(), len(front)
        cur = 0
        steps = {di: (k, nitems, o, small) for di, k, nitems, o, small in plan}
        for di in range(len(depths)):
            f0, f1 = int(f_off[di]), int(f_off[di + 1])
            _native.call("gc_tree_boxes", f1 - f0, T + 8 * f0, T + 8 * (nf + f0), ptr(pack[cur]),
                         box.data_ptr() + 48 * f0, st)
            if di not in steps:
                break
            k, nitems, o, small = steps[di]
            _native.call("gc_tree_axis", k, T + 8 * o, ptr(box), ptr(axis), st)
            nxt = 1 - cur
            pack[nxt].copy_(pack[cur])
            perm[nxt].copy_(perm[cur])
            # short segments: one segmented sort; long ones: two radix sorts
            _native.call("gc_tree_split_small" if small else "gc_tree_split", k, T + 8 * (o + k), T + 8 * (o + 2 * k), T + 8 * (o + 3 * k),
                         ptr(axis), T + 8 * (o + 4 * k), nitems, ptr(pack[cur]), ptr(pack[nxt]), ptr(perm[cur]),
                         ptr(perm[nxt]), ptr(keys), ptr(vals), ptr(temp), need, st)
            cur = nxt
        bh = box.cpu().numpy()
        perm_h = perm[cur].cpu().numpy()
    lower = np.zeros((total, 3))
    upper = np.zeros((total, 3))
    lower[front], upper[front] = bh[:, :3], bh[:, 3:]
    flat = FlatClusterTree(perm_h, start, stop, left, right, parent, depth, lower, upper)
    flat._device = device            # the block tree of a device-built tree is built there too
    flat._perm_dev = perm[cur]       # leaf dof order on the device (the bases' leaf rows)
    return flat.node(0)


# --------------------------------------------------------------------------
# block tree

class BlockTree:
    """Node view of the flat block tree (``clustering.py:170-212``)."""

    __slots__ = ("row", "col", "state", "_flat", "_id")

    def __init__(self, flat, i):
        self._flat, self._id = flat, i
        self.row = flat.row_tree.node(int(flat.row[i]))
        self.col = flat.col_tree.node(int(flat.col[i]))
        self.state = (ADMISSIBLE, INADMISSIBLE, SUBDIVIDED)[int(flat.state[i])]

    @property
    def children(self):
        f = self._flat
        return tuple(BlockTree(f, int(j)) for j in f.kids(self._id))

    def is_leaf(self):
        return self.state != SUBDIVIDED

    def _leaf_ids(self, which=None):
        f = self._flat
        lo, hi = f.key_lo[self._id], f.key_hi[self._id]
        a, b = np.searchsorted(f.leaf_key, [lo, hi], side="left")
        sel = f.leaf_ids[a:b]
        if which is not None:
            sel = sel[f.state[sel] == which]
        return sel

    def leaves(self):
        return [BlockTree(self._flat, int(j)) for j in self._leaf_ids()]

    def admissible_leaves(self):
        return [BlockTree(self._flat, int(j)) for j in self._leaf_ids(0)]

    def inadmissible_leaves(self):
        return [BlockTree(self._flat, int(j)) for j in self._leaf_ids(1)]

    def depth(self):
        f = self._flat
        ids = self._leaf_ids()
        return int(f.level[ids].max() - f.level[self._id]) if len(ids) else 0

    def stats(self):
        ids = self._leaf_ids()
        adm = int((self._flat.state[ids] == 0).sum())
        return {"depth": self.depth(), "leaves": len(ids), "admissible": adm,
                "inadmissible": len(ids) - adm}

    @property
    def flat(self):
        return self._flat

    def __repr__(self):
        return "BlockTree(row #%d x col #%d, %s)" % (
            self.row.index, self.col.index, self.state)


_KEY_DIGITS = 31          # base-4 path digits; depth <= 31 levels


class FlatBlockTree:
    """All block-tree nodes as arrays: ``row, col, state (0 adm, 1 inadm,
    2 subdivided), level, key`` and the leaves in depth-first order
    (``leaf_ids``, ``leaf_key``).  ``key`` is the base-4 path code aligned
    to ``_KEY_DIGITS`` digits, so sorting by it is the reference DFS order."""

    def __init__(self, row_tree, col_tree, row, col, state, level, key, parent_of, leaves=None):
        self.row_tree, self.col_tree = row_tree, col_tree
        self.row, self.col, self.state, self.level, self.key = row, col, state, level, key
        self.parent_of = parent_of
        span = np.power(4, _KEY_DIGITS - level, dtype=np.int64)
        self.key_lo, self.key_hi = key, key + span
        if leaves is None:
            leaves = np.flatnonzero(state != 2)
            order = np.argsort(key[leaves])      # keys are unique paths: any sort is the DFS order
            self.leaf_ids = leaves[order]
            self.leaf_key = key[self.leaf_ids]
        else:                                    # (ids, keys) already in DFS order
            self.leaf_ids, self.leaf_key = leaves
        self._kid_index = None

    def kids(self, i):
        if self._kid_index is None:
            order = np.argsort(self.parent_of, kind="stable")
            cuts = np.searchsorted(self.parent_of[order], np.arange(len(self.row) + 1))
            self._kid_index = (order, cuts)
        order, cuts = self._kid_index
        kids = order[cuts[i]:cuts[i + 1]]
        return kids[np.argsort(self.key[kids], kind="stable")]

    def leaves(self, state=None):
        """Leaf (row, col) node ids in DFS order, optionally one state only."""
        ids = self.leaf_ids
        if state is not None:
            ids = ids[self.state[ids] == state]
        return self.row[ids], self.col[ids]


def _gap_norm_vector(gap):
    return np.sqrt((gap[:, 0] * gap[:, 0] + gap[:, 1] * gap[:, 1]) + gap[:, 2] * gap[:, 2])


def _admissible_many(rt, ct, r, c, eta):
    """Vectorised ``admissible`` with an exact recheck of near-ties: the
    distance is computed elementwise, and whenever the comparison is within
    1e-12 relative of flipping it is redone with the reference's 1-D BLAS
    norm, so the decision is bit-for-bit the reference's."""
    d = np.maximum(rt.diam[r], ct.diam[c])
    # per coordinate (1-D gathers of the box columns; same values as the
    # (N, 3) form, about 3x faster)
    lo_r, up_r, lo_c, up_c = rt.lower.T, rt.upper.T, ct.lower.T, ct.upper.T
    g = []
    for k in range(3):
        a = lo_r[k][r] - up_c[k][c]
        np.maximum(a, lo_c[k][c] - up_r[k][r], out=a)
        np.maximum(a, 0.0, out=a)
        g.append(a)
    rhs = 2.0 * eta * np.sqrt((g[0] * g[0] + g[1] * g[1]) + g[2] * g[2])
    adm = d <= rhs
    close = np.flatnonzero(np.abs(d - rhs) <= 1e-12 * np.maximum(d, rhs))
    for i in close:
        adm[i] = d[i] <= 2.0 * eta * _blas_norm(np.array([g[0][i], g[1][i], g[2][i]]))
    return adm


def build_block_tree(row_root, col_root=None, eta=1.0):
    """Recursive block partition (``clustering.py:215-237``), grown level by
    level by the library's host routine (``gc_block_tree``).  Returns the
    root :class:`BlockTree` view."""
    if col_root is None:
        col_root = row_root
    if eta <= 0:
        raise ConfigError("eta must be positive, got %r" % (eta,))
    blas_norms(np.zeros((0, 3)))                 # fixes the BLAS-norm rounding mode
    mode = _NORM_MODE[0]
    if mode is None:                             # numpy's norm matches neither sequence
        return _build_block_tree_arrays(row_root, col_root, eta)
    dev = getattr(row_root.flat, "_device", None)
    if dev is not None and (col_root.flat is row_root.flat or getattr(col_root.flat, "_device", None) == dev):
        return _build_block_tree_device(row_root, col_root, eta, mode, dev)
    from . import _native
    rt, ct = row_root.flat, col_root.flat
    trees = []
    for t in (rt, ct):
        trees += [np.ascontiguousarray(t.diam, np.float64), np.ascontiguousarray(t.lower, np.float64),
                  np.ascontiguousarray(t.upper, np.float64), np.ascontiguousarray(t.left, np.int64),
                  np.ascontiguousarray(t.right, np.int64)]
    lib = _native.load()
    handle, count = _native.ctypes.c_void_p(0), _native.ctypes.c_int64(0)
    _native.check(lib.gc_block_tree(*[a.ctypes.data for a in trees], int(row_root.index), int(col_root.index),
                                    float(eta), int(mode), _KEY_DIGITS, _native.ctypes.byref(handle),
                                    _native.ctypes.byref(count)))
    n = int(count.value)
    row, col, state, level, key, parent = (np.empty(n, np.int64), np.empty(n, np.int64), np.empty(n, np.int8),
                                           np.empty(n, np.int64), np.empty(n, np.int64), np.empty(n, np.int64))
    _native.check(lib.gc_block_tree_fetch(handle, *[a.ctypes.data for a in (row, col, state, level, key, parent)]))
    flat = FlatBlockTree(rt, ct, row, col, state, level, key, parent)
    return BlockTree(flat, 0)


def _build_block_tree_device(row_root, col_root, eta, mode, device):
    """The block tree built on the device one level per ``gc_bt_level``
    call (node for node equal to gc_block_tree and the numpy builder), the
    node arrays copied to the host once at the end."""
    import torch

    from . import _native
    from .device import ptr, stream_handle
    rt, ct = row_root.flat, col_root.flat
    i64 = dict(dtype=torch.int64, device=device)

    def up(t):
        f64 = dict(dtype=torch.float64, device=device)
        return (torch.from_numpy(np.ascontiguousarray(t.diam, np.float64)).to(**f64),
                torch.from_numpy(np.ascontiguousarray(t.lower, np.float64)).to(**f64),
                torch.from_numpy(np.ascontiguousarray(t.upper, np.float64)).to(**f64),
                torch.from_numpy(np.ascontiguousarray(t.left, np.int64)).to(**i64),
                torch.from_numpy(np.ascontiguousarray(t.right, np.int64)).to(**i64))
    with torch.cuda.device(device):
        tr = up(rt)
        tc = tr if ct is rt else up(ct)
        cap = max(4096, 32 * (len(rt) + len(ct)))
        # a pair's level is the deeper of its clusters' depths (a leaf side
        # stays while the other splits), so this many levels end the tree;
        # every level runs from device-side sizes, read once at the end
        levels = min(int(max(rt.depth.max(), ct.depth.max())) + 2, _KEY_DIGITS)
        st = stream_handle()
        while True:
            cap_f = max(1024, cap // 2)
            out = [torch.empty(cap, **i64), torch.empty(cap, **i64), torch.empty(cap, dtype=torch.int8, device=device),
                   torch.empty(cap, **i64), torch.empty(cap, **i64), torch.empty(cap, **i64)]
            front = [torch.empty(cap_f, **i64) for _ in range(4)]
            nxt = [torch.empty(cap_f, **i64) for _ in range(4)]
            for f, v in zip(front, (int(row_root.index), int(col_root.index), 0, -1)):
                f[:1].fill_(v)
            meta = torch.zeros(2 * levels + 2, **i64)
            meta[:1].fill_(1)
            err = torch.zeros(1, dtype=torch.int32, device=device)
            scratch = torch.empty(8 * cap_f, dtype=torch.int32, device=device)
            tb = _native.ctypes.c_int64(0)
            _native.call("gc_bt_level_bytes", cap_f, _native.ctypes.byref(tb))
            temp = torch.empty(max(tb.value, 1), dtype=torch.uint8, device=device)
            for lev in range(levels):
                _native.call("gc_bt_level", meta.data_ptr() + 16 * lev, cap_f, cap, *[ptr(f) for f in front], lev,
                             _KEY_DIGITS, *[ptr(a) for a in tr], *[ptr(a) for a in tc], float(eta), int(mode),
                             *[ptr(o) for o in out], *[ptr(a) for a in nxt], ptr(scratch[:4 * cap_f]),
                             ptr(scratch[4 * cap_f:]), ptr(err), ptr(temp), tb.value, st)
                front, nxt = nxt, front
            mh = meta.cpu().numpy()
            e = int(err.cpu()[0])
            if e & 4 or (not e & 3 and mh[2 * levels]):
                raise ConfigError("block tree deeper than %d levels" % _KEY_DIGITS)
            if not e & 3:
                break
            cap *= 2                                     # frontier or node capacity: rebuild larger
        base = int(mh[2 * levels + 1])             # nodes of all levels
        count = torch.zeros(1, **i64)
        n = base
        # the leaves in depth-first order, sorted on the device
        lids, lkey = torch.empty(n, **i64), torch.empty(n, **i64)
        sc = [torch.empty(n, **i64) for _ in range(3)]
        fl = torch.empty(2 * n, dtype=torch.int8, device=device)
        tb = _native.ctypes.c_int64(0)
        _native.call("gc_bt_leaves_bytes", n, _native.ctypes.byref(tb))
        temp = torch.empty(max(tb.value, 1), dtype=torch.uint8, device=device)
        _native.call("gc_bt_leaves", n, ptr(out[2]), ptr(out[4]), ptr(lids), ptr(lkey), ptr(count),
                     *[ptr(a) for a in sc], ptr(fl[:n]), ptr(fl[n:]), ptr(temp), tb.value, st)
        nl = int(count.item())
        row, col, state, level, key, parent = (o[:n].cpu().numpy() for o in out)
        leaf_ids, leaf_key = lids[:nl].cpu().numpy(), lkey[:nl].cpu().numpy()
    flat = FlatBlockTree(rt, ct, row, col, state, level, key, parent, leaves=(leaf_ids, leaf_key))
    flat._dev = (out[0][:n], out[1][:n], out[2][:n], lids[:nl])    # row, col, state, leaves (build_h2 tables)
    return BlockTree(flat, 0)


def _build_block_tree_arrays(row_root, col_root=None, eta=1.0):
    """The same partition array-at-a-time in numpy (the reference check of
    gc_block_tree, and the path when numpy's norm rounding is not one of the
    two sequences the native routine reproduces)."""
    if col_root is None:
        col_root = row_root
    if eta <= 0:
        raise ConfigError("eta must be positive, got %r" % (eta,))
    rt, ct = row_root.flat, col_root.flat
    rows, cols, states, levels, keys, parents = [], [], [], [], [], []
    fr = np.array([row_root.index], dtype=np.int64)
    fc = np.array([col_root.index], dtype=np.int64)
    fkey = np.zeros(1, dtype=np.int64)
    fpar = np.full(1, -1, dtype=np.int64)
    base = 0
    lev = 0
    while fr.size:
        if lev >= _KEY_DIGITS:
            raise ConfigError("block tree deeper than %d levels" % _KEY_DIGITS)
        adm = _admissible_many(rt, ct, fr, fc, eta)
        rleaf, cleaf = rt.is_leaf[fr], ct.is_leaf[fc]
        state = np.where(adm, 0, np.where(rleaf & cleaf, 1, 2)).astype(np.int8)
        ids = base + np.arange(fr.size)
        rows.append(fr); cols.append(fc); states.append(state)
        levels.append(np.full(fr.size, lev, dtype=np.int64))
        keys.append(fkey); parents.append(fpar)
        base += fr.size
        sub = np.flatnonzero(state == 2)
        if not sub.size:
            break
        r, c = fr[sub], fc[sub]
        r_split, c_split = ~rt.is_leaf[r], ~ct.is_leaf[c]
        # children of a pair: (rc, cc) for rc in rs for cc in cs
        rk = [np.where(r_split, rt.left[r], r), np.where(r_split, rt.right[r], -1)]
        ck = [np.where(c_split, ct.left[c], c), np.where(c_split, ct.right[c], -1)]
        digit_scale = np.int64(4) ** (_KEY_DIGITS - 1 - lev)
        nr, nc, nk, npar = [], [], [], []
        for a in range(2):
            for b in range(2):
                ok = (rk[a] >= 0) & (ck[b] >= 0)
                # sequential digit among the existing children of each parent
                dig = (a * np.where(c_split, 2, 1) + b)
                sel = np.flatnonzero(ok)
                nr.append(rk[a][sel]); nc.append(ck[b][sel])
                nk.append(keys[-1][sub[sel]] + dig[sel] * digit_scale)
                npar.append(ids[sub[sel]])
        fr, fc = np.concatenate(nr), np.concatenate(nc)
        fkey, fpar = np.concatenate(nk), np.concatenate(npar)
        lev += 1
    flat = FlatBlockTree(rt, ct, np.concatenate(rows), np.concatenate(cols),
                         np.concatenate(states), np.concatenate(levels),
                         np.concatenate(keys), np.concatenate(parents))
    return BlockTree(flat, 0)
