"""Tiered transforms of the H^2 matvec (the forward / backward transforms of
``h2.py:63-80``, regrouped for the B200).

The reference applies a nested basis level by level: x-hat of a node is
its transfer matrix times the x-hat of its two children (``h2.py:63-70``),
and the backward transform mirrors it top-down (``h2.py:74-80``).  On the
device every level is one dependent launch, and while the coupling phase
streams HBM each level costs a loaded memory round trip plus a wait for
SM slots: at sphere level 6 the 16 transform levels alone take ~100 us
of a ~145 us product.

A *tier* is a run of consecutive tree heights (lo, hi].  Its nodes are
applied in ONE launch from the x-hat of the tier's *frontier* - the live
nodes at height <= lo whose parent is in the tier - or, for the lowest
tier (lo = -1), from the degrees of freedom of the live leaves:

    x-hat_u = M_u^T [x-hat_f1; x-hat_f2; ...],
    M_u = stack over live children c of (M_c E_c   if c is in the tier,
                                         E_c       if c is a frontier node),
    M_leaf = V_leaf,

E_c being the rows of the parent's V-hat that belong to c.  M_u is the
nested basis multiplied out across the tier, so the result equals the
level-by-level one up to rounding (the matvec tolerance, not bit-exact).
The backward transform of a tier reads the same blocks transposed and
grouped per frontier node (lowest tier: per live leaf, written straight
into the output rows).  Tier boundaries are chosen by a dynamic programme
over heights minimising (extra bytes streamed) / bandwidth + launches x
latency; single-height tiers reproduce the level-by-level transform.
"""
import numpy as np
import torch

from . import _native
from .device import padded_empty, ptr, stream_handle, to_dev

_BW = 6.5e12             # B/s, the measured HBM copy bandwidth (MEASURED_PEAKS.json)
_LATENCY_S = 5e-6        # hand-off between dependent tier launches
_CTA_BPS = 20e9          # one CTA's streaming rate (B/s)


def live_nodes(store):
    return store.materialized & (store.rank > 0)


def _pairs(store, flat, lo, hi, ordered=True):
    """(u, f) pairs of tier (lo, hi]: u a live tier node, f a frontier
    element under it (a frontier node, or for lo < 0 a live leaf, the leaf
    itself included), plus the element weights w_f (rank, or leaf size).
    ``ordered``: sorted by (u, position of f) - the layout of M_u."""
    live = live_nodes(store)
    H = flat.height
    par = flat.parent
    if lo < 0:
        elems = np.flatnonzero(live & flat.is_leaf)
        w = store.rows[elems]
        us, fs = [elems], [elems]
        cur, src = elems, elems
    else:
        p = np.where(par >= 0, par, 0)
        cand = live & (H <= lo) & (par >= 0)
        cand &= live[p] & (H[p] > lo) & (H[p] <= hi)
        elems = np.flatnonzero(cand)
        w = store.rank[elems]
        us, fs = [], []
        cur, src = elems, elems
    wmap = np.zeros(len(flat), np.int64)
    wmap[elems] = w
    while cur.size:
        up = par[cur]
        ok = up >= 0
        up, src = up[ok], src[ok]
        q = np.where(up >= 0, up, 0)
        ok = live[q] & (H[q] <= hi) & (H[q] > lo)
        up, src = up[ok], src[ok]
        if not up.size:
            break
        us.append(up)
        fs.append(src)
        cur = up
    u = np.concatenate(us) if us else np.zeros(0, np.int64)
    f = np.concatenate(fs) if fs else np.zeros(0, np.int64)
    if not ordered:
        return u, f, wmap
    order = np.lexsort((flat.start[f], u))
    return u[order], f[order], wmap


def tier_elems(store, flat, lo, hi):
    """Matrix elements of a tier's composed transfers."""
    u, f, wmap = _pairs(store, flat, lo, hi)
    return int((wmap[f] * store.rank[u]).sum())


def choose_tiers(store, flat, bounds=None, latency_s=None, cta_bps=None, max_rows=1024):
    """Tier upper boundaries (ascending heights) for one transform
    direction of one store: minimise, summed over tiers, streamed bytes /
    HBM bandwidth + the largest work item / one CTA's streaming rate
    (``cta_bps``) + the hand-off latency between dependent phases
    (``latency_s``); a panel's work items hold at most ``max_rows`` rows
    (h2.PanelPlan).  ``bounds`` (a list of heights) overrides the choice."""
    live = live_nodes(store)
    if not live.any():
        return []
    top = int(flat.height[live].max())
    if bounds is not None:
        return sorted({min(int(v), top) for v in bounds} | {top})
    lat = _LATENCY_S if latency_s is None else latency_s
    cta_bw = _CTA_BPS if cta_bps is None else cta_bps
    # elems(lo, hi) for every hi from ONE walk per lo: the pairs of tier
    # (lo, hi] are those of (lo, top] whose u lies at height <= hi.  A tier
    # launch costs its bytes at full bandwidth plus its largest work item
    # (<= 1024 rows of one panel) streamed by one CTA (the max of the two
    # measured worse: L6 (5, 7) at 4.85 TB/s) plus a launch latency.
    cost = {}
    for lo in range(-1, top):
        u, f, wmap = _pairs(store, flat, lo, top, ordered=False)     # sums only
        el = (wmap[f] * store.rank[u]).astype(np.float64)
        per_h = np.bincount(flat.height[u], weights=el, minlength=top + 1)
        acc = np.cumsum(per_h)
        m = np.bincount(u, weights=wmap[f].astype(np.float64), minlength=len(flat))
        nodes = np.flatnonzero(np.bincount(u, minlength=len(flat)))
        item = np.minimum(m[nodes], max_rows) * store.rank[nodes] * 8.0
        big = np.zeros(top + 1)
        np.maximum.at(big, flat.height[nodes], item)
        big = np.maximum.accumulate(big)
        for hi in range(lo + 1, top + 1):
            cost[lo, hi] = 8.0 * acc[hi] / _BW + big[hi] / cta_bw + lat
    best = {-1: (0.0, [])}
    for hi in range(0, top + 1):
        best[hi] = min(((best[lo][0] + cost[lo, hi], best[lo][1] + [hi]) for lo in range(-1, hi)),
                       key=lambda c: c[0])
    return best[top][1]


def tier_tables(store, flat, bounds):
    """Host-side plan of a store's tiers: per tier the (u, f) pair table,
    the positions of f inside M_u, m_u and the offsets of the blocks M_u
    in one buffer; plus the composition descriptors (one (n, 6) array per
    launch, children before parents; gc_tier_compose) and the total
    element count."""
    tiers, launches, total = [], [], 0
    H, live, k = flat.height, live_nodes(store), store.rank
    lo = -1
    for hi in bounds:
        u, f, wmap = _pairs(store, flat, lo, hi)
        nodes = u[np.r_[True, u[1:] != u[:-1]]] if u.size else u      # u is sorted
        m = np.zeros(len(flat), np.int64)
        np.add.at(m, u, wmap[f])
        moff = np.full(len(flat), -1, np.int64)
        sizes = m[nodes] * k[nodes]
        if nodes.size:
            moff[nodes] = total + np.concatenate([[0], np.cumsum(sizes)[:-1]])
        total += int(sizes.sum())
        # position of f inside u's stack: exclusive cumsum of w per u group
        wf = wmap[f]
        cs = np.cumsum(wf) - wf
        first = np.r_[0, np.flatnonzero(u[1:] != u[:-1]) + 1] if u.size else np.zeros(0, np.int64)
        pos = cs - np.repeat(cs[first], np.diff(np.r_[first, u.size])) if u.size else cs
        tiers.append(dict(lo=lo, hi=hi, u=u, f=f, w=wf, pos=pos, nodes=nodes, m=m, moff=moff))
        for h in np.unique(H[nodes]):
            ids = nodes[H[nodes] == h]
            desc = []
            lv = ids[flat.is_leaf[ids] & (lo < 0)]
            if lv.size:                                  # M_leaf = V_leaf
                z = np.zeros_like(lv)
                desc.append(np.stack([z - 1, store.rows[lv], z, store.v_off[lv], k[lv], moff[lv]], 1))
            inner = ids[~flat.is_leaf[ids]]
            if inner.size:
                ku = k[inner]
                row_off = np.zeros(inner.size, np.int64)
                for c in (flat.left[inner], flat.right[inner]):
                    lc = live[c]
                    intier = lc & (H[c] > lo)
                    mc = np.where(intier, m[c], np.where(lc, k[c], 0))
                    desc.append(np.stack([np.where(intier, moff[c], -1), mc, k[c],
                                          store.v_off[inner] + store.child_row[c] * ku, ku,
                                          moff[inner] + row_off * ku], 1)[lc])
                    row_off = row_off + mc
            if desc:
                launches.append(np.ascontiguousarray(np.concatenate(desc), np.int64))
        lo = hi
    return tiers, launches, total


def transpose_tables(tiers, store, flat):
    """The backward blocks: per tier, per output element (frontier node;
    lowest tier: live leaf) the stack over its tier ancestors u (bottom
    up) of the rows of M_u that map to it, transposed (k_u x w_f
    row-major).  Returns the per-tier groups, the (n, 5) descriptors
    (gc_block_transpose) and the total element count."""
    k = store.rank
    out, total, desc = [], 0, []
    for t in tiers:
        u, f, w, pos, moff = t["u"], t["f"], t["w"], t["pos"], t["moff"]
        order = np.lexsort((flat.height[u], f))
        uu, ff, ww, pp = u[order], f[order], w[order], pos[order]
        blk = k[uu] * ww
        first = np.r_[0, np.flatnonzero(ff[1:] != ff[:-1]) + 1] if ff.size else np.zeros(0, np.int64)
        dst = total + np.concatenate([[0], np.cumsum(blk)[:-1]]) if ff.size else np.zeros(0, np.int64)
        total += int(blk.sum())
        desc.append(np.stack([moff[uu] + pp * k[uu], k[uu], ww, k[uu], dst], 1))
        out.append(dict(first=first, u=uu, f=ff, w=ww, dst=dst))
    d = np.ascontiguousarray(np.concatenate(desc) if desc else np.zeros((0, 5), np.int64), np.int64)
    return out, d, total


class StoreTiers:
    """Composed transfers of one basis store for the given tiers, on the
    device: ``M`` (forward blocks M_u, row-major m_u x k_u) and the
    per-tier pair tables the phases are built from."""

    def __init__(self, store, flat, bounds, dev):
        self.bounds = bounds
        self.store, self.flat = store, flat
        self.tiers, launches, total = tier_tables(store, flat, bounds)
        self.M = padded_empty(max(total, 1), dev)     # streamed by 16-byte bulk copies
        self.elems = total
        st = stream_handle()
        tile = int(_native.load().gc_tier_tile())
        for desc in launches:                    # children before parents
            nt = -(-(desc[:, 1] * desc[:, 4]) // tile)
            idx = np.repeat(np.arange(len(desc)), nt)
            first = (np.arange(int(nt.sum())) - np.repeat(np.cumsum(nt) - nt, nt)) * tile
            tl = to_dev(np.ascontiguousarray(np.stack([idx, first], 1), np.int64), dev)
            dd = to_dev(desc, dev)
            _native.call("gc_tier_compose", len(idx), ptr(tl), ptr(dd), ptr(store.V), ptr(self.M), st)

    def transposed(self, dev):
        """(per-tier groups, device buffer) of the backward blocks."""
        groups, desc, total = transpose_tables(self.tiers, self.store, self.flat)
        MT = padded_empty(max(total, 1), dev)
        if len(desc):
            dd = to_dev(desc, dev)
            _native.call("gc_block_transpose", len(desc), ptr(dd), ptr(self.M), ptr(MT), stream_handle())
        return groups, MT
