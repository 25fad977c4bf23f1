"""Host-side plan of the tiered transforms (paper_1810_08429_b200/tiers.py),
checked on CPU: the composition / transposition descriptors, executed by a
numpy interpreter of the two plan kernels (csrc/tiers.cu) and of the panel
product, reproduce the level-by-level nested-basis transforms of the
reference (h2.py:63-80) on a real cluster tree with a random nested basis,
including rank-0 (dead) nodes and a materialised forest below the root."""
import types

import numpy as np
import pytest

from paper_1810_08429_b200 import geometry, tiers
from paper_1810_08429_b200.clustering import build_cluster_tree


def _store(flat, rng, dead_frac=0.1, forest=False):
    n = len(flat)
    order = np.argsort(flat.height, kind="stable")          # children before parents
    mat = np.ones(n, bool)
    if forest:                                               # drop the top two levels
        mat[flat.depth < 2] = False
    rank = np.zeros(n, np.int64)
    rows = np.zeros(n, np.int64)
    child_row = np.zeros(n, np.int64)
    size = flat.stop - flat.start
    for i in order:
        if not mat[i]:
            continue
        if flat.is_leaf[i]:
            rows[i] = size[i]
        else:
            l, r = flat.left[i], flat.right[i]
            child_row[l], child_row[r] = 0, rank[l]
            rows[i] = rank[l] + rank[r]
        rank[i] = 0 if rng.random() < dead_frac else int(rng.integers(1, max(rows[i], 1) + 1)) if rows[i] else 0
    v_off = np.full(n, -1, np.int64)
    pos = 0
    for i in range(n):
        if mat[i]:
            v_off[i] = pos
            pos += rows[i] * rank[i]
    coef_off = np.full(n, -1, np.int64)
    c = 0
    for i in range(n):
        if mat[i]:
            coef_off[i] = c
            c += rank[i]
    return types.SimpleNamespace(materialized=mat, rank=rank, rows=rows, child_row=child_row, v_off=v_off,
                                 coef_off=coef_off, V=rng.standard_normal(max(pos, 1)), coef_size=c)


def _vmat(s, i):
    return s.V[s.v_off[i]:s.v_off[i] + s.rows[i] * s.rank[i]].reshape(s.rows[i], s.rank[i])


def _forward_ref(s, flat, x):
    """x-hat level by level (h2.py:63-70)."""
    xh = np.zeros(s.coef_size)
    live = tiers.live_nodes(s)
    for i in np.argsort(flat.height, kind="stable"):
        if not live[i]:
            continue
        if flat.is_leaf[i]:
            inp = x[flat.start[i]:flat.stop[i]]
        else:
            parts = [xh[s.coef_off[c]:s.coef_off[c] + s.rank[c]] for c in (flat.left[i], flat.right[i])]
            inp = np.concatenate(parts)
        xh[s.coef_off[i]:s.coef_off[i] + s.rank[i]] = _vmat(s, i).T @ inp
    return xh


def _backward_ref(s, flat, yh, n):
    """y = sum over nodes of the expanded basis times y-hat (h2.py:74-80)."""
    tot = yh.copy()
    live = tiers.live_nodes(s)
    y = np.zeros(n)
    for i in np.argsort(-flat.height, kind="stable"):
        if not live[i]:
            continue
        v = _vmat(s, i) @ tot[s.coef_off[i]:s.coef_off[i] + s.rank[i]]
        if flat.is_leaf[i]:
            y[flat.start[i]:flat.stop[i]] += v
        else:
            for c in (flat.left[i], flat.right[i]):
                if live[c]:
                    tot[s.coef_off[c]:s.coef_off[c] + s.rank[c]] += v[s.child_row[c]:s.child_row[c] + s.rank[c]]
    return y


def _compose(s, launches, total):
    M = np.full(max(total, 1), np.nan)
    for desc in launches:
        for s_off, m, kc, e_off, ku, o in desc:
            if s_off < 0:
                blk = s.V[e_off:e_off + m * ku].reshape(m, ku)
            else:
                blk = M[s_off:s_off + m * kc].reshape(m, kc) @ s.V[e_off:e_off + kc * ku].reshape(kc, ku)
            M[o:o + m * ku] = blk.ravel()
    return M


def _transpose(M, desc, total):
    MT = np.full(max(total, 1), np.nan)
    for s_off, ld, rows, cols, o in desc:
        src = np.lib.stride_tricks.as_strided(M[s_off:], shape=(rows, cols), strides=(8 * ld, 8))
        MT[o:o + rows * cols] = src.T.ravel()
    return MT


@pytest.mark.parametrize("bounds,forest", [([0, 1, 2, 3, 4, 5], False), ([2, 5], False), ([5], False),
                                           ([1, 3, 5], True), (None, False)])
def test_tier_plan_reproduces_level_by_level(bounds, forest):
    mesh = geometry.build_sphere_mesh(3)
    flat = build_cluster_tree(mesh, leaf_size=8).flat
    rng = np.random.default_rng(7)
    s = _store(flat, rng, forest=forest)
    top = int(flat.height[tiers.live_nodes(s)].max())
    bounds = tiers.choose_tiers(s, flat) if bounds is None else sorted({min(b, top) for b in bounds} | {top})
    n = int(flat.stop[0])
    x = rng.standard_normal(n)
    tabs, launches, total = tiers.tier_tables(s, flat, bounds)
    M = _compose(s, launches, total)
    assert not np.isnan(M[:total]).any()
    # forward: tier by tier from the dofs / the frontier x-hat
    xh = np.zeros(s.coef_size)
    covered = np.zeros(len(flat), bool)
    for t in tabs:
        for u in t["nodes"]:
            sel = t["u"] == u
            f, w = t["f"][sel], t["w"][sel]
            if t["lo"] < 0:
                inp = np.concatenate([x[flat.start[e]:flat.start[e] + ww] for e, ww in zip(f, w)])
            else:
                inp = np.concatenate([xh[s.coef_off[e]:s.coef_off[e] + ww] for e, ww in zip(f, w)])
            Mu = M[t["moff"][u]:t["moff"][u] + t["m"][u] * s.rank[u]].reshape(t["m"][u], s.rank[u])
            xh[s.coef_off[u]:s.coef_off[u] + s.rank[u]] = Mu.T @ inp
            assert not covered[u]
            covered[u] = True
    assert np.array_equal(covered, tiers.live_nodes(s))
    ref = _forward_ref(s, flat, x)
    assert np.allclose(xh, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
    # backward: top tier first, y-hat-t accumulated per frontier element
    groups, tdesc, ttotal = tiers.transpose_tables(tabs, s, flat)
    MT = _transpose(M, tdesc, ttotal)
    yh = rng.standard_normal(s.coef_size)
    yt = np.zeros(s.coef_size)
    y = np.zeros(n)
    for t, g in reversed(list(zip(tabs, groups))):
        first = g["first"]
        ends = np.r_[first[1:], len(g["f"])]
        for a, b in zip(first, ends):
            e, w = g["f"][a], g["w"][a]
            us = g["u"][a:b]
            K = int(s.rank[us].sum())
            A = MT[g["dst"][a]:g["dst"][a] + K * w].reshape(K, w)
            inp = np.concatenate([(yh + yt)[s.coef_off[u]:s.coef_off[u] + s.rank[u]] for u in us])
            if t["lo"] < 0:
                y[flat.start[e]:flat.start[e] + w] = A.T @ inp
            else:
                yt[s.coef_off[e]:s.coef_off[e] + w] += A.T @ inp
    ref = _backward_ref(s, flat, yh, n)
    assert np.allclose(y, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


def _random_tree(n, rng, leaf=12):
    """A preorder FlatTree with random, unbalanced splits (frontier nodes of
    every tier then sit at many different heights)."""
    from paper_1810_08429_b200.clustering import FlatClusterTree as FlatTree
    start, stop, left, right, parent, depth = [], [], [], [], [], []

    def node(lo, hi, par, d):
        i = len(start)
        start.append(lo); stop.append(hi); left.append(-1); right.append(-1); parent.append(par); depth.append(d)
        if hi - lo > leaf or (hi - lo > 1 and rng.random() < 0.2):
            cut = int(rng.integers(lo + 1, hi))
            left[i] = node(lo, cut, i, d + 1)
            right[i] = node(cut, hi, i, d + 1)
        return i
    node(0, n, -1, 0)
    a = [np.asarray(v, np.int64) for v in (start, stop, left, right, parent, depth)]
    z = np.zeros((len(start), 3))
    return FlatTree(np.arange(n), *a, z, z + 1.0)


@pytest.mark.parametrize("seed,bounds", [(1, None), (2, [1, 4]), (3, [0, 2, 5]), (4, [3])])
def test_tier_plan_unbalanced_tree(seed, bounds):
    """The same check on random unbalanced trees with dead nodes and a
    forest: frontier elements at mixed heights, tiers built from both."""
    rng = np.random.default_rng(seed)
    flat = _random_tree(700, rng)
    s = _store(flat, rng, dead_frac=0.15, forest=seed % 2 == 0)
    live = tiers.live_nodes(s)
    top = int(flat.height[live].max())
    b = tiers.choose_tiers(s, flat) if bounds is None else sorted({min(v, top) for v in bounds} | {top})
    n = int(flat.stop[0])
    x = rng.standard_normal(n)
    tabs, launches, total = tiers.tier_tables(s, flat, b)
    M = _compose(s, launches, total)
    xh = np.zeros(s.coef_size)
    for t in tabs:
        for u in t["nodes"]:
            sel = t["u"] == u
            f, w = t["f"][sel], t["w"][sel]
            src = [x[flat.start[e]:flat.start[e] + ww] if t["lo"] < 0 else xh[s.coef_off[e]:s.coef_off[e] + ww]
                   for e, ww in zip(f, w)]
            Mu = M[t["moff"][u]:t["moff"][u] + t["m"][u] * s.rank[u]].reshape(t["m"][u], s.rank[u])
            xh[s.coef_off[u]:s.coef_off[u] + s.rank[u]] = Mu.T @ np.concatenate(src)
    ref = _forward_ref(s, flat, x)
    assert np.allclose(xh, ref, rtol=1e-11, atol=1e-11 * np.abs(ref).max())
    groups, tdesc, ttotal = tiers.transpose_tables(tabs, s, flat)
    MT = _transpose(M, tdesc, ttotal)
    yh = rng.standard_normal(s.coef_size)
    yt = np.zeros(s.coef_size)
    y = np.zeros(n)
    for t, g in reversed(list(zip(tabs, groups))):
        ends = np.r_[g["first"][1:], len(g["f"])]
        for a, e_ in zip(g["first"], ends):
            e, w = g["f"][a], g["w"][a]
            us = g["u"][a:e_]
            K = int(s.rank[us].sum())
            A = MT[g["dst"][a]:g["dst"][a] + K * w].reshape(K, w)
            inp = np.concatenate([(yh + yt)[s.coef_off[u]:s.coef_off[u] + s.rank[u]] for u in us])
            if t["lo"] < 0:
                y[flat.start[e]:flat.start[e] + w] = A.T @ inp
            else:
                yt[s.coef_off[e]:s.coef_off[e] + w] += A.T @ inp
    ref = _backward_ref(s, flat, yh, n)
    assert np.allclose(y, ref, rtol=1e-11, atol=1e-11 * np.abs(ref).max())


def test_choose_tiers_override_and_cost():
    mesh = geometry.build_sphere_mesh(3)
    flat = build_cluster_tree(mesh, leaf_size=8).flat
    s = _store(flat, np.random.default_rng(1), dead_frac=0.0)
    top = int(flat.height.max())
    assert tiers.choose_tiers(s, flat, bounds=[1, 3]) == [1, 3, top]
    # no hand-off latency and a fast single CTA: the cheapest plan streams
    # the fewest bytes, which is the level-by-level one (every composed tier
    # is at least as large)
    lvl = tiers.choose_tiers(s, flat, latency_s=0.0, cta_bps=1e21)
    assert lvl == list(range(top + 1))
    # huge latency: one tier
    assert tiers.choose_tiers(s, flat, latency_s=1.0, cta_bps=1e21) == [top]
    # a slow single CTA makes the large composed panels of a tall tier
    # expensive: the plan gets more tiers than with bytes alone
    assert (len(tiers.choose_tiers(s, flat, latency_s=1e-6, cta_bps=1e6))
            > len(tiers.choose_tiers(s, flat, latency_s=1.0, cta_bps=1e6)))


def test_coef_layout_generations_equal_queue_order():
    """gca.coef_layout (one BFS generation per numpy step) == the explicit
    FIFO-queue layout, on random unbalanced trees and root sets."""
    from paper_1810_08429_b200 import gca
    for seed in range(10):
        rng = np.random.default_rng(seed)
        flat = _random_tree(400, rng)
        rank = rng.integers(0, 20, len(flat))
        roots = np.flatnonzero(flat.depth == min(2, int(flat.depth.max())))
        rng.shuffle(roots)
        a = gca.coef_layout(flat, roots, rank, base=3)
        b = gca._coef_layout_queue(flat, roots, rank, base=3)
        assert np.array_equal(a[0], b[0]) and a[1] == b[1]
