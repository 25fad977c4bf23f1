"""CPU restatement of the reference's hot-path arithmetic (numpy).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
cpu_baseline leg of bench.py may import this module, and only as the
checker; the product (paper_1810_08429_b200) never calls it.

Every function restates one reference routine (paths relative to
/root/reference/pkg/src/greencross) with the same floating-point operation
order, so on the same host it reproduces the reference bit for bit; that
claim is pinned by tests/test_oracle.py against the fixtures in
tests/golden/ (generated from the reference itself by
tests/golden/make_golden.py).
"""

import numpy as np

FOUR_PI = 4.0 * np.pi

# ---------------------------------------------------------------- rules
# quadrature.py:49-76


def gauss01(m):
    p, w = np.polynomial.legendre.leggauss(m)
    return 0.5 * (p + 1.0), 0.5 * w


def triangle_rule(q):
    s, ws = gauss01(q)
    S, T = np.meshgrid(s, s, indexing="ij")
    return (np.column_stack([(S * (1.0 - T)).ravel(), (S * T).ravel()]),
            (np.outer(ws, ws) * S).ravel())


def shape6(xh):
    """geometry.py:213-225"""
    x, y = xh[..., 0], xh[..., 1]
    l0 = 1.0 - x - y
    return np.stack([l0 * (2.0 * l0 - 1.0), x * (2.0 * x - 1.0), y * (2.0 * y - 1.0),
                     4.0 * l0 * x, 4.0 * x * y, 4.0 * y * l0], axis=-1)


PERMS3 = np.array([[0, 1, 2], [1, 2, 0], [2, 0, 1], [0, 2, 1], [2, 1, 0], [1, 0, 2]])
_MID = {frozenset((0, 1)): 3, frozenset((1, 2)): 4, frozenset((0, 2)): 5}
ORDER6 = np.array([[p[0], p[1], p[2], _MID[frozenset((p[0], p[1]))],
                    _MID[frozenset((p[1], p[2]))], _MID[frozenset((p[2], p[0]))]]
                   for p in PERMS3.tolist()])


def sauter(case, q):
    """quadrature.py:211-284 (relative coordinates, symmetrised edge rule)."""
    g, w = gauss01(q)
    xi, e1, e2, e3 = (a.ravel() for a in np.meshgrid(g, g, g, g, indexing="ij"))
    w4 = np.einsum("i,j,k,l->ijkl", w, w, w, w).ravel()
    parts = []
    if case == 3:
        jac = xi ** 3 * e1 ** 2 * e2
        v = (xi, xi * e1, xi * e1 * e2, xi * e1 * e2 * e3)
        for z in ((v[0], v[0] - v[1] + v[2], v[3], v[2]),
                  (v[0], v[1] - v[2] + v[3], v[2], v[3]),
                  (v[0] - v[3], v[1] - v[3], -v[3], v[2] - v[3])):
            parts += [(z[0], z[1], z[0] - z[2], z[1] - z[3], jac),
                      (z[0] - z[2], z[1] - z[3], z[0], z[1], jac)]
    elif case == 1:
        jac = xi ** 3 * e2
        parts = [(xi, xi * e1, xi * e2, xi * e2 * e3, jac),
                 (xi * e2, xi * e2 * e3, xi, xi * e1, jac)]
    elif case == 2:
        ja, jb = xi ** 3 * e1 ** 2, xi ** 3 * e1 ** 2 * e2
        for (a, b, c, d), j in (
                ((xi, -xi * e1 * e2, xi * e1 * (1.0 - e2), xi * e1 * e3), ja),
                ((xi, -xi * e1 * e2 * e3, xi * e1 * e2 * (1.0 - e3), xi * e1), jb),
                ((xi * (1.0 - e1 * e2), xi * e1 * e2, xi * e1 * e2 * e3, xi * e1 * (1.0 - e2)), jb),
                ((xi * (1.0 - e1 * e2 * e3), xi * e1 * e2 * e3, xi * e1,
                  xi * e1 * e2 * (1.0 - e3)), jb),
                ((xi * (1.0 - e1 * e2 * e3), xi * e1 * e2 * e3, xi * e1 * e2,
                  xi * e1 * (1.0 - e2 * e3)), jb)):
            parts.append((a, d, a + b, c, j))
    x = np.concatenate([np.column_stack([p[0] - p[1], p[1]]) for p in parts])
    y = np.concatenate([np.column_stack([p[2] - p[3], p[3]]) for p in parts])
    wt = np.concatenate([w4 * p[4] for p in parts])
    if case == 2:
        fl = lambda u: np.stack([1.0 - u[:, 0] - u[:, 1], u[:, 1]], axis=1)
        x, y = np.concatenate([x, fl(y)]), np.concatenate([y, fl(x)])
        wt = np.concatenate([0.5 * wt, 0.5 * wt])
    return x, y, wt


def classify(rt, ct):
    """quadrature.py:129-171: case = #shared vertices, alignment perms."""
    hit = rt[:, :, None] == ct[:, None, :]
    rh, ch = hit.any(2), hit.any(1)
    case = rh.sum(1)
    px = np.zeros(len(rt), dtype=np.int64)
    py = np.zeros(len(rt), dtype=np.int64)
    for i in np.flatnonzero(case == 1):
        px[i], py[i] = np.argmax(rh[i]), np.argmax(ch[i])
    for i in np.flatnonzero(case == 2):
        bits = int(rh[i, 0]) + 2 * int(rh[i, 1]) + 4 * int(rh[i, 2])
        rot = {3: 0, 6: 1, 5: 2}[bits]
        px[i] = rot
        c0 = int(np.argmax(ct[i] == rt[i, PERMS3[rot, 0]]))
        c1 = int(np.argmax(ct[i] == rt[i, PERMS3[rot, 1]]))
        py[i] = [tuple(p) for p in PERMS3.tolist()].index((c0, c1, 3 - c0 - c1))
    return case, px, py


# ---------------------------------------------------------------- geometry
# geometry.py:266-293 (plane charts)

def chart_nodes(vertices, triangles):
    nodes = np.empty((len(triangles), 6, 3))
    nodes[:, :3] = vertices[triangles]
    nodes[:, 3] = 0.5 * (nodes[:, 0] + nodes[:, 1])
    nodes[:, 4] = 0.5 * (nodes[:, 1] + nodes[:, 2])
    nodes[:, 5] = 0.5 * (nodes[:, 2] + nodes[:, 0])
    # chart partials at the six reference nodes (geometry.py:228-246), the
    # normal at node 0 and its norm
    ref = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [0.5, 0.0], [0.5, 0.5], [0.0, 0.5]])
    x, y = ref[:, 0], ref[:, 1]
    l0 = 1.0 - x - y
    z = np.zeros(6)
    gx = np.stack([1.0 - 4.0 * l0, 4.0 * x - 1.0, z, 4.0 * (l0 - x), 4.0 * y, -4.0 * y], 1)
    gy = np.stack([1.0 - 4.0 * l0, z, 4.0 * y - 1.0, -4.0 * x, 4.0 * x, 4.0 * (l0 - y)], 1)
    du = np.einsum("ma,tac->tmc", gx, nodes)
    dv = np.einsum("ma,tac->tmc", gy, nodes)
    gram = np.linalg.norm(np.cross(du, dv)[:, 0], axis=1)
    return nodes, gram


def chart_normals(vertices, triangles):
    """Unnormalised chart normals at the six nodes (geometry.py:281-290):
    for plane charts the node-0 normal repeated (|n| = gram)."""
    nodes, _ = chart_nodes(vertices, triangles)
    ref = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [0.5, 0.0], [0.5, 0.5], [0.0, 0.5]])
    x, y = ref[:, 0], ref[:, 1]
    l0 = 1.0 - x - y
    z = np.zeros(6)
    gx = np.stack([1.0 - 4.0 * l0, 4.0 * x - 1.0, z, 4.0 * (l0 - x), 4.0 * y, -4.0 * y], 1)
    gy = np.stack([1.0 - 4.0 * l0, z, 4.0 * y - 1.0, -4.0 * x, 4.0 * x, 4.0 * (l0 - y)], 1)
    n = np.cross(np.einsum("ma,tac->tmc", gx, nodes), np.einsum("ma,tac->tmc", gy, nodes))
    return np.repeat(n[:, :1], 6, axis=1)


def _interp(coef, nodes6):
    """assembly.py:138-143, sequential over the 6 nodes, no BLAS."""
    out = np.zeros((nodes6.shape[0], coef.shape[0], 3))
    for a in range(6):
        out += coef[:, a][None, :, None] * nodes6[:, a][:, None, :]
    return out


# ---------------------------------------------------------------- pair quadrature

def pair_values(nodes, gram, case, rows, cols, px, py, q_reg=3, q_sing=5, kind="slp", normals=None):
    """assembly.py:175-214 for the single layer (or, kind="dlp" with the
    chart ``normals``, the double layer), constant basis, plane charts:
    value per task, same operation order as the reference."""
    if case == 0:
        p, w1 = triangle_rule(q_reg)
        m = len(w1)
        xh, yh, w = np.repeat(p, m, axis=0), np.tile(p, (m, 1)), np.outer(w1, w1).ravel()
    else:
        xh, yh, w = sauter(case, q_sing)
    nx, ny = shape6(xh), shape6(yh)
    out = np.empty(len(rows))
    step = max(1, (1 << 19) // len(w))
    for s in range(0, len(rows), step):
        sl = slice(s, s + step)
        X = _interp(nx, nodes[rows[sl][:, None], ORDER6[px[sl]]])
        Y = _interp(ny, nodes[cols[sl][:, None], ORDER6[py[sl]]])
        D = X - Y
        r2 = D[..., 0] ** 2 + D[..., 1] ** 2 + D[..., 2] ** 2
        r = np.sqrt(r2)
        gx, gy = _gramians(nx, ny, gram, normals, rows[sl], cols[sl], px[sl], py[sl], kind)
        if kind == "dlp":
            nyv = _interp(ny, normals[cols[sl][:, None], ORDER6[py[sl]]])
            dot = D[..., 0] * nyv[..., 0] + D[..., 1] * nyv[..., 1] + D[..., 2] * nyv[..., 2]
            kg = dot / (FOUR_PI * r2 * r) * gx
        else:
            kg = gx * gy / (FOUR_PI * r)
        out[sl] = np.sum(kg * w[None, :], axis=1)
    return out


def _norm3(v):
    return np.sqrt(v[..., 0] ** 2 + v[..., 1] ** 2 + v[..., 2] ** 2)


def _gramians(nx, ny, gram, normals, rows, cols, px, py, kind):
    """Row / column Gramian factors (assembly.py:189-205): the plane
    Gramians, or (gram is None: curved charts) the norms of the interpolated
    node normals at every rule point."""
    if gram is not None:
        return gram[rows][:, None], gram[cols][:, None]
    gx = _norm3(_interp(nx, normals[rows[:, None], ORDER6[px]]))
    gy = None if kind == "dlp" else _norm3(_interp(ny, normals[cols[:, None], ORDER6[py]]))
    return gx, gy


def chart_curved(vertices, triangles, midpoints, tri_edges):
    """geometry.py:266-293 for a CurvedTriangleMesh: chart nodes with the
    curved midpoints and the unnormalised normals at the six nodes."""
    nodes = np.empty((len(triangles), 6, 3))
    nodes[:, :3] = vertices[triangles]
    nodes[:, 3:] = midpoints[tri_edges]
    ref = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [0.5, 0.0], [0.5, 0.5], [0.0, 0.5]])
    x, y = ref[:, 0], ref[:, 1]
    l0 = 1.0 - x - y
    z = np.zeros(6)
    gx = np.stack([1.0 - 4.0 * l0, 4.0 * x - 1.0, z, 4.0 * (l0 - x), 4.0 * y, -4.0 * y], 1)
    gy = np.stack([1.0 - 4.0 * l0, z, 4.0 * y - 1.0, -4.0 * x, 4.0 * x, 4.0 * (l0 - y)], 1)
    n = np.cross(np.einsum("ma,tac->tmc", gx, nodes), np.einsum("ma,tac->tmc", gy, nodes))
    return nodes, n


def _bary(pts):
    return np.stack([1.0 - pts[:, 0] - pts[:, 1], pts[:, 0], pts[:, 1]], axis=1)


def pair_values_linear(nodes, gram, case, rows, cols, px, py, q_reg=3, q_sing=5, kind="slp",
                       normals=None):
    """assembly.py:122-135, 175-214 for the piecewise-linear basis: the
    (B, 3, 3) pair integrals in the canonical permuted local order."""
    if case == 0:
        p, w1 = triangle_rule(q_reg)
        m = len(w1)
        xh, yh, w = np.repeat(p, m, axis=0), np.tile(p, (m, 1)), np.outer(w1, w1).ravel()
    else:
        xh, yh, w = sauter(case, q_sing)
    nx, ny = shape6(xh), shape6(yh)
    wb = np.einsum("m,ma,mb->abm", w, _bary(xh), _bary(yh))
    out = np.empty((len(rows), 3, 3))
    step = max(1, (1 << 19) // len(w))
    for s in range(0, len(rows), step):
        sl = slice(s, s + step)
        X = _interp(nx, nodes[rows[sl][:, None], ORDER6[px[sl]]])
        Y = _interp(ny, nodes[cols[sl][:, None], ORDER6[py[sl]]])
        D = X - Y
        r2 = D[..., 0] ** 2 + D[..., 1] ** 2 + D[..., 2] ** 2
        r = np.sqrt(r2)
        gx, gy = _gramians(nx, ny, gram, normals, rows[sl], cols[sl], px[sl], py[sl], kind)
        if kind == "dlp":
            nyv = _interp(ny, normals[cols[sl][:, None], ORDER6[py[sl]]])
            dot = D[..., 0] * nyv[..., 0] + D[..., 1] * nyv[..., 1] + D[..., 2] * nyv[..., 2]
            kg = dot / (FOUR_PI * r2 * r) * gx
        else:
            kg = gx * gy / (FOUR_PI * r)
        for a in range(3):
            for c in range(3):
                out[sl, a, c] = np.sum(kg * wb[a, c][None, :], axis=1)
    return out


def triangle_table(indices, triangles, nv):
    """assembly.py:54-89: rows (triangle, slot0..2) sorted by triangle, slot
    = 1-based position of the vertex in ``indices`` (0 if absent)."""
    pos = np.zeros(nv, dtype=np.int64)
    pos[np.asarray(indices)] = np.arange(1, len(indices) + 1)
    slots = pos[triangles]
    tri = np.flatnonzero(slots.any(axis=1))
    return np.column_stack([tri, slots[tri]])


def block_linear(nodes, gram, triangles, rows, cols, q=(3, 5), kind="slp", normals=None):
    """Dense linear-basis Galerkin block (assembly.py:279-304, 330-337) with
    the executor's scatter order (batchexec.py:178-209): contributions in
    enqueue order, one np.add.at per (row slot, column slot)."""
    nv = int(triangles.max()) + 1
    tr = triangle_table(rows, triangles, nv)
    tc = triangle_table(cols, triangles, nv)
    nr, nc = len(tr), len(tc)
    R, C = np.repeat(tr[:, 0], nc), np.tile(tc[:, 0], nr)
    rs = np.repeat(tr[:, 1:] - 1, nc, axis=0)
    cs = np.tile(tc[:, 1:] - 1, (nr, 1))
    case, px, py = classify(triangles[R], triangles[C])
    rs = np.take_along_axis(rs, PERMS3[px], axis=1)
    cs = np.take_along_axis(cs, PERMS3[py], axis=1)
    vals = np.empty((len(R), 3, 3))
    for k in range(4):
        m = case == k
        if m.any():
            vals[m] = pair_values_linear(nodes, gram, k, R[m], C[m], px[m], py[m], *q, kind=kind,
                                         normals=normals)
    mat = np.zeros((len(rows), len(cols)))
    for a in range(3):
        for b in range(3):
            ok = (rs[:, a] >= 0) & (cs[:, b] >= 0)
            np.add.at(mat, (rs[ok, a], cs[ok, b]), vals[ok, a, b])
    return mat


def collocation_values(nodes, gram, vertices, case, rows, cols, py, q_reg=3, q_sing=5, kind="slp",
                       normals=None):
    """assembly.py:231-276: single integrals of g(x_v, y) phi_c(y) over the
    triangle, (B, 1, 3) in the rotated column order."""
    pts, wts = triangle_rule(q_reg if case == 0 else q_sing)
    n6 = shape6(pts)
    wb = wts[None, :] * _bary(pts).T
    out = np.empty((len(rows), 1, 3))
    Y = _interp(n6, nodes[cols[:, None], ORDER6[py]])
    D = vertices[rows][:, None, :] - Y
    r2 = D[..., 0] ** 2 + D[..., 1] ** 2 + D[..., 2] ** 2
    r = np.sqrt(r2)
    if kind == "dlp":
        nyv = _interp(n6, normals[cols[:, None], ORDER6[py]])
        dot = D[..., 0] * nyv[..., 0] + D[..., 1] * nyv[..., 1] + D[..., 2] * nyv[..., 2]
        kg = dot / (FOUR_PI * r2 * r)
    else:
        kg = gram[cols][:, None] / (FOUR_PI * r)
    for c in range(3):
        out[:, 0, c] = np.sum(kg * wb[c][None, :], axis=1)
    return out


def collocation_classify(triangles, rows, cols):
    hit = triangles[cols] == rows[:, None]
    return hit.any(axis=1).astype(np.int64), np.argmax(hit, axis=1)


def block_collocation(nodes, gram, vertices, triangles, rows, cols, q=(3, 5), kind="slp", normals=None):
    """Collocation block (assembly.py:340-362) with the executor's scatter
    (row width 1, column slots permuted by the rotation)."""
    nv = int(triangles.max()) + 1
    tc = triangle_table(cols, triangles, nv)
    rows = np.asarray(rows)
    nr, nt_ = len(rows), len(tc)
    R, C = np.repeat(rows, nt_), np.tile(tc[:, 0], nr)
    rs = np.repeat(np.arange(nr), nt_)
    cs = np.tile(tc[:, 1:] - 1, (nr, 1))
    case, py = collocation_classify(triangles, R, C)
    cs = np.take_along_axis(cs, PERMS3[py], axis=1)
    vals = np.empty((len(R), 1, 3))
    for k in (0, 1):
        m = case == k
        if m.any():
            vals[m] = collocation_values(nodes, gram, vertices, k, R[m], C[m], py[m], *q, kind=kind,
                                         normals=normals)
    mat = np.zeros((nr, len(cols)))
    for b in range(3):
        ok = cs[:, b] >= 0
        np.add.at(mat, (rs[ok], cs[ok, b]), vals[ok, 0, b])
    return mat


def block(nodes, gram, triangles, rows, cols, q=(3, 5), kind="slp", normals=None):
    """Dense block G[rows, cols] (assembly.py:330-337)."""
    rows = np.asarray(rows)
    cols = np.asarray(cols)
    R, C = np.repeat(rows, len(cols)), np.tile(cols, len(rows))
    case, px, py = classify(triangles[R], triangles[C])
    vals = np.empty(len(R))
    for k in range(4):
        m = case == k
        if m.any():
            vals[m] = pair_values(nodes, gram, k, R[m], C[m], px[m], py[m], *q, kind=kind, normals=normals)
    return vals.reshape(len(rows), len(cols))


# ---------------------------------------------------------------- Green factors
# quadrature.py:95-126, assembly.py:371-455

def box_rule(lower, upper, delta, m):
    lo, hi = np.asarray(lower) - delta, np.asarray(upper) + delta
    g, w = gauss01(m)
    Z, W, N = [], [], []
    for ax in range(3):
        b, c = [a for a in range(3) if a != ax]
        gb, gc = np.meshgrid(lo[b] + (hi[b] - lo[b]) * g, lo[c] + (hi[c] - lo[c]) * g,
                             indexing="ij")
        fw = np.outer(w, w).ravel() * (hi[b] - lo[b]) * (hi[c] - lo[c])
        for sgn, lev in ((-1.0, lo[ax]), (1.0, hi[ax])):
            z = np.empty((m * m, 3))
            z[:, ax], z[:, b], z[:, c] = lev, gb.ravel(), gc.ravel()
            nrm = np.zeros((m * m, 3))
            nrm[:, ax] = sgn
            Z.append(z)
            W.append(fw)
            N.append(nrm)
    return np.concatenate(Z), np.concatenate(W), np.concatenate(N)


def green_factor(nodes, gram, rows, lower, upper, diam, side, m=3, delta_factor=0.5, q=3):
    """Row factor A = [sqrt w g, -d sqrt w h] or column factor
    B = [sqrt w h, sqrt w / d g] of the dof list ``rows`` under the box
    rule of (lower, upper) enlarged by delta_factor*diam; d = diam."""
    z, wz, nz = box_rule(lower, upper, delta_factor * diam, m)
    pts, wts = triangle_rule(q)
    xq = np.einsum("ma,tac->tmc", shape6(pts), nodes[rows])
    gw = np.repeat(gram[rows][:, None], len(wts), axis=1) * wts[None, :]
    d = xq[:, :, None, :] - z[None, None, :, :]
    r = np.sqrt(d[..., 0] ** 2 + d[..., 1] ** 2 + d[..., 2] ** 2)
    if r.size and r.min() <= 1e-12:
        raise ValueError("expansion point touches the surface")
    g = 1.0 / (FOUR_PI * r)
    h = np.einsum("tmkc,kc->tmk", d, nz) / (FOUR_PI * r ** 3)
    ig, ih = np.einsum("tm,tmk->tk", gw, g), np.einsum("tm,tmk->tk", gw, h)
    sq = np.sqrt(wz)
    k = len(z)
    out = np.empty((len(rows), 2 * k))
    if side == "row":
        out[:, :k], out[:, k:] = sq[None, :] * ig, -diam * sq[None, :] * ih
    else:
        out[:, :k], out[:, k:] = sq[None, :] * ih, sq[None, :] / diam * ig
    return out


# ---------------------------------------------------------------- ACA
# gca.py:41-79

def aca(a, eps, max_rank=None):
    a = np.array(a, dtype=np.float64)
    n, w = a.shape
    limit = min(n, w if max_rank is None else int(max_rank))
    nrm = np.linalg.norm(a)
    piv, cols = [], []
    while len(piv) < limit and np.linalg.norm(a) > eps * nrm:
        i, j = np.unravel_index(np.argmax(np.abs(a)), a.shape)
        p = a[i, j]
        if p == 0.0:
            break
        u = a[:, j] / p
        a -= np.outer(u, a[i, :])
        piv.append(int(i))
        cols.append(u)
    piv = np.asarray(piv, dtype=np.intp)
    if not len(piv):
        return piv, np.zeros((n, 0))
    U = np.stack(cols, axis=1)
    v = np.linalg.solve(U[piv].T, U.T).T
    v[piv] = np.eye(len(piv))
    return piv, v


# ---------------------------------------------------------------- trees
# clustering.py:15-237 (recursive restatement)

class Tree:
    """Flat record of the recursive median-split cluster tree."""

    def __init__(self, vertices, triangles, leaf=16):
        nodes, _ = chart_nodes(vertices, triangles)
        ctrl = nodes.copy()
        for s_, (i, j) in zip((3, 4, 5), ((0, 1), (1, 2), (2, 0))):
            ctrl[:, s_] = 0.5 * (4.0 * nodes[:, s_] - nodes[:, i] - nodes[:, j])
        lo, hi = ctrl.min(axis=1), ctrl.max(axis=1)
        pts = vertices[triangles].mean(axis=1)
        self.perm = np.arange(len(triangles))
        self.start, self.stop, self.lower, self.upper, self.kids = [], [], [], [], []

        def rec(a, b):
            idx = self.perm[a:b]
            me = len(self.start)
            self.start.append(a)
            self.stop.append(b)
            self.lower.append(lo[idx].min(axis=0))
            self.upper.append(hi[idx].max(axis=0))
            self.kids.append(())
            if b - a <= leaf:
                return me
            ax = int(np.argmax(self.upper[me] - self.lower[me]))
            self.perm[a:b] = idx[np.argsort(pts[idx, ax], kind="stable")]
            mid = a + (b - a) // 2
            self.kids[me] = (rec(a, mid), rec(mid, b))
            return me

        rec(0, len(triangles))
        self.lower, self.upper = np.array(self.lower), np.array(self.upper)
        self.diam = np.array([float(np.linalg.norm(u - l)) for l, u in zip(self.lower, self.upper)])

    def dofs(self, i):
        return self.perm[self.start[i]:self.stop[i]]


def block_leaves(t, eta=1.0):
    """clustering.py:215-237: leaves (row, col, admissible) in DFS order."""
    out = []

    def dist(i, j):
        gap = np.maximum(0.0, np.maximum(t.lower[i] - t.upper[j], t.lower[j] - t.upper[i]))
        return float(np.linalg.norm(gap))

    def rec(i, j):
        if max(t.diam[i], t.diam[j]) <= 2.0 * eta * dist(i, j):
            out.append((i, j, True))
            return
        ri, cj = t.kids[i] or (i,), t.kids[j] or (j,)
        if ri == (i,) and cj == (j,):
            out.append((i, j, False))
            return
        for a in ri:
            for b in cj:
                rec(a, b)

    rec(0, 0)
    return out


# ---------------------------------------------------------------- GCA-H2
# gca.py:162-220 (bases), 282-312 (build), h2.py:19-80 (matvec)

class H2:
    """Reference-algorithm GCA-H2 on the host: bases, blocks, matvec."""

    def __init__(self, vertices, triangles, eps, m=3, leaf=16, eta=1.0, q=(3, 5),
                 tree=None, leaves=None, assemble=True):
        self.t = tree or Tree(vertices, triangles, leaf)
        self.nodes, self.gram = chart_nodes(vertices, triangles)
        self.tris = triangles
        self.leaves = leaves if leaves is not None else block_leaves(self.t, eta)
        adm = {(i, j) for i, j, a in self.leaves if a}
        self.bases = {}
        for side, marks in (("row", {i for i, _ in adm}), ("col", {j for _, j in adm})):
            self.bases[side] = self._basis(side, marks, eps, m, q[0])
        self.blocks = {}
        if assemble:
            for i, j, a in self.leaves:
                r = self.bases["row"][i]["piv"] if a else self.t.dofs(i)
                c = self.bases["col"][j]["piv"] if a else self.t.dofs(j)
                self.blocks[(i, j)] = block(self.nodes, self.gram, self.tris, r, c, q)

    def _basis(self, side, marks, eps, m, q):
        t, out = self.t, {}

        def build(i):
            if not t.kids[i]:
                rows = t.dofs(i)
            else:
                for c in t.kids[i]:
                    build(c)
                rows = np.concatenate([out[c]["piv"] for c in t.kids[i]])
            A = green_factor(self.nodes, self.gram, rows, t.lower[i], t.upper[i], t.diam[i],
                             side, m, 0.5, q)
            piv, v = aca(A, eps)
            out[i] = {"piv": rows[piv], "v": v}
            if t.kids[i]:
                o = 0
                for c in t.kids[i]:
                    r = len(out[c]["piv"])
                    out[c]["E"] = v[o:o + r]
                    o += r

        def walk(i):
            if i in marks:
                build(i)
                out.setdefault("_roots", []).append(i)
                return
            for c in t.kids[i]:
                walk(c)

        walk(0)
        return out

    def mvm(self, x):
        t = self.t
        xt = np.asarray(x, dtype=np.float64)[t.perm]
        cb, rb = self.bases["col"], self.bases["row"]
        xh = {}

        def fwd(i):
            if not t.kids[i]:
                xh[i] = cb[i]["v"].T @ xt[t.start[i]:t.stop[i]]
                return
            acc = np.zeros(len(cb[i]["piv"]))
            for c in t.kids[i]:
                fwd(c)
                acc += cb[c]["E"].T @ xh[c]
            xh[i] = acc

        for r in cb.get("_roots", []):
            fwd(r)
        yh = {i: np.zeros(len(b["piv"])) for i, b in rb.items() if i != "_roots"}
        for i, j, a in self.leaves:
            if a:
                yh[i] += self.blocks[(i, j)] @ xh[j]
        yt = np.zeros(len(xt))

        def bwd(i):
            if not t.kids[i]:
                yt[t.start[i]:t.stop[i]] += rb[i]["v"] @ yh[i]
                return
            for c in t.kids[i]:
                yh[c] += rb[c]["E"] @ yh[i]
                bwd(c)

        for r in rb.get("_roots", []):
            bwd(r)
        for i, j, a in self.leaves:
            if not a:
                yt[t.start[i]:t.stop[i]] += self.blocks[(i, j)] @ xt[t.start[j]:t.stop[j]]
        y = np.empty(len(yt))
        y[t.perm] = yt
        return y


def reference_baseline(args, steps, cpu_sample):
    """bench.py cpu_baseline fallback when baseline/_ref is absent: the
    oracle port timed on the host cores (kind "port")."""
    import os
    import time
    from paper_1810_08429_b200 import geometry  # mesh input generation only
    mesh = geometry.build_sphere_mesh(args.level)
    t0 = time.perf_counter()
    h = H2(mesh.vertices, mesh.triangles, args.eps, assemble=False)
    t1 = time.perf_counter()
    rng = np.random.default_rng(0)
    pick = [lf for lf in h.leaves if rng.random() < cpu_sample]
    tasks_all = sum(len(h.bases["row"][i]["piv"]) * len(h.bases["col"][j]["piv"]) if a
                    else (h.t.stop[i] - h.t.start[i]) * (h.t.stop[j] - h.t.start[j])
                    for i, j, a in h.leaves)
    tasks_s = 0
    t2 = time.perf_counter()
    for i, j, a in pick:
        r = h.bases["row"][i]["piv"] if a else h.t.dofs(i)
        c = h.bases["col"][j]["piv"] if a else h.t.dofs(j)
        block(h.nodes, h.gram, h.tris, r, c)
        tasks_s += len(r) * len(c)
    t3 = time.perf_counter()
    quad = (t3 - t2) * tasks_all / max(tasks_s, 1)
    return {"kind": "port", "cores": 1, "matvec_gbs": float("nan"), "matvec_s": float("nan"),
            "bytes": 0, "assembly_s_extrapolated": (t1 - t0) + quad, "trees_s": 0.0,
            "bases_s": t1 - t0, "quadrature_sampled_s": t3 - t2,
            "quadrature_sample_tasks": tasks_s, "quadrature_tasks": tasks_all,
            "sample": "oracle port: bases full, quadrature on %.1f%% of blocks extrapolated; "
                      "matvec not timed" % (100 * cpu_sample)}
