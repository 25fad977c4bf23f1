"""Quadrature rule tables and triangle-pair classification.

Host-side generators for every table the device kernels read.  They restate
``greencross/quadrature.py``: Gauss-Legendre (``:49-61``), the collapsed
triangle rule (``:64-76``), the Green box-boundary rule (``:95-126``), the
Sauter-Schwab relative-coordinate rules (``:191-284``) and the shared-vertex
classification with its alignment permutations (``:26-46, 129-179``).  The
tables are generated once per order, cached, and uploaded to HBM by
``assembly.DeviceRules``; the classification runs on the device inside the
near-field kernel (``csrc/quadrature.cu``) and here only for the evaluator
seam and the tests.
"""

from collections import namedtuple
from functools import lru_cache

import numpy as np

Rule1D = namedtuple("Rule1D", "points weights")
GreenRule = namedtuple("GreenRule", "points weights normals k")
PairRule = namedtuple("PairRule", "x y w")
SingularityCase = namedtuple("SingularityCase", "kind row_perm col_perm")

DISJOINT, VERTEX, EDGE, IDENTICAL = 0, 1, 2, 3
KIND_NAMES = ("disjoint", "vertex", "edge", "identical")
KIND_CODES = {name: code for code, name in enumerate(KIND_NAMES)}

# Vertex permutations of the reference triangle: the three rotations, then
# the three odd permutations (quadrature.py:26-31).  A permutation id is an
# index into this table; the device uses the same numbering.
PERMS3 = np.array([[0, 1, 2], [1, 2, 0], [2, 0, 1],
                   [0, 2, 1], [2, 1, 0], [1, 0, 2]], dtype=np.int64)
INV_PERMS3 = np.argsort(PERMS3, axis=1)


def _midpoint_slot(i, j):
    return {frozenset((0, 1)): 3, frozenset((1, 2)): 4,
            frozenset((2, 0)): 5}[frozenset((i, j))]


# chart-node order induced by each vertex permutation (quadrature.py:35-46)
ORDER6 = np.array([[p[0], p[1], p[2], _midpoint_slot(p[0], p[1]),
                    _midpoint_slot(p[1], p[2]), _midpoint_slot(p[2], p[0])]
                   for p in PERMS3.tolist()], dtype=np.int64)

# PERM_ID[a, b, c] = id of the permutation (a, b, c)
PERM_ID = np.zeros((3, 3, 3), dtype=np.int64)
for _pid, (_a, _b, _c) in enumerate(PERMS3.tolist()):
    PERM_ID[_a, _b, _c] = _pid


@lru_cache(maxsize=None)
def gauss_legendre(m):
    if not 1 <= m <= 32:
        raise ValueError("Gauss order %r outside [1, 32]" % (m,))
    return Rule1D(*np.polynomial.legendre.leggauss(m))


@lru_cache(maxsize=None)
def _gauss01(m):
    pts, wts = gauss_legendre(m)
    return 0.5 * (pts + 1.0), 0.5 * wts


@lru_cache(maxsize=None)
def triangle_gauss(q):
    """q*q collapsed tensor rule on the reference triangle:
    (s, t) -> (s(1-t), st) with weight w_s w_t s."""
    s, ws = _gauss01(q)
    t, wt = _gauss01(q)
    S, T = np.meshgrid(s, t, indexing="ij")
    pts = np.column_stack([(S * (1.0 - T)).ravel(), (S * T).ravel()])
    return pts, (np.outer(ws, wt) * S).ravel()


def green_box_rule(box, delta, m):
    """Tensor Gauss rule on the boundary of ``box`` enlarged by ``delta``:
    6 faces x m^2 points, outward axis normals, weights summing to the
    enlarged surface area.  Face order: axis 0,1,2, low side then high side."""
    if delta <= 0.0:
        raise ValueError("delta must be positive")
    lower, upper = (box.lower, box.upper) if hasattr(box, "lower") else box
    lo = np.asarray(lower, dtype=np.float64) - delta
    hi = np.asarray(upper, dtype=np.float64) + delta
    g, w = _gauss01(m)
    ww = np.outer(w, w).ravel()
    pts, wts, nrm = [], [], []
    for axis in range(3):
        b, c = (axis + 1) % 3, (axis + 2) % 3
        if b > c:
            b, c = c, b
        span_b, span_c = hi[b] - lo[b], hi[c] - lo[c]
        gb, gc = np.meshgrid(lo[b] + span_b * g, lo[c] + span_c * g, indexing="ij")
        for sign, level in ((-1.0, lo[axis]), (1.0, hi[axis])):
            z = np.zeros((m * m, 3))
            z[:, axis] = level
            z[:, b] = gb.ravel()
            z[:, c] = gc.ravel()
            n = np.zeros((m * m, 3))
            n[:, axis] = sign
            pts.append(z)
            wts.append(ww * span_b * span_c)
            nrm.append(n)
    pts = np.concatenate(pts)
    return GreenRule(pts, np.concatenate(wts), np.concatenate(nrm), len(pts))


# --------------------------------------------------------------------------
# classification (host twin of the device classifier in csrc/quadrature.cu)

def classify_pairs(row_tris, col_tris):
    """Case and alignment permutations of triangle pairs given as (B,3)
    vertex-id arrays.  Shared vertices move to the leading slots, in the
    same order on both sides (quadrature.py:129-171)."""
    rt = np.asarray(row_tris)
    ct = np.asarray(col_tris)
    hit = rt[:, :, None] == ct[:, None, :]
    rhit, chit = hit.any(2), hit.any(1)
    kind = rhit.sum(1).astype(np.int64)       # 0..3 shared = case code
    rperm = np.zeros(len(rt), dtype=np.int64)
    cperm = np.zeros(len(rt), dtype=np.int64)
    v = kind == VERTEX
    rperm[v] = rhit[v].argmax(1)              # rotation k puts vertex k first
    cperm[v] = chit[v].argmax(1)
    e = np.flatnonzero(kind == EDGE)
    if e.size:
        missing = (~rhit[e]).argmax(1)        # the row vertex not shared
        rot = (missing + 1) % 3               # rotation putting the shared
        rperm[e] = rot                        # edge into slots 0, 1
        g0 = rt[e, PERMS3[rot, 0]]
        g1 = rt[e, PERMS3[rot, 1]]
        c0 = (ct[e] == g0[:, None]).argmax(1)
        c1 = (ct[e] == g1[:, None]).argmax(1)
        cperm[e] = PERM_ID[c0, c1, 3 - c0 - c1]
    return kind, rperm, cperm


def classify_pair(t, s):
    k, rp, cp = classify_pairs(np.asarray(t).reshape(1, 3), np.asarray(s).reshape(1, 3))
    return SingularityCase(KIND_NAMES[k[0]], tuple(PERMS3[rp[0]].tolist()),
                           tuple(PERMS3[cp[0]].tolist()))


# --------------------------------------------------------------------------
# Sauter-Schwab rules in relative coordinates 0 <= r2 <= r1 <= 1; a point
# (r1, r2) maps to simplex coordinates (r1 - r2, r2).

def _hypercube(q):
    g, w = _gauss01(q)
    grid = np.meshgrid(g, g, g, g, indexing="ij")
    return [a.ravel() for a in grid], np.einsum("i,j,k,l->ijkl", w, w, w, w).ravel()


def _identical_parts(xi, e1, e2, e3):
    jac = xi ** 3 * e1 ** 2 * e2
    w = (xi, xi * e1, xi * e1 * e2, xi * e1 * e2 * e3)
    # three coordinate maps z = M w (rows as signed index lists), each giving
    # a mirrored pair of subdomains
    maps = ((((1, 0),), ((1, 0), (-1, 1), (1, 2)), ((1, 3),), ((1, 2),)),
            (((1, 0),), ((1, 1), (-1, 2), (1, 3)), ((1, 2),), ((1, 3),)),
            (((1, 0), (-1, 3)), ((1, 1), (-1, 3)), ((-1, 3),), ((1, 2), (-1, 3))))
    parts = []
    for m in maps:
        z = []
        for row in m:
            acc = 0
            for sign, idx in row:
                acc = acc + (w[idx] if sign > 0 else -w[idx])
            z.append(acc)
        parts.append((z[0], z[1], z[0] - z[2], z[1] - z[3], jac))
        parts.append((z[0] - z[2], z[1] - z[3], z[0], z[1], jac))
    return parts


def _vertex_parts(xi, e1, e2, e3):
    jac = xi ** 3 * e2
    return [(xi, xi * e1, xi * e2, xi * e2 * e3, jac),
            (xi * e2, xi * e2 * e3, xi, xi * e1, jac)]


def _edge_parts(xi, e1, e2, e3):
    ja = xi ** 3 * e1 ** 2
    jb = xi ** 3 * e1 ** 2 * e2
    quads = (
        ((xi, -xi * e1 * e2, xi * e1 * (1.0 - e2), xi * e1 * e3), ja),
        ((xi, -xi * e1 * e2 * e3, xi * e1 * e2 * (1.0 - e3), xi * e1), jb),
        ((xi * (1.0 - e1 * e2), xi * e1 * e2, xi * e1 * e2 * e3,
          xi * e1 * (1.0 - e2)), jb),
        ((xi * (1.0 - e1 * e2 * e3), xi * e1 * e2 * e3, xi * e1,
          xi * e1 * e2 * (1.0 - e3)), jb),
        ((xi * (1.0 - e1 * e2 * e3), xi * e1 * e2 * e3, xi * e1 * e2,
          xi * e1 * (1.0 - e2 * e3)), jb),
    )
    return [(a, d, a + b, c, j) for (a, b, c, d), j in quads]


@lru_cache(maxsize=None)
def sauter_rule(kind, q):
    """Pair rule on t-hat x t-hat for one case; 6/10/2/1 x q^4 nodes for
    identical/edge/vertex/disjoint, weights summing to 1/4.  The edge rule
    is symmetrised under (x, y) -> (Sy, Sx), S the 0<->1 vertex exchange
    (quadrature.py:272-283)."""
    if q < 1:
        raise ValueError("quadrature order must be positive")
    code = KIND_CODES[kind] if isinstance(kind, str) else int(kind)
    if code == DISJOINT:
        p, w = triangle_gauss(q)
        n = len(p)
        return PairRule(np.repeat(p, n, axis=0), np.tile(p, (n, 1)),
                        np.outer(w, w).ravel())
    (xi, e1, e2, e3), w4 = _hypercube(q)
    builder = {IDENTICAL: _identical_parts, VERTEX: _vertex_parts,
               EDGE: _edge_parts}.get(code)
    if builder is None:
        raise ValueError("unknown singularity kind %r" % (kind,))
    parts = builder(xi, e1, e2, e3)
    x = np.concatenate([np.column_stack([a - b, b]) for a, b, _, _, _ in parts])
    y = np.concatenate([np.column_stack([c - d, d]) for _, _, c, d, _ in parts])
    w = np.concatenate([w4 * j for *_, j in parts])
    if code == EDGE:
        flip = lambda p: np.stack([1.0 - p[:, 0] - p[:, 1], p[:, 1]], axis=1)
        x, y = np.concatenate([x, flip(y)]), np.concatenate([y, flip(x)])
        w = np.concatenate([0.5 * w, 0.5 * w])
    return PairRule(x, y, w)


ReducedRule = namedtuple("ReducedRule", "coef w ncoef")


@lru_cache(maxsize=None)
def reduced_sauter_rule(kind, q, xi_power=2):
    """The Sauter-Schwab rule of ``sauter_rule(kind, q)`` with the xi
    (radial) sum done exactly.

    In every subdomain all four relative coordinates carry the factor xi and
    the Jacobian carries xi^3 (quadrature.py:246-271), so the pair distance
    is xi * rhat(eta) and the 1/(4 pi r) integrand times the Jacobian is
    xi^2 * j(eta) / (4 pi rhat(eta)).  The xi sum therefore factors out as
    S2 = sum_xi w_xi xi^2 (= 1/3 for q >= 2) and the rule keeps q^3 points
    per subdomain (2/10/6 q^3) - the same quadrature sum, 5x fewer kernel
    evaluations at q = 5.  The double-layer integrand <x-y, n_y>/r^3 is
    homogeneous of degree -2, so its xi factor is xi^1: ``xi_power=1``
    gives the same points with S1 = sum_xi w_xi xi.

    Points are returned as coefficients of the aligned chart edge vectors,
    ``D = x - y = sum_k coef[k] * G_k`` with
      vertex:    G = (E1, E2, -F1, -F2)        (4 coefficients)
      edge:      G = (E1, E2, -F2), E1 == F1   (3)
      identical: G = (E1, E2), E == F          (2)
    where E_k = P_k - P_0 and F_k = Q_k - Q_0 after the alignment
    permutations (P_0 = Q_0 is a shared vertex).
    """
    code = KIND_CODES[kind] if isinstance(kind, str) else int(kind)
    if code not in (VERTEX, EDGE, IDENTICAL):
        raise ValueError("reduced rules exist for the singular cases only")
    g, w = _gauss01(q)
    if xi_power not in (1, 2):
        raise ValueError("xi_power must be 1 (double layer) or 2 (single layer)")
    s2 = float(np.sum(w * g * g)) if xi_power == 2 else float(np.sum(w * g))
    e1, e2, e3 = (a.ravel() for a in np.meshgrid(g, g, g, indexing="ij"))
    w3 = np.einsum("i,j,k->ijk", w, w, w).ravel()
    one = np.ones_like(e1)
    builder = {IDENTICAL: _identical_parts, VERTEX: _vertex_parts, EDGE: _edge_parts}[code]
    parts = builder(one, e1, e2, e3)
    x = np.concatenate([np.column_stack([a - b, b]) for a, b, _, _, _ in parts])
    y = np.concatenate([np.column_stack([c - d, d]) for _, _, c, d, _ in parts])
    wt = np.concatenate([w3 * j * s2 for *_, j in parts])
    if code == VERTEX:
        coef = np.column_stack([x[:, 0], x[:, 1], y[:, 0], y[:, 1]])
    elif code == IDENTICAL:
        coef = np.column_stack([x[:, 0] - y[:, 0], x[:, 1] - y[:, 1]])
    else:
        # D = x1 E1 + x2 E2 - y1 F1 - y2 F2 with F1 = E1; the mirrored half
        # (x, y) -> (S y, S x) gives (x1+x2-y1-y2) E1 + y2 E2 - x2 F2
        direct = np.column_stack([x[:, 0] - y[:, 0], x[:, 1], y[:, 1]])
        mirror = np.column_stack([x[:, 0] + x[:, 1] - y[:, 0] - y[:, 1], y[:, 1], x[:, 1]])
        coef = np.concatenate([direct, mirror])
        wt = np.concatenate([0.5 * wt, 0.5 * wt])
    return ReducedRule(np.ascontiguousarray(coef), wt, coef.shape[1])
