"""Surface meshes and the per-triangle chart data the device kernels consume.

Host-side mirror of ``greencross/geometry.py`` restricted to what the hot
path needs: plane triangle meshes (``TriangleMesh``, ``geometry.py:21-66``),
the octahedral sphere (``build_sphere_mesh``, ``geometry.py:168-201``), the
chart pack that becomes device-resident geometry (``chart_pack``,
``geometry.py:266-293``), Bernstein control points for support boxes
(``geometry.py:324-338``) and the text mesh format (``geometry.py:355-440``)
used to hand builder-generated meshes (the cube of config C3) to the
reference.  Curved charts are out of scope (SURVEY.md §8 f, rank 2).

Everything that feeds a kernel or a tree decision is computed with the same
floating-point primitives as the reference so trees, boxes and Gramians are
bit-identical on the same host (SURVEY.md §7 hard part 1).
"""

import numpy as np

from .errors import ConfigError, GeometryError, MeshFormatError, SizeLimitError

# The reference caps sphere generation at level 8 (geometry.py:12); the
# C5 sweep needs level 9 (2,097,152 triangles), so the cap is lifted here.
LEVEL_CAP = 9

# reference-triangle chart nodes: 3 vertices, then midpoints of the edges
# (0,1), (1,2), (2,0)  (geometry.py:16-18)
CHART_NODES_REF = np.array(
    [[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [0.5, 0.0], [0.5, 0.5], [0.0, 0.5]])


def _norm3_blas(v):
    """Euclidean norm of one 3-vector through numpy's 1-D norm (BLAS dot).

    The reference normalises sphere vertices and measures boxes with
    ``np.linalg.norm`` on 1-D vectors, whose rounding (an FMA chain inside
    ddot) differs from an elementwise formula; reusing the same primitive
    keeps vertex coordinates and box diameters bit-identical.
    """
    return float(np.linalg.norm(v))


class TriangleMesh:
    """Closed, consistently oriented plane-triangle surface.

    Attributes follow ``geometry.py:21-66``: ``vertices (nv,3) f64``,
    ``triangles (nt,3) i64`` counter-clockwise from outside, derived
    ``edges (ne,2)`` with ``a < b`` and ``tri_edges (nt,3)`` giving the
    edge index of (v0,v1), (v1,v2), (v2,v0).
    """

    def __init__(self, vertices, triangles):
        self.vertices = np.ascontiguousarray(vertices, dtype=np.float64)
        self.triangles = np.ascontiguousarray(triangles, dtype=np.int64)
        if self.vertices.ndim != 2 or self.vertices.shape[1] != 3:
            raise MeshFormatError("vertices must be an (nv, 3) array")
        if self.triangles.ndim != 2 or self.triangles.shape[1] != 3:
            raise MeshFormatError("triangles must be an (nt, 3) array")
        nv = len(self.vertices)
        if self.triangles.size and (self.triangles.min() < 0
                                    or self.triangles.max() >= nv):
            raise MeshFormatError("triangle vertex index out of range")
        _reject_degenerate(self.vertices, self.triangles)
        self.edges, self.tri_edges = _edge_topology(self.triangles)
        self._stars = None
        self._pack = None

    nv = property(lambda self: len(self.vertices))
    nt = property(lambda self: len(self.triangles))
    ne = property(lambda self: len(self.edges))

    def vertex_stars(self):
        """Per vertex, the ascending indices of the triangles touching it."""
        if self._stars is None:
            flat = self.triangles.ravel()
            order = np.argsort(flat, kind="stable")
            cuts = np.searchsorted(flat[order], np.arange(self.nv + 1))
            owner = order // 3
            self._stars = [owner[cuts[v]:cuts[v + 1]] for v in range(self.nv)]
        return self._stars

    def centroids(self):
        # same reduction as the reference (mean over the 3 corners: the sum
        # in corner order, then / 3), without the (nt, 3, 3) gather
        V, T = self.vertices, self.triangles
        return (V[T[:, 0]] + V[T[:, 1]] + V[T[:, 2]]) / 3.0

    def __repr__(self):
        return "TriangleMesh(nv=%d, nt=%d)" % (self.nv, self.nt)


def _reject_degenerate(vertices, triangles):
    corners = vertices[triangles]
    e01 = corners[:, 1] - corners[:, 0]
    e02 = corners[:, 2] - corners[:, 0]
    e12 = corners[:, 2] - corners[:, 1]
    twice_area = np.linalg.norm(np.cross(e01, e02), axis=1)
    longest2 = np.maximum.reduce([(e * e).sum(1) for e in (e01, e02, e12)])
    bad = np.flatnonzero(twice_area < 2e-14 * longest2)
    if bad.size:
        raise MeshFormatError("degenerate triangle %d" % int(bad[0]))


def _edge_topology(triangles):
    """Unique undirected edges and the per-triangle edge map; rejects open,
    non-manifold and inconsistently oriented surfaces."""
    nt = len(triangles)
    directed = np.concatenate([triangles[:, [0, 1]], triangles[:, [1, 2]],
                               triangles[:, [2, 0]]])
    undirected = np.sort(directed, axis=1)
    edges, inverse, counts = np.unique(undirected, axis=0, return_inverse=True,
                                       return_counts=True)
    if np.any(counts != 2):
        raise MeshFormatError(
            "mesh is not a closed surface (open or non-manifold edge)")
    width = int(directed.max()) + 1 if directed.size else 1
    code = directed[:, 0] * width + directed[:, 1]
    if np.unique(code).size != code.size:
        raise MeshFormatError("inconsistently oriented triangles share an edge")
    tri_edges = np.ascontiguousarray(inverse.reshape(3, nt).T)
    return edges, tri_edges


# --------------------------------------------------------------------------
# mesh generators

_OCTAHEDRON_V = ((1.0, 0.0, 0.0), (-1.0, 0.0, 0.0), (0.0, 1.0, 0.0),
                 (0.0, -1.0, 0.0), (0.0, 0.0, 1.0), (0.0, 0.0, -1.0))
_OCTAHEDRON_F = ((0, 2, 4), (2, 1, 4), (1, 3, 4), (3, 0, 4),
                 (2, 0, 5), (1, 2, 5), (3, 1, 5), (0, 3, 5))


def _octahedral_refinement(level):
    """Vertices and faces of the level-``level`` midpoint refinement.

    Topology is generated array-at-a-time: per level the 3 edge keys of
    every face are listed in face order, new vertex ids follow the order of
    first appearance (exactly the insertion order of the reference's
    per-face midpoint cache, ``geometry.py:185-200``), and each face splits
    into (a,ab,ca), (ab,b,bc), (ca,bc,c), (ab,bc,ca).
    """
    verts = [np.array(v) for v in _OCTAHEDRON_V]
    faces = np.array(_OCTAHEDRON_F, dtype=np.int64)
    for _ in range(level):
        a, b, c = faces[:, 0], faces[:, 1], faces[:, 2]
        ends = np.stack([np.stack([a, b], 1), np.stack([b, c], 1),
                         np.stack([c, a], 1)], axis=1).reshape(-1, 2)
        key_lo = np.minimum(ends[:, 0], ends[:, 1])
        key_hi = np.maximum(ends[:, 0], ends[:, 1])
        key = key_lo * (len(verts) + 1) + key_hi
        uniq, first, inv = np.unique(key, return_index=True, return_inverse=True)
        # rank unique keys by first appearance -> consecutive new vertex ids
        appearance = np.argsort(first, kind="stable")
        new_id = np.empty(len(uniq), dtype=np.int64)
        new_id[appearance] = len(verts) + np.arange(len(uniq))
        base = len(verts)
        for u in appearance:
            i, j = int(key_lo[first[u]]), int(key_hi[first[u]])
            s = verts[i] + verts[j]
            verts.append(s / _norm3_blas(s))
        assert len(verts) == base + len(uniq)
        mids = new_id[inv].reshape(-1, 3)
        ab, bc, ca = mids[:, 0], mids[:, 1], mids[:, 2]
        faces = np.stack([np.stack([a, ab, ca], 1), np.stack([ab, b, bc], 1),
                          np.stack([ca, bc, c], 1), np.stack([ab, bc, ca], 1)],
                         axis=1).reshape(-1, 3)
    return np.array(verts), faces


def build_sphere_mesh(level):
    """Unit-sphere octahedral mesh with ``8 * 4**level`` triangles
    (``geometry.py:168-201``; vertices bit-identical)."""
    if level < 0 or level > LEVEL_CAP:
        raise SizeLimitError("sphere level %r outside [0, %d]" % (level, LEVEL_CAP))
    verts, faces = _octahedral_refinement(int(level))
    return TriangleMesh(verts, faces)


def build_cube_mesh(level):
    """Cube-surface mesh of config C3 (builder-defined, SURVEY.md §7 part 7).

    Level-``level`` octahedral connectivity with each sphere vertex mapped to
    the cube surface by ``v / max|v_i|``; 131,072 triangles at level 7.  The
    edges and corners of the cube stress the singular quadrature.
    """
    sphere = build_sphere_mesh(level)
    v = sphere.vertices
    return TriangleMesh(v / np.abs(v).max(axis=1, keepdims=True), sphere.triangles)


# --------------------------------------------------------------------------
# charts

def shape_functions(xhat):
    """Quadratic Lagrange basis on the reference triangle, (...,2) -> (...,6)
    (``geometry.py:213-225``)."""
    xhat = np.asarray(xhat, dtype=np.float64)
    x, y = xhat[..., 0], xhat[..., 1]
    l0 = 1.0 - x - y
    return np.stack([l0 * (2.0 * l0 - 1.0), x * (2.0 * x - 1.0),
                     y * (2.0 * y - 1.0), 4.0 * l0 * x, 4.0 * x * y,
                     4.0 * y * l0], axis=-1)


def _shape_gradients_at_nodes():
    """d/dx and d/dy of the 6 shape functions at the 6 chart nodes, (6,6,2)."""
    x, y = CHART_NODES_REF[:, 0], CHART_NODES_REF[:, 1]
    l0 = 1.0 - x - y
    zero = np.zeros_like(x)
    dx = np.stack([1.0 - 4.0 * l0, 4.0 * x - 1.0, zero, 4.0 * (l0 - x),
                   4.0 * y, -4.0 * y], axis=-1)
    dy = np.stack([1.0 - 4.0 * l0, zero, 4.0 * y - 1.0, -4.0 * x,
                   4.0 * x, 4.0 * (l0 - y)], axis=-1)
    return np.stack([dx, dy], axis=-1)


class ChartPack:
    """Per-triangle chart data: ``nodes (nt,6,3)``, ``normals (nt,6,3)``,
    ``gram (nt,)`` (``geometry.py:249-263``).  ``nodes`` and ``gram`` are
    what the device keeps resident; ``gram`` is never recomputed on the
    device because its rounding comes from numpy's norm."""

    __slots__ = ("nodes", "normals", "gram", "curved")

    def __init__(self, nodes, normals, gram, curved=False):
        self.nodes = nodes
        self.normals = normals
        self.gram = gram
        self.curved = curved


class CurvedTriangleMesh:
    """A plane mesh whose edges carry one (curved) midpoint each: quadratic
    charts (``geometry.py:69-114``).  Straight midpoints reproduce the plane
    chart exactly."""

    def __init__(self, base, midpoints):
        midpoints = np.ascontiguousarray(midpoints, dtype=np.float64)
        if midpoints.shape != (base.ne, 3):
            raise MeshFormatError("expected %d midpoints, got %d" % (base.ne, len(midpoints)))
        self.base = base
        self.midpoints = midpoints
        self._pack = None

    vertices = property(lambda self: self.base.vertices)
    triangles = property(lambda self: self.base.triangles)
    edges = property(lambda self: self.base.edges)
    tri_edges = property(lambda self: self.base.tri_edges)
    nv = property(lambda self: self.base.nv)
    nt = property(lambda self: self.base.nt)
    ne = property(lambda self: self.base.ne)

    def vertex_stars(self):
        return self.base.vertex_stars()

    def centroids(self):
        return self.base.centroids()

    def __repr__(self):
        return "CurvedTriangleMesh(nv=%d, nt=%d)" % (self.nv, self.nt)


def to_curved(mesh, project_to_unit_sphere=False):
    """One midpoint per edge (``geometry.py:204-210``): the straight edge
    midpoint, optionally projected onto the unit sphere."""
    v, e = mesh.vertices, mesh.edges
    mid = 0.5 * (v[e[:, 0]] + v[e[:, 1]])
    if project_to_unit_sphere:
        mid = mid / np.linalg.norm(mid, axis=1, keepdims=True)
    return CurvedTriangleMesh(mesh, mid)


def chart_pack(mesh):
    """Build and cache the :class:`ChartPack` of ``mesh``
    (``geometry.py:266-293``): plane charts (constant normal and Gramian)
    or quadratic charts of a :class:`CurvedTriangleMesh` (normals at the six
    nodes, no constant Gramian)."""
    if getattr(mesh, "_pack", None) is not None:
        return mesh._pack
    if isinstance(mesh, CurvedTriangleMesh):
        nodes = np.empty((mesh.nt, 6, 3))
        nodes[:, :3] = mesh.vertices[mesh.triangles]
        nodes[:, 3:] = mesh.midpoints[mesh.tri_edges]
        grads = _shape_gradients_at_nodes()                 # (6 nodes, 6 shapes, 2)
        du = np.einsum("ma,tac->tmc", grads[:, :, 0], nodes)
        dv = np.einsum("ma,tac->tmc", grads[:, :, 1], nodes)
        mesh._pack = ChartPack(np.ascontiguousarray(nodes), np.ascontiguousarray(np.cross(du, dv)),
                               None, True)
        return mesh._pack
    if not isinstance(mesh, TriangleMesh):
        raise ConfigError("unsupported mesh type %r" % (type(mesh).__name__,))
    corners = mesh.vertices[mesh.triangles]
    nodes = np.empty((mesh.nt, 6, 3))
    nodes[:, :3] = corners
    for slot, (i, j) in zip((3, 4, 5), ((0, 1), (1, 2), (2, 0))):
        nodes[:, slot] = 0.5 * (nodes[:, i] + nodes[:, j])
    # plane charts: the normal is constant, so only the partials at node 0
    # are needed (same sequential sum over the 6 nodes as the reference's
    # all-node einsum, bit for bit)
    grads = _shape_gradients_at_nodes()
    du = np.einsum("a,tac->tc", grads[0, :, 0], nodes)
    dv = np.einsum("a,tac->tc", grads[0, :, 1], nodes)
    n0 = np.cross(du, dv)
    gram = np.linalg.norm(n0, axis=1)
    normals = np.broadcast_to(n0[:, None, :], (mesh.nt, 6, 3))
    mesh._pack = ChartPack(np.ascontiguousarray(nodes), normals, gram, False)
    return mesh._pack


def control_points(mesh):
    """Bernstein control points of every chart, (nt,6,3)
    (``geometry.py:324-338``); for plane charts the edge control points
    coincide with the midpoints up to rounding."""
    nodes = chart_pack(mesh).nodes
    ctrl = nodes.copy()
    for slot, (i, j) in zip((3, 4, 5), ((0, 1), (1, 2), (2, 0))):
        ctrl[:, slot] = 0.5 * (4.0 * nodes[:, slot] - nodes[:, i] - nodes[:, j])
    return ctrl


def chart_eval(mesh, triangle, xhat):
    """Point, normal and Gramian of one chart at ``xhat``."""
    xhat = np.asarray(xhat, dtype=np.float64)
    if xhat[0] < -1e-12 or xhat[1] < -1e-12 or xhat.sum() > 1.0 + 1e-12:
        raise GeometryError("point (%g, %g) outside the reference triangle"
                            % (xhat[0], xhat[1]))
    pack = chart_pack(mesh)
    n6 = shape_functions(xhat)
    normal = n6 @ pack.normals[triangle]
    return n6 @ pack.nodes[triangle], normal, float(np.linalg.norm(normal))


def surface_area(mesh, quad_order=4):
    """Integral of the Gramian over all charts (``geometry.py:341-352``)."""
    from .quadrature import triangle_gauss
    pts, w = triangle_gauss(quad_order)
    pack = chart_pack(mesh)
    if not pack.curved:
        return float(w.sum() * pack.gram.sum())
    normals = np.einsum("ma,tac->tmc", shape_functions(pts), pack.normals)
    return float((np.linalg.norm(normals, axis=2) @ w).sum())


def point_gramians(mesh, pts):
    """Per-triangle Gramians at reference points ``pts`` (nt, M): |n| of the
    interpolated chart normal (``assembly.py:371-381`` for curved charts);
    the plane Gramian repeated for plane charts."""
    pack = chart_pack(mesh)
    if not pack.curved:
        return np.repeat(pack.gram[:, None], len(pts), axis=1)
    normals = np.einsum("ma,tac->tmc", shape_functions(pts), pack.normals)
    return np.sqrt(normals[..., 0] ** 2 + normals[..., 1] ** 2 + normals[..., 2] ** 2)


# --------------------------------------------------------------------------
# text format (geometry.py:355-440): header "nv nt ne", 17-digit vertices,
# triangles, edges; round-trips bit-exactly.

def write_mesh(mesh, path):
    with open(path, "w") as fh:
        fh.write("%d %d %d\n" % (mesh.nv, mesh.nt, mesh.ne))
        np.savetxt(fh, mesh.vertices, fmt="%.17g")
        np.savetxt(fh, mesh.triangles, fmt="%d")
        np.savetxt(fh, mesh.edges, fmt="%d")


def read_mesh(path):
    with open(path) as fh:
        lines = [(k + 1, ln.split()) for k, ln in enumerate(fh) if ln.strip()]
    if not lines:
        raise MeshFormatError("empty mesh file", line=1)
    head_line, head = lines[0]
    try:
        if len(head) != 3:
            raise ValueError
        nv, nt, ne = (int(t) for t in head)
    except ValueError:
        raise MeshFormatError("header must be 'nv nt ne'", line=head_line) from None
    if min(nv, nt, ne) < 0:
        raise MeshFormatError("negative count in header", line=head_line)

    cursor = 1

    def section(count, width, conv, what):
        nonlocal cursor
        rows = lines[cursor:cursor + count]
        if len(rows) < count:
            raise MeshFormatError("unexpected end of file in %s section" % what,
                                  line=lines[-1][0])
        out = []
        for lineno, tok in rows:
            if len(tok) != width:
                raise MeshFormatError("expected %d %s fields" % (width, what),
                                      line=lineno)
            try:
                out.append([conv(t) for t in tok])
            except ValueError:
                raise MeshFormatError("bad %s value" % what, line=lineno) from None
        cursor += count
        return out

    verts = section(nv, 3, float, "vertex")
    tris = section(nt, 3, int, "triangle")
    edges = section(ne, 2, int, "edge")
    if cursor < len(lines):
        raise MeshFormatError("curved meshes (midpoint section) are out of scope",
                              line=lines[cursor][0])
    tri_arr = np.array(tris, dtype=np.int64).reshape(nt, 3)
    if tri_arr.size and (tri_arr.min() < 0 or tri_arr.max() >= nv):
        raise MeshFormatError("triangle vertex index out of range",
                              line=lines[1 + nv][0])
    mesh = TriangleMesh(np.array(verts, dtype=np.float64).reshape(nv, 3), tri_arr)
    file_edges = np.array(edges, dtype=np.int64).reshape(ne, 2)
    if mesh.ne != ne or not np.array_equal(
            np.unique(file_edges, axis=0), mesh.edges):
        raise MeshFormatError("edge section does not match triangle edges",
                              line=head_line)
    return mesh
