"""Device-resident geometry, rule tables and singular-task queues.

PyTorch is used only for allocation, streams and host<->device copies; all
arithmetic happens in ``libgcb200.so``.  Uploads are cached on the mesh
object (meshes are immutable), so one mesh is uploaded once
per device and quadrature order.
"""

import ctypes

import numpy as np

from . import _native
from .errors import ConfigError, DeviceError
from .geometry import chart_pack, shape_functions
from .quadrature import reduced_sauter_rule, triangle_gauss

try:  # torch is plumbing only; importing the package must not need a GPU
    import torch
except ImportError:  # pragma: no cover
    torch = None


def require_device(device=None):
    """torch.device for the hot path; raises DeviceError without CUDA."""
    if torch is None or not torch.cuda.is_available():
        raise DeviceError("the GCA-H2 hot path needs a CUDA device (B200); "
                          "there is no CPU fallback")
    _native.load()
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def stream_handle():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None and t.numel() else ctypes.c_void_p(0)


# uploads from this size on are staged in pinned memory: a pageable upload
# is staged by the driver, whose staging buffers drain only as the stream
# reaches the copies - behind queued quadrature, a plan's uploads then wait
# for it (C4 assembly 0.42 -> 0.35 s when the threshold fell from 1 MB)
_PINNED_UPLOAD_BYTES = 4096


def to_dev(a, device, dtype=None):
    a = np.ascontiguousarray(a)
    if not a.flags.writeable:          # read-only views (broadcasts): copy
        a = a.copy()
    t = torch.from_numpy(a)
    if dtype is not None:
        t = t.to(dtype)
    if t.numel() * t.element_size() >= _PINNED_UPLOAD_BYTES:
        # staged in pinned memory (torch's caching host allocator, which
        # keeps the block until the copy ran) the copy is queued without
        # waiting for the work ahead of it on the stream
        p = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        p.copy_(t)
        return p.to(device, non_blocking=True)
    # tiny uploads: staged by the driver before the call returns
    return t.to(device, non_blocking=True)


def zeros(shape, device, dtype=None):
    return torch.zeros(shape, dtype=dtype or torch.float64, device=device)


def empty(shape, device, dtype=None):
    return torch.empty(shape, dtype=dtype or torch.float64, device=device)


TAIL_PAD = 4   # doubles readable past the end of a panel buffer (16-byte bulk copies)


def padded_empty(n, device):
    """float64 vector of n entries whose storage extends TAIL_PAD zeros past
    the end (matrix storage streamed by widened cp.async.bulk copies)."""
    t = torch.empty(n + TAIL_PAD, dtype=torch.float64, device=device)
    t[n:].zero_()
    return t[:n]


def padded_copy(src):
    out = padded_empty(src.numel(), src.device)
    out.copy_(src)
    return out


def device_charts(mesh, device):
    """Plane chart data of a TriangleMesh computed on the device
    (``gc_chart_pack``), bit-identical to the host ``chart_pack`` /
    ``control_points`` / centroids: dict of device tensors ``verts``,
    ``tris`` (int64), ``corners`` (nt,3,3), ``gram``, ``normal`` (nt,3) and
    ``support`` (nt,9) = control-point box lower | upper | centroid.  Cached
    on the mesh per device; None for other mesh types (host path)."""
    from .geometry import TriangleMesh, _shape_gradients_at_nodes
    if type(mesh) is not TriangleMesh:
        return None
    cache = mesh.__dict__.setdefault("_device_cache", {})
    key = ("charts", str(device))
    if key not in cache:
        g = _shape_gradients_at_nodes()
        gu = np.ascontiguousarray(g[0, :, 0], dtype=np.float64)
        gv = np.ascontiguousarray(g[0, :, 1], dtype=np.float64)
        nt = mesh.nt
        out = dict(verts=to_dev(np.ascontiguousarray(mesh.vertices, dtype=np.float64), device),
                   tris=to_dev(mesh.triangles.astype(np.int64), device),
                   corners=empty((nt, 3, 3), device), gram=empty(nt, device), normal=empty((nt, 3), device),
                   support=empty((nt, 9), device))
        with torch.cuda.device(device):
            _native.call("gc_chart_pack", ptr(out["verts"]), ptr(out["tris"]), nt, gu.ctypes.data,
                         gv.ctypes.data, ptr(out["corners"]), ptr(out["gram"]), ptr(out["normal"]),
                         ptr(out["support"]), stream_handle())
        cache[key] = out
    return cache[key]


class DeviceMesh:
    """Chart data of one plane mesh on one device, for one regular order.

    ``corners (nt,3,3)``, ``gram (nt,)``, ``tri_vid (nt,3)`` (plane meshes:
    ``device_charts``, bit-identical to the host chart pack; quadratic
    charts: uploaded from the host), and the regular-rule surface points
    ``xq (nt,q^2,3)`` computed on the device in the reference's operation
    order.
    """

    def __init__(self, mesh, q_reg, device):
        self.mesh = mesh
        self.device = device
        self.nt = mesh.nt
        self.q_reg = q_reg
        pts, wts = triangle_gauss(q_reg)
        charts = device_charts(mesh, device)
        if charts is not None:           # plane mesh: chart data built on the device
            pack = None
            self.curved = False
            self.corners, self.gram, self.tri_vid = charts["corners"], charts["gram"], charts["tris"]
        else:
            pack = chart_pack(mesh)
            self.curved = bool(pack.curved)
            self.corners = to_dev(pack.nodes[:, :3], device)
            self.gram = to_dev(pack.gram if not self.curved else np.zeros(self.nt), device)
            self.tri_vid = to_dev(mesh.triangles.astype(np.int64), device)
        self.wq = to_dev(wts, device)
        self.mq = len(wts)
        n6h = shape_functions(pts)
        if self.curved:
            # quadratic charts: points, point Gramians and normals on the host
            # with the reference's einsum/norm (assembly.py:371-381)
            self.xq = to_dev(np.einsum("ma,tac->tmc", n6h, pack.nodes), device)
            nrm = np.einsum("ma,tac->tmc", n6h, pack.normals)
            self.gq = to_dev(np.sqrt(nrm[..., 0] ** 2 + nrm[..., 1] ** 2 + nrm[..., 2] ** 2), device)
            self.nq = to_dev(nrm, device)
            self.nodes6 = to_dev(pack.nodes, device)
            self.nrm6 = to_dev(pack.normals, device)
        else:
            n6 = to_dev(n6h, device)
            self.xq = empty((self.nt, self.mq, 3), device)
            with torch.cuda.device(device):
                _native.call("gc_surface_points", ptr(self.corners), self.nt, ptr(n6), self.mq,
                             ptr(self.xq), stream_handle())
            self.gq = self.nq = self.nodes6 = self.nrm6 = None
        self.wq_host = np.ascontiguousarray(wts, dtype=np.float64)
        # chart normal per triangle (|n| = gram), for the double layer of plane charts
        self.normals = (charts["normal"] if charts is not None
                        else to_dev(np.ascontiguousarray(pack.normals[:, 0]), device))
        # linear basis: the barycentric values of the regular rule's points;
        # vertex stars built on first use (_stars)
        self.vstar_ptr = self.vstar_ent = None
        self.bq = to_dev(np.stack([1.0 - pts[:, 0] - pts[:, 1], pts[:, 0], pts[:, 1]], 1), device)
        self.verts = (charts["verts"] if charts is not None
                      else to_dev(np.ascontiguousarray(mesh.vertices, dtype=np.float64), device))
        self._geoms = {}
        self.geom = self.geom_of("slp")
        self.geom_dlp = self.geom_of("dlp")

    def geom_of(self, kind, basis="constant"):
        """The gc_geom of the single-layer ("slp") or double-layer ("dlp")
        kernel, for the constant or the linear basis."""
        if kind not in ("slp", "dlp"):
            raise ConfigError("unknown kernel kind %r" % (kind,))
        codes = {"constant": 0, "linear": 1, "collocation": 2}
        if basis not in codes:
            raise ConfigError("unknown basis %r" % (basis,))
        key = (kind, basis)
        if key not in self._geoms:
            if basis != "constant":
                self._stars()
            self._geoms[key] = _native.GcGeom(
                ptr(self.corners), ptr(self.gram), ptr(self.tri_vid), ptr(self.xq), ptr(self.wq),
                self.nt, self.mq, self.wq_host.ctypes.data, ptr(self.normals), int(kind == "dlp"),
                ptr(self.vstar_ptr), ptr(self.vstar_ent), ptr(self.bq), codes[basis], ptr(self.verts),
                ptr(self.nodes6), ptr(self.nrm6), ptr(self.gq), ptr(self.nq))
        return self._geoms[key]

    def _stars(self):
        """Vertex stars of the linear basis, ordered by (vertex, corner,
        triangle)."""
        if self.vstar_ptr is None:
            tris = self.mesh.triangles
            t_of = np.repeat(np.arange(self.nt, dtype=np.int64), 3)
            corner = np.tile(np.arange(3, dtype=np.int64), self.nt)
            vert = tris.ravel().astype(np.int64)
            order = np.lexsort((t_of, corner, vert))
            self.vstar_ptr = to_dev(np.searchsorted(vert[order], np.arange(self.mesh.nv + 1)).astype(np.int64),
                                    self.device)
            self.vstar_ent = to_dev((t_of[order] << 2) | corner[order], self.device)

    @classmethod
    def get(cls, mesh, q_reg, device):
        cache = mesh.__dict__.setdefault("_device_cache", {})
        key = ("mesh", str(device), int(q_reg))
        if key not in cache:
            cache[key] = cls(mesh, int(q_reg), device)
        return cache[key]


class DeviceRules:
    """Sauter-Schwab vertex / edge / identical rules of order ``q_sing`` in
    the xi-reduced coefficient form (quadrature.reduced_sauter_rule): SoA
    (NC coefficient columns, then weights) per case."""

    def __init__(self, q_sing, device, kind="slp"):
        self.q_sing = q_sing
        self.kind = kind
        self.tables = [None] * 4
        self.npts = [0] * 4
        self.struct = _native.GcRules()
        for case in (1, 2, 3):
            rule = reduced_sauter_rule(case, q_sing, 2 if kind == "slp" else 1)
            t = to_dev(np.concatenate([rule.coef.T.ravel(), rule.w]), device)
            self.tables[case] = t
            self.npts[case] = len(rule.w)
            self.struct.table[case] = t.data_ptr()
            self.struct.npts[case] = len(rule.w)

    @classmethod
    def get(cls, q_sing, device, kind="slp"):
        if kind not in ("slp", "dlp"):
            raise ConfigError("unknown kernel kind %r" % (kind,))
        key = (str(device), int(q_sing), kind)
        if key not in _RULE_CACHE:
            _RULE_CACHE[key] = cls(int(q_sing), device, kind)
        return _RULE_CACHE[key]


_RULE_CACHE = {}


def singular_capacity(mesh):
    """Number of ordered triangle pairs per singular case over the whole
    mesh: identical nt, edge 2 ne, vertex sum_v deg(v)^2 - 3 nt - 4 ne
    (pairs sharing v counted once per shared vertex)."""
    deg = np.bincount(mesh.triangles.ravel(), minlength=mesh.nv).astype(np.int64)
    ident, edge = mesh.nt, 2 * mesh.ne
    vert = int((deg * deg).sum()) - 3 * ident - 2 * edge
    return [0, max(vert, 0), edge, ident]


class SingularQueue:
    """Device task queues for the singular cases of one mesh."""

    def __init__(self, mesh, device):
        caps = singular_capacity(mesh)
        self.count = torch.zeros(4, dtype=torch.int32, device=device)
        self.flags = torch.zeros(1, dtype=torch.int32, device=device)
        self.tasks = [torch.empty((max(c, 1), 4), dtype=torch.int64, device=device)
                      for c in caps]
        self.struct = _native.GcQueue()
        for k in range(4):
            self.struct.tasks[k] = self.tasks[k].data_ptr()
            self.struct.cap[k] = caps[k]
        self.struct.count = self.count.data_ptr()

    @classmethod
    def get(cls, mesh, device):
        cache = mesh.__dict__.setdefault("_device_cache", {})
        key = ("queue", str(device))
        if key not in cache:
            cache[key] = cls(mesh, device)
        return cache[key]

    def check_flags(self):
        f = int(self.flags.item())
        if f & 2:
            raise DeviceError("singular task queue overflow")
        if f:
            self.flags.zero_()


def check_mesh(mesh, kind="slp", basis="constant", linear_ok=False):
    """Validate (kernel, basis, geometry) for a device path; ``linear_ok``
    marks the paths that implement the linear basis."""
    if basis in ("linear", "collocation") and not linear_ok:
        raise ConfigError("this path supports the constant basis only")
    if kind not in ("slp", "dlp"):
        raise ConfigError("unknown kernel kind %r" % (kind,))
    if basis not in ("constant", "linear", "collocation"):
        raise ConfigError("unknown basis %r" % (basis,))

