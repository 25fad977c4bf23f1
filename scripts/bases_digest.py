"""Digest of the nested bases (ranks, pivot offsets, pivots, V bytes) of
one configuration, plus the device time of the ACA launches - run against
two builds of the library (GC_LIB=...) to check a kernel change is
bitwise neutral.  Usage: python scripts/bases_digest.py LEVEL EPS [basis disc]"""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_08429_b200 import _native, cli, geometry  # noqa: E402

L, eps = int(sys.argv[1]), float(sys.argv[2])
kw = dict(basis=sys.argv[3], disc=sys.argv[4]) if len(sys.argv) > 4 else {}
cfg = cli.default_config(eps=eps, **kw)
mesh = geometry.build_sphere_mesh(L)
cli.build_h2_operator(mesh, cfg)
torch.cuda.synchronize()
orig, ev = _native.call, []


def timed(name, *args):
    if name != "gc_aca":
        return orig(name, *args)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    r = orig(name, *args)
    b.record()
    ev.append((a, b))
    return r


_native.call = timed
hm, _, _ = cli.build_h2_operator(geometry.build_sphere_mesh(L), cfg)
torch.cuda.synchronize()
hsh = hashlib.sha256()
for side in ("row_basis", "col_basis"):
    st = getattr(hm, side).store
    for a in (st.rank, st.piv_off, st.pivots_host):
        hsh.update(a.tobytes())
    hsh.update(st.V.cpu().numpy().tobytes())
print("L%d eps %g %s lib %s digest %s aca %.3f ms" % (L, eps, kw or "", os.path.basename(_native.LIB_PATH),
                                                   hsh.hexdigest()[:16], sum(a.elapsed_time(b) for a, b in ev)))
