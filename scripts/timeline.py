"""Timeline of the product DAG inside its CUDA graph: every panel kernel
stamps min(start) / max(end) %globaltimer into a trace slot (median of 10
replays).  Usage: python scripts/timeline.py level eps [key=value ...]
(PanelPlan keyword arguments, e.g. tiers=off)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_08429_b200 import cli, geometry, h2  # noqa: E402

L, eps = int(sys.argv[1]), float(sys.argv[2])
kw = {}
for a in sys.argv[3:]:
    k, v = a.split("=")
    kw[k] = int(v) if v.lstrip("-").isdigit() else v
mesh = (geometry.build_cube_mesh if os.environ.get("GC_GEO") == "cube" else geometry.build_sphere_mesh)(L)
hm, _, _ = cli.build_h2_operator(mesh, cli.default_config(eps=eps))
p = h2.PanelPlan(hm, **kw)
x = torch.randn(mesh.nt, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
slots = {}
for n in p.nodes:
    if n.phase is not None:
        t = torch.zeros(2, dtype=torch.int64, device="cuda")
        p.trace[id(n.phase)] = t
        slots[id(n.phase)] = t
p.capture()
for _ in range(3):
    p.run(x, y)
res = []
for rep in range(10):
    for t in slots.values():
        t[0] = 2 ** 63 - 1
        t[1] = 0
    torch.cuda.synchronize()
    p.run(x, y)
    torch.cuda.synchronize()
    res.append({k: v.cpu().numpy().copy() for k, v in slots.items()})
rows = []
for i, n in enumerate(p.nodes):
    if n.phase is None:
        continue
    st = [r[id(n.phase)][0] - min(v[0] for v in r.values()) for r in res]
    en = [r[id(n.phase)][1] - min(v[0] for v in r.values()) for r in res]
    rows.append((np.median(st) / 1e3, np.median(en) / 1e3, i, n))
print("L%d eps %g %s: timeline (us from the first panel kernel; median of 10 replays)" % (L, eps, kw))
for a_, b_, i, n in sorted(rows, key=lambda r: r[0]):
    print("  %2d %-10s %-8s p%-2d h%-2d items %5d %7.1f -> %7.1f  (%5.1f)  %6.1f MB  deps %s" % (
        i, n.name, n.stream, n.priority, n.phase.height, n.phase.nitems, a_, b_, b_ - a_, n.phase.bytes / 1e6,
        n.deps))
