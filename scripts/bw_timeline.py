"""HBM traffic of the product over time, from per-CTA %globaltimer records
(PanelPhase.trace with a per-CTA table): every CTA's algorithmic bytes
(matrix + gathered inputs + indices + outputs) spread over its [start, end]
and summed into 2 us bins, median replay of 5.  Usage:
python scripts/bw_timeline.py level eps [key=value ...] (PanelPlan kwargs)."""
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
mesh = geometry.build_sphere_mesh(L)
hm, _, _ = cli.build_h2_operator(mesh, cli.default_config(eps=eps))
p = h2.PanelPlan(hm, **kw)
x = torch.randn(mesh.nt, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
info = {}
for i, n in enumerate(p.nodes):
    P = n.phase
    if P is None:
        continue
    it = P.items.cpu().numpy().reshape(-1, 8)
    b = 8 * it[:, 3] * it[:, 4] + 12 * it[:, 4] + 8 * it[:, 3]
    ncta = (P.nitems + 1) // 2 if P.pair else P.nitems
    if P.pair:
        b = np.add.reduceat(b, np.arange(0, len(b), 2))
    t = torch.zeros(4 + 2 * ncta, dtype=torch.int64, device="cuda")
    p.trace[id(P)] = t
    info[id(P)] = (i, n, ncta, b, t)
p.capture()
for _ in range(3):
    p.run(x, y)
runs = []
for rep in range(5):
    for (_, _, ncta, _, t) in info.values():
        t.zero_()
        t[0] = 2 ** 63 - 1
        t[2] = ncta
    torch.cuda.synchronize()
    p.run(x, y)
    torch.cuda.synchronize()
    runs.append({k: v[4].cpu().numpy().copy() for k, v in info.items()})
# the median-length replay
span = [max(r[k][5::2].max() for k in r) - min(r[k][4::2].min() for k in r) for r in runs]
r = runs[int(np.argsort(span)[len(span) // 2])]
t0 = min(r[k][4::2].min() for k in r)
T = (max(r[k][5::2].max() for k in r) - t0) / 1e3
nb = int(np.ceil(T / 2.0))
tot = np.zeros(nb)
per = {}
for k, (i, n, ncta, b, _) in info.items():
    st = (r[k][4::2] - t0) / 1e3
    en = (r[k][5::2] - t0) / 1e3
    acc = np.zeros(nb)
    for s_, e_, by in zip(st, en, b):
        e_ = max(e_, s_ + 1e-3)
        lo, hi = int(s_ // 2), min(int(e_ // 2), nb - 1)
        for q in range(lo, hi + 1):
            ov = min(e_, 2.0 * (q + 1)) - max(s_, 2.0 * q)
            if ov > 0:
                acc[q] += by * ov / (e_ - s_)
    tot += acc
    per["%d %s h%d" % (i, n.name[:4], n.phase.height)] = acc
print("L%d eps %g %s: product %.1f us (first CTA start to last CTA end), %.1f MB algorithmic" % (
    L, eps, kw, T, sum(v.sum() for v in per.values()) / 1e6))
for q in range(nb):
    top = sorted(((v[q], name) for name, v in per.items() if v[q] > 0), reverse=True)[:4]
    print("%6.1f us %6.2f TB/s  %s" % (2.0 * q, tot[q] / 2e-6 / 1e12,
                                       "  ".join("%s %.1f" % (nm, val / 2e-6 / 1e12) for val, nm in top)))
