"""Assembly time (fresh mesh, after a warm-up) for values of one device /
gca / h2 module constant, alternating, N repetitions each.  Usage:
python scripts/asm_ab.py NAME v1,v2 level eps [reps]"""
import ast
import gc
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_08429_b200 import cli, clustering, device as _device, gca, geometry, h2  # noqa: E402

name, vals = sys.argv[1], [ast.literal_eval(v) for v in sys.argv[2].split(",")]
L, eps = int(sys.argv[3]), float(sys.argv[4])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 4
cfg = cli.default_config(eps=eps)
hm, _, _ = cli.build_h2_operator(geometry.build_sphere_mesh(L), cfg)
h2.plan(hm)
del hm
gc.collect()
torch.cuda.synchronize()
res = {v: [] for v in vals}
for r in range(reps):
    for v in vals:
        setattr(next(mod for mod in (_device, gca, h2, clustering) if hasattr(mod, name)), name, v)
        mesh = geometry.build_sphere_mesh(L)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hm, _, _ = cli.build_h2_operator(mesh, cfg)
        h2.plan(hm)
        torch.cuda.synchronize()
        res[v].append(time.perf_counter() - t0)
        del hm
        gc.collect()
        torch.cuda.synchronize()
for v in vals:
    ts = sorted(res[v])
    print("L%d %s=%s  min %.4f  median %.4f s" % (L, name, v, ts[0], ts[len(ts) // 2]), flush=True)
