"""Print the matvec plan's node table (name, stream, priority, deps, phase
size) and each phase replayed alone; run from a repo root (works on older
trees too, for A/B comparisons)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_1810_08429_b200 import cli, geometry, h2

L = int(sys.argv[1]) if len(sys.argv) > 1 else 6
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
mesh = geometry.build_sphere_mesh(L)
hm, tree, bt = cli.build_h2_operator(mesh, cli.default_config(level=L, eps=eps))
p = h2.plan(hm)
x = torch.randn(mesh.nt, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(5):
    p.run(x, y)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(100):
    p.run(x, y)
b.record()
torch.cuda.synchronize()
print("product us %.1f" % (a.elapsed_time(b) * 10))
flush = torch.empty(32 << 20, dtype=torch.float64, device="cuda")
for i, n in enumerate(p.nodes):
    P = n.phase
    line = "%2d %-10s %-6s prio %3s deps %-16s" % (i, n.name, n.stream, n.priority, n.deps)
    if P is not None:
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
        for e0, e1 in ev:
            flush.zero_()
            e0.record()
            p._launch(P, h2.stream_handle() if hasattr(h2, "stream_handle") else torch.cuda.current_stream().cuda_stream)
            e1.record()
        torch.cuda.synchronize()
        t = np.median([e0.elapsed_time(e1) for e0, e1 in ev]) * 1e3
        line += " h %2d items %6d MB %8.2f in %7d out %7d pair %d ring %d  alone %7.1f us" % (
            P.height, P.nitems, P.bytes / 1e6, P.in_elems, P.out_elems, int(bool(getattr(P, "pair", 0))),
            int(bool(getattr(P, "ring", 0))), t)
    print(line, flush=True)
