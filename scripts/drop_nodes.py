"""Upper bound of fusing the gather / scatter into the panel phases: the
product DAG replayed as a graph with those nodes dropped (results wrong,
timing only).  Usage: python scripts/drop_nodes.py level:eps"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_08429_b200 import cli, geometry, h2  # noqa: E402

L, eps = sys.argv[1].split(":")
L, eps = int(L), float(eps)
mesh = geometry.build_sphere_mesh(L)
hm, _, _ = cli.build_h2_operator(mesh, cli.default_config(eps=eps))
nbytes = h2.storage_report(hm)["total"] + 16 * mesh.nt
p = h2.plan(hm)


def subset(drop):
    idx = [i for i, n in enumerate(p.nodes) if n.name not in drop]
    remap = {o: k for k, o in enumerate(idx)}
    out = []
    for i in idx:
        n = p.nodes[i]
        deps = set()
        stack = list(n.deps)
        while stack:                       # inherit the dropped nodes' dependencies
            d = stack.pop()
            if d in remap:
                deps.add(remap[d])
            else:
                stack.extend(p.nodes[d].deps)
        out.append(h2._Node(n.name, n.stream, sorted(deps), n.phase, n.fn, n.priority))
    return out


def time_graph(nodes, reps=100):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        p._exec(nodes)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        p._exec(nodes)
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / reps * 1e3)
    return best


x = torch.randn(mesh.nt, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
p.run(x, y)
torch.cuda.synchronize()
for drop in [(), ("gather",), ("scatter",), ("gather", "scatter"), ("zero",), ("zero", "gather", "scatter")]:
    t = time_graph(subset(set(drop)))
    print("L%d drop %-28s %7.1f us  %6.0f GB/s" % (L, ",".join(drop) or "-", t, nbytes / t / 1e3), flush=True)
