"""Where does the panel-plan DAG spend its time?  Graph-replay timings of
node subsets: full DAG, serial DAG, chain only, bulk only (coupling + near
with no chain dependencies), and each phase replayed alone as a graph."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1810_08429_b200 import cli, geometry, h2

L = int(sys.argv[1]) if len(sys.argv) > 1 else 6
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
geo = sys.argv[3] if len(sys.argv) > 3 else "sphere"
mesh = (geometry.build_sphere_mesh if geo == "sphere" else geometry.build_cube_mesh)(L)
hm, tree, bt = cli.build_h2_operator(mesh, cli.default_config(level=L, eps=eps))
p = h2.plan(hm)
x = torch.randn(mesh.nt, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
nbytes = h2.storage_report(hm)["total"] + 16 * mesh.nt


def subset(keep):
    idx = [i for i, n in enumerate(p.nodes) if keep(n)]
    remap = {o: k for k, o in enumerate(idx)}
    out = []
    for i in idx:
        n = p.nodes[i]
        out.append(h2._Node(n.name, n.stream, [remap[d] for d in n.deps if d in remap], n.phase, n.fn, n.priority))
    return out


def time_graph(nodes, serial=False, reps=50):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        p._exec(nodes, serial=serial)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        p._exec(nodes, serial=serial)
    torch.cuda.synchronize()
    for _ in range(5):
        g.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


p.run(x, y)
for _ in range(3):
    full = time_graph(p.nodes)
    print("full DAG        %7.1f us  %6.0f GB/s" % (full, nbytes / full / 1e3))
print("serial          %7.1f us" % time_graph(p.nodes, serial=True))
chain = subset(lambda n: n.stream == "chain")
print("chain only      %7.1f us  (%d nodes)" % (time_graph(chain), len(chain)))
for n in p.nodes: print("   node", n.name, n.stream, n.deps, n.priority, (n.phase.height, n.phase.nitems, round(n.phase.bytes / 1e6, 1)) if n.phase else "")
bulk = [h2._Node(n.name, n.stream, [], n.phase, n.fn, n.priority) for n in p.nodes
        if n.name in ("coupling", "nearfield")]
print("bulk only       %7.1f us  (%d nodes, concurrent)" % (time_graph(bulk), len(bulk)))
print("bulk serial     %7.1f us" % time_graph(bulk, serial=True))
print("per node (graph of one node):")
for n in p.nodes:
    if n.phase is None and n.name not in ("forward", "backward"):
        continue
    t = time_graph([h2._Node(n.name, "chain", [], n.phase, n.fn)], reps=100)
    P = n.phase
    if P is None:
        print("  %-10s segment                       %7.1f us" % (n.name, t))
        continue
    print("  %-10s h%-2d items %6d red %5d  %7.1f us  %6.1f MB  %6.0f GB/s" % (
        P.name, P.height, P.nitems, P.nred, t, P.bytes / 1e6, P.bytes / t / 1e3))

# timeline of the concurrent DAG inside the CUDA graph: every panel kernel
# stamps min(start)/max(end) %globaltimer into its trace slot
if os.environ.get("TIMELINE", "1") == "1":
    slots = {}
    for n in p.nodes:
        if n.phase is not None:
            t = torch.zeros(2, dtype=torch.int64, device="cuda")
            p.trace[id(n.phase)] = t
            slots[id(n.phase)] = t
    p.graph = None
    p.capture()
    res = []
    for rep in range(10):
        for t in slots.values():
            t[0] = 2 ** 63 - 1
            t[1] = 0
        torch.cuda.synchronize()
        p.run(x, y)
        torch.cuda.synchronize()
        res.append({k: v.cpu().numpy().copy() for k, v in slots.items()})
    print("graph timeline (us from the first panel kernel; median of 10 replays):")
    rows = []
    for i, n in enumerate(p.nodes):
        if n.phase is None:
            continue
        st = [r[id(n.phase)][0] - min(v[0] for v in r.values()) for r in res]
        en = [r[id(n.phase)][1] - min(v[0] for v in r.values()) for r in res]
        rows.append((np.median(st) / 1e3, np.median(en) / 1e3, n))
    for a_, b_, n in sorted(rows, key=lambda r: r[0]):
        print("  %-10s %-5s p%-2d h%-2d %7.1f -> %7.1f  (%5.1f)  %6.1f MB" % (
            n.name, n.stream, n.priority, n.phase.height, a_, b_, b_ - a_, n.phase.bytes / 1e6))
    p.trace.clear()
