"""The device block tables of build_h2 (gc_h2_blocks) against a numpy
restatement of the same rule (leaves in DFS order, admissible -> coupling,
stable grouping by block row), unsharded and for block-row shards.
Usage: python scripts/tables_check.py LEVEL EPS [parts]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_08429_b200 import cli, gca, geometry  # noqa: E402


def grouped(keys, sizes):
    order = np.argsort(keys, kind="stable")
    off = np.empty(len(keys), dtype=np.int64)
    off[order] = np.cumsum(sizes[order]) - sizes[order]
    return off, order


def expect(bt, rf, cf, rs, cs, rng):
    fb = bt.flat
    ids = fb.leaf_ids
    st, lr, lc = fb.state[ids], fb.row[ids], fb.col[ids]
    if rng is not None:
        k = (rf.start[lr] >= rng[0]) & (rf.stop[lr] <= rng[1])
        st, lr, lc = st[k], lr[k], lc[k]
    adm = st == 0
    out = []
    for rows, cols, nr, nc in ((lr[adm], lc[adm], rs.rank[lr[adm]], cs.rank[lc[adm]]),
                               (lr[~adm], lc[~adm], (rf.stop - rf.start)[lr[~adm]], (cf.stop - cf.start)[lc[~adm]])):
        key = rows if rng is None else 2 * rows + ~((cf.start[cols] >= rng[0]) & (cf.stop[cols] <= rng[1]))
        off, order = grouped(key, nr * nc)
        out.append((rows, cols, nr, nc, off, order))
    return out


L, eps = int(sys.argv[1]), float(sys.argv[2])
parts = int(sys.argv[3]) if len(sys.argv) > 3 else 4
cfg = cli.default_config(eps=eps)
mesh = geometry.build_sphere_mesh(L)
hm, tree, bt = cli.build_h2_operator(mesh, cfg)
rf = cf = tree.flat
rs, cs = hm.row_basis.store, hm.col_basis.store
dev = torch.device("cuda", 0)
ok = True
n = len(rf.perm)
ranges = [None] + [(p * n // parts, (p + 1) * n // parts) for p in range(parts)]
for rng in ranges:
    if rng is not None:
        # a shard's rows: clusters inside [lo, hi)
        pass
    tabs = gca._device_block_tables(bt, rf, cf, rs, cs, rng, dev)
    got = tabs.host()
    for kind, (g, e) in enumerate(zip(got, expect(bt, rf, cf, rs, cs, rng))):
        same = all(np.array_equal(a, b) for a, b in zip(g, e))
        ok &= same
        print("range %s kind %s: %d blocks %s" % (rng, ("coupling", "near")[kind], len(e[0]),
                                                 "equal" if same else "DIFFER"))
    torch.cuda.synchronize()
print("ALL EQUAL" if ok else "MISMATCH")
