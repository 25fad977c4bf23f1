"""Block-row sharding (paper_1810_08429_b200.parallel) on the CPU with
gloo, world size 2 and 4: partition, coefficient layout and the exchange
pattern of the sharded matvec, emulated with the oracle's blocks and
checked against the oracle's full product."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import port as P
from paper_1810_08429_b200 import clustering, geometry
from paper_1810_08429_b200.errors import ConfigError
from paper_1810_08429_b200.parallel import ShardLayout, check_shardable, shard_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _setup(level=3, eps=1e-4):
    mesh = geometry.build_sphere_mesh(level)
    tree = clustering.build_cluster_tree(mesh, "constant", 16)
    bt = clustering.build_block_tree(tree, eta=1.0)
    oh = P.H2(mesh.vertices, mesh.triangles, eps)
    return mesh, tree, bt, oh


def _worker(rank, world, port, level, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mesh, tree, bt, oh = _setup(level)
        flat = tree.flat
        lay = ShardLayout(tree, bt, world, rank)
        lo, hi = lay.lo, lay.hi
        inside = lambda i: flat.start[i] >= lo and flat.stop[i] <= hi
        cb = {i: b for i, b in oh.bases["col"].items() if i != "_roots"}
        rb = {i: b for i, b in oh.bases["row"].items() if i != "_roots"}
        own_c = np.array(sorted(i for i in cb if inside(i)), dtype=np.int64)
        mine = (own_c, np.array([len(cb[i]["piv"]) for i in own_c], dtype=np.int64))
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        off, slot = ShardLayout.global_coef(flat, gathered)
        # rank-major layout: own slot, siblings adjacent
        for i in own_c:
            assert rank * slot <= off[i] < (rank + 1) * slot
            if flat.left[i] >= 0:
                l, r = flat.left[i], flat.right[i]
                assert off[r] == off[l] + len(cb[l]["piv"])
        # 1. all-gather of the owned slice of x (tree order)
        x = np.random.default_rng(0).standard_normal(mesh.nt)
        xt_full = x[flat.perm]
        parts = [torch.zeros(hi - lo, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(xt_full[lo:hi].copy()))
        xt = torch.cat(parts).numpy()
        assert np.array_equal(xt, xt_full)
        # 2. forward transform of the own column subtree into the own slot
        xhat = np.zeros(world * slot)
        for i in sorted(own_c, key=lambda i: -flat.depth[i]):
            r = len(cb[i]["piv"])
            if flat.left[i] < 0:
                xhat[off[i]:off[i] + r] = cb[i]["v"].T @ xt[flat.start[i]:flat.stop[i]]
            else:
                acc = np.zeros(r)
                for c in (flat.left[i], flat.right[i]):
                    acc += cb[c]["E"].T @ xhat[off[c]:off[c] + len(cb[c]["piv"])]
                xhat[off[i]:off[i] + r] = acc
        # 3. all-gather of the x-hat slots
        slots = [torch.zeros(slot, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(slots, torch.from_numpy(xhat[rank * slot:(rank + 1) * slot].copy()))
        xhat = torch.cat(slots).numpy()
        # 4. own rows: coupling, backward, near field
        leaves = [bt.flat.row[j] for j in lay.own_leaves]
        yhat = {i: np.zeros(len(b["piv"])) for i, b in rb.items() if inside(i)}
        yt = np.zeros(hi - lo)
        for j in lay.own_leaves:
            i, c = int(bt.flat.row[j]), int(bt.flat.col[j])
            blk = oh.blocks[(i, c)]
            if bt.flat.state[j] == 0:
                yhat[i] += blk @ xhat[off[c]:off[c] + len(cb[c]["piv"])]
            else:
                yt[flat.start[i] - lo:flat.stop[i] - lo] += blk @ xt[flat.start[c]:flat.stop[c]]
        for i in sorted(yhat, key=lambda i: flat.depth[i]):
            if flat.left[i] >= 0:
                for c in (flat.left[i], flat.right[i]):
                    yhat[c] = yhat[c] + rb[c]["E"] @ yhat[i]
            else:
                yt[flat.start[i] - lo:flat.stop[i] - lo] += rb[i]["v"] @ yhat[i]
        ys = [torch.zeros(hi - lo, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(ys, torch.from_numpy(yt))
        y = np.empty(mesh.nt)
        y[flat.perm] = torch.cat(ys).numpy()
        ref = oh.mvm(x)
        q.put((rank, float(np.linalg.norm(y - ref) / np.linalg.norm(ref)), (lo, hi), len(leaves)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_matvec_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 3, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(err < 1e-13 for _, err, _, _ in res), res
    # contiguous, disjoint, covering row ranges
    spans = [r[2] for r in res]
    assert spans[0][0] == 0 and spans[-1][1] == 512
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_partition_covers_every_block_row_once():
    mesh, tree, bt, _ = _setup(4)
    for world in (1, 2, 4, 8):
        owned = np.concatenate([ShardLayout(tree, bt, world, r).own_leaves for r in range(world)])
        assert np.array_equal(np.sort(owned), np.sort(bt.flat.leaf_ids))
        assert shard_range(tree.flat, world, world - 1)[1] == mesh.nt


def test_unshardable_configurations():
    mesh = geometry.build_sphere_mesh(2)
    tree = clustering.build_cluster_tree(mesh, "constant", 16)
    bt = clustering.build_block_tree(tree, eta=1.0)
    with pytest.raises(ConfigError):
        shard_range(tree.flat, 3, 0)
    with pytest.raises(ConfigError):
        check_shardable(bt, 64)
