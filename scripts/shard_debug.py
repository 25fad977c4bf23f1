"""Per-rank error of the sharded product (gloo ranks sharing one GPU) against
the full operator; SPLIT=0 disables the local-first blocks."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def worker(rank, world, port, level, q):
    from paper_1810_08429_b200 import cli, geometry, h2, parallel
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    if os.environ.get("SPLIT", "1") == "0":
        orig = h2.PanelPlan.__init__

        def init(self, h, *a, **kw):
            kw["col_local"] = None
            orig(self, h, *a, **kw)
        h2.PanelPlan.__init__ = init
    mesh = geometry.build_sphere_mesh(level)
    cfg = cli.default_config(eps=1e-6)
    sh = parallel.build_sharded_operator(mesh, cfg)
    n = sh.shape[1]
    x = np.random.default_rng(3).standard_normal(n)
    perm = sh.h.row_tree.flat.perm
    xt = torch.from_numpy(x[perm][sh.layout.lo:sh.layout.hi].copy()).cuda()
    y = sh.mvm_slice(xt).cpu().numpy()
    hm, tree, _ = cli.build_h2_operator(mesh, cfg)
    ref = h2.mvm(hm, x)[perm][sh.layout.lo:sh.layout.hi]
    p = sh.plan
    print("rank %d rows [%d,%d) err %.3e  near_remote %s cpl_remote %d" % (
        rank, sh.layout.lo, sh.layout.hi, np.linalg.norm(y - ref) / np.linalg.norm(ref),
        None if p._near_remote is None else p._near_remote.nitems, len(p._cpl_remote)), flush=True)
    for i, nd in enumerate(p.nodes):
        if rank == 0:
            print("   ", i, nd.name, nd.stream, nd.deps, nd.priority,
                  (nd.phase.height, nd.phase.nitems, nd.phase.acc) if nd.phase is not None else "", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    import socket
    world, level = int(sys.argv[1]), int(sys.argv[2])
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(worker, args=(world, port, level, None), nprocs=world, join=True)
