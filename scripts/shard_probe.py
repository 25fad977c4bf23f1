"""Per-rank work of the block-row sharded product (parallel.py) at world
sizes W, measured on ONE GPU without letting any kernel wait on another
rank: W processes (gloo, host-staged collectives) build their shards of the
same operator; then, one rank at a time between host barriers, each times
its LOCAL product (gather-free plan: forward tiers of its column subtree,
its coupling rows, backward, near field) as a CUDA graph.  The x and x-hat
all-gathers are not in the timed region (they are NCCL collectives on the
real multi-GPU path) and are reported as byte counts.

    python scripts/shard_probe.py LEVEL EPS W [W ...]    -> one JSON line per W
"""
import json, os, socket, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def worker(rank, world, port, level, eps, out):
    from paper_1810_08429_b200 import cli, geometry, h2, parallel
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        mesh = geometry.build_sphere_mesh(level)
        t0 = time.perf_counter()
        sh = parallel.build_sharded_operator(mesh, cli.default_config(level=level, eps=eps))
        torch.cuda.synchronize()
        t_build = time.perf_counter() - t0
        p = parallel.ShardPlan(sh)
        # local work only: no x / x-hat exchange nodes
        nodes = p._build_nodes(gather=False, before_coupling=None, scatter=False)
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            p._exec(nodes)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(st):
            g.capture_begin()
            p._exec(nodes)
            g.capture_end()
        torch.cuda.synchronize()
        rep = h2.storage_report(sh.h)
        res = None
        for r in range(world):
            dist.barrier()
            if r == rank:
                for _ in range(5):
                    g.replay()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(20):
                    g.replay()
                b.record()
                torch.cuda.synchronize()
                res = dict(rank=rank, us=a.elapsed_time(b) / 20 * 1e3, bytes=int(rep["total"]),
                           rows=int(sh.layout.hi - sh.layout.lo), build_s=round(t_build, 3),
                           xhat_slot=int(sh.slot), tiers=p.tiers and [p.tiers["col"], p.tiers["row"]])
            dist.barrier()
        with open(os.path.join(out, "r%d.json" % rank), "w") as f:
            json.dump(res, f)
    finally:
        dist.destroy_process_group()


def main():
    level, eps = int(sys.argv[1]), float(sys.argv[2])
    for world in [int(w) for w in sys.argv[3:]]:
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        out = os.path.join("gpurun_out", "shard_probe_%d" % world)
        os.makedirs(out, exist_ok=True)
        mp.spawn(worker, args=(world, port, level, eps, out), nprocs=world, join=True)
        rs = [json.load(open(os.path.join(out, "r%d.json" % r))) for r in range(world)]
        t = max(r["us"] for r in rs)
        tot = sum(r["bytes"] for r in rs)
        print(json.dumps({"level": level, "eps": eps, "world": world, "max_rank_us": round(t, 1),
                          "mean_rank_us": round(float(np.mean([r["us"] for r in rs])), 1),
                          "bytes_total": tot, "bytes_max_rank": max(r["bytes"] for r in rs),
                          "aggregate_gbs_local": round(tot / t / 1e3, 1),
                          "x_allgather_bytes": 8 * sum(r["rows"] for r in rs),
                          "xhat_allgather_bytes": 8 * world * rs[0]["xhat_slot"],
                          "ranks": rs}), flush=True)


if __name__ == "__main__":
    main()
