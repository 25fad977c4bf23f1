"""Block-row sharding of the H2 operator over GPUs (SURVEY.md §8 e).

One process per GPU (``torch.distributed``, NCCL over NVLink).  With
P = 2^k ranks, rank g owns the g-th cluster-tree node at depth k: a
contiguous range of tree-ordered rows.

* Assembly needs no communication for the row side.  Every admissible
  block sits at tree level >= 4 and every near-field block at the leaf
  level, so all block rows of a shard lie inside it.  Each rank builds the
  row and column bases of its own subtree.  Every basis root sits at tree
  depth >= 4 >= k, so no node straddles shards.
* Coupling entries on rank g need the column pivots of remote clusters
  sigma.  Tensor all-gathers of the per-rank (node, rank, pivots) arrays
  (:func:`_all_gather_arrays`: lengths, then the arrays padded to the
  longest; a few MB) give every rank the global column pivot table.
* Matvec:
  1. all-gather the owned slice of x (tree order) -> full x_t;
  2. forward transform of the own column subtree into the own slot of a
     rank-major x-hat layout;
  3. all-gather the x-hat slots;
  4. coupling, backward transform, near field and leaf basis for the own
     rows -> the owned slice of y (tree order).
  Rows are disjoint, so no reduction is needed.

The host-side layout logic (``ShardLayout``) is pure numpy and is tested
with ``gloo`` on the CPU (tests/test_parallel.py).  The device path reuses
the single-GPU kernels unchanged.
"""

import numpy as np

from .errors import ConfigError, StateError


def shard_nodes(flat, world):
    """Tree nodes owning the shards: the nodes at depth log2(world), in row
    order."""
    if world < 1 or world & (world - 1):
        raise ConfigError("world size must be a power of two, got %d" % world)
    k = world.bit_length() - 1
    ids = np.flatnonzero(flat.depth == k)
    ids = ids[np.argsort(flat.start[ids], kind="stable")]
    if len(ids) != world or (k and not np.all(flat.left[flat.parent[ids]] >= 0)):
        raise ConfigError("cluster tree too shallow for %d shards" % world)
    return ids


def shard_range(flat, world, rank):
    node = shard_nodes(flat, world)[rank]
    return int(flat.start[node]), int(flat.stop[node])


def check_shardable(btree, world):
    """Every block row must lie inside one shard (block rows at depth >= k)."""
    fb = btree.flat
    k = world.bit_length() - 1
    rows = fb.row[fb.leaf_ids]
    depth = fb.row_tree.depth[rows]
    if np.any(depth < k):
        raise ConfigError("block rows above tree depth %d: shard with fewer GPUs" % k)


class ShardLayout:
    """Per-rank partition data that needs no GPU.

    ``lo, hi`` own tree rows; ``own_leaves`` block-tree leaf ids (DFS order)
    of the own block rows; ``global_coef(...)`` the rank-major column
    coefficient layout assembled from every rank's (nodes, ranks).
    """

    def __init__(self, tree, btree, world, rank):
        self.world, self.rank = world, rank
        flat = tree.flat
        check_shardable(btree, world)
        self.lo, self.hi = shard_range(flat, world, rank)
        fb = btree.flat
        rows = fb.row[fb.leaf_ids]
        inside = (flat.start[rows] >= self.lo) & (flat.stop[rows] <= self.hi)
        self.own_leaves = fb.leaf_ids[inside]

    @staticmethod
    def global_coef(flat, per_rank):
        """per_rank: list of (nodes, ranks) of each rank's column basis.
        Returns (offset per tree node (-1 absent), slot size): rank g's
        coefficients occupy [g*slot, g*slot + size_g) laid out breadth
        first with siblings adjacent (gca.coef_layout)."""
        from .gca import coef_layout
        n = len(flat)
        rank_all = np.zeros(n, dtype=np.int64)
        off = np.full(n, -1, dtype=np.int64)
        layouts = []
        for nodes, ranks in per_rank:
            nodes = np.asarray(nodes, dtype=np.int64)
            rank_all[nodes] = ranks
            present = np.zeros(n, dtype=bool)
            present[nodes] = True
            par = flat.parent[nodes]
            roots = nodes[(par < 0) | ~present[np.maximum(par, 0)]]
            roots = roots[np.argsort(roots, kind="stable")]
            o, size = coef_layout(flat, roots, rank_all)
            layouts.append((nodes, o, size))
        slot = max([size for _, _, size in layouts] + [1])
        for g, (nodes, o, _) in enumerate(layouts):
            off[nodes] = g * slot + o[nodes]
        return off, slot


# --------------------------------------------------------------------------
# device path

def _all_gather_arrays(arr, group, device):
    """Variable-length int64 arrays from every rank (tensor all-gathers:
    the lengths, then the arrays padded to the longest)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    on = device if dist.get_backend(group) == "nccl" else torch.device("cpu")
    a = torch.as_tensor(np.asarray(arr, np.int64)).to(on)
    n = torch.tensor([a.numel()], dtype=torch.int64, device=on)
    ns = torch.zeros(world, dtype=torch.int64, device=on)
    dist.all_gather_into_tensor(ns, n, group=group)
    ns = ns.cpu().numpy()
    m = max(int(ns.max()), 1)
    pad = torch.zeros(m, dtype=torch.int64, device=on)
    pad[:a.numel()] = a
    out = torch.zeros(world * m, dtype=torch.int64, device=on)
    dist.all_gather_into_tensor(out, pad, group=group)
    out = out.cpu().numpy()
    return [out[g * m:g * m + int(ns[g])] for g in range(world)]


def all_gather_into(out, inp, group):
    """out = concat over ranks of inp (equal sizes).  NCCL gathers device
    tensors directly, in place when inp is out's own slot; other backends
    (gloo: the multi-process functional test on one GPU) stage through host
    memory."""
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, inp, group=group)
        return
    parts = [torch.empty(inp.numel(), dtype=inp.dtype) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, inp.detach().cpu(), group=group)
    out.copy_(torch.cat(parts).to(out.device))


class ShardedH2:
    """Own block rows of the H2 operator on this rank's GPU.

    ``mvm(x)`` is the reference's ``mvm(h, x)`` (``h2.py:63-80``): the full
    vector in external ordering on every rank, the full product back on
    every rank.  ``mvm_slice`` works on this rank's tree-ordered slice
    (device tensors) - the per-rank hot path of the benchmark."""

    def __init__(self, h, layout, group, slot, ranges):
        self.h = h
        self.layout = layout
        self.group = group
        self.slot = slot
        self.ranges = ranges            # (lo, hi) of every rank
        self.plan = None
        self.shape = h.shape

    def _plan(self):
        import torch
        if self.plan is None:
            with torch.cuda.device(self.h.dev.device):
                self.plan = ShardPlan(self)
        return self.plan

    def mvm_slice(self, x_slice, out=None):
        """Own slice of y = H x (tree order, device) from the own slice of x
        (device); written into ``out`` when given, else a new tensor."""
        import torch
        p = self._plan()
        with torch.cuda.device(p.dev):
            return p.run_slice(x_slice, out)

    mvm_local = mvm_slice

    def mvm(self, x):
        """y = H x for the full host vector x (external order), on every
        rank: the shard's rows gathered on the device, the three all-gathers
        (x slices, x-hat slots, y slices) over NCCL, the product scattered
        back to external order, one host copy in and one out."""
        import torch
        n = self.shape[1]
        x = np.asarray(x, dtype=np.float64)
        if x.shape != (n,):
            raise ConfigError("vector of length %d, operator wants %d" % (x.size, n))
        p = self._plan()
        with torch.cuda.device(p.dev):
            return p.run_external(x)


def build_sharded_operator(mesh, cfg, group=None, device=None, timings=None):
    """Trees, block tree, own bases, all-gathered column pivots and the own
    block rows of the GCA-H2 matrix for this rank."""
    import time

    import torch
    import torch.distributed as dist

    from . import gca
    from .clustering import build_block_tree, build_cluster_tree
    from .device import require_device, to_dev
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = require_device(device)
    t0 = time.perf_counter()
    tree = build_cluster_tree(mesh, basis_kind=cfg.basis, leaf_size=cfg.leaf_size, device=dev)
    btree = build_block_tree(tree, eta=cfg.eta)
    layout = ShardLayout(tree, btree, world, rank)
    rng = (layout.lo, layout.hi)
    orders = (cfg.q_reg, cfg.q_sing)
    rmarks, cmarks = gca.coupling_mark_arrays(btree)
    t1 = time.perf_counter()
    row_kind = "collocation" if cfg.disc == "collocation" else cfg.basis      # cli.py:167
    rb, cb = gca.build_cluster_bases(tree, mesh, cfg.basis, cfg.m, cfg.delta_factor, cfg.eps,
                                     [("row", rmarks, row_kind), ("col", cmarks, cfg.basis)], orders,
                                     dev, row_range=rng)
    t2 = time.perf_counter()
    cs = cb.store
    flat = tree.flat
    own = np.flatnonzero(cs.materialized)
    own_piv = (np.concatenate([cs.pivots_host[cs.piv_off[i]:cs.piv_off[i] + cs.rank[i]] for i in own])
               if own.size else np.zeros(0, np.int64))
    nodes_g = _all_gather_arrays(own, group, dev)
    ranks_g = _all_gather_arrays(cs.rank[own], group, dev)
    pivs_g = _all_gather_arrays(own_piv, group, dev)
    # global column pivot table (host and device) and rank-major coefficient layout
    pos = 0
    for nodes, ranks in zip(nodes_g, ranks_g):
        cs.rank[nodes] = ranks
        cs.piv_off[nodes] = pos + np.cumsum(ranks) - ranks
        pos += int(ranks.sum())
    cs.pivots_host = np.concatenate(pivs_g) if pos else np.zeros(0, np.int64)
    cs.pivots = to_dev(cs.pivots_host if pos else np.zeros(1, np.int64), dev)
    cs.coef_off, slot = ShardLayout.global_coef(flat, list(zip(nodes_g, ranks_g)))
    cs.coef_size = world * slot
    cs.available = cs.available.copy()
    for nodes in nodes_g:
        cs.available[nodes] = True
    h = gca.build_h2(btree, rb, cb, mesh, kind="slp", basis=cfg.basis, disc=cfg.disc,
                     orders=orders, device=dev, row_range=rng)
    torch.cuda.synchronize(dev)
    t3 = time.perf_counter()
    if timings is not None:
        timings.update(trees_s=t1 - t0, bases_s=t2 - t1, build_h2_s=t3 - t2, total_s=t3 - t0)
    ranges = [shard_range(flat, world, g) for g in range(world)]
    return ShardedH2(h, layout, group, slot, ranges)


def _shard_plan_class():
    from .device import ptr, stream_handle, to_dev
    from .h2 import PanelPlan

    class ShardPlan(PanelPlan):
        """PanelPlan of one shard.  x_t is the all-gather buffer of the
        ranks' tree-ordered slices, each padded to the longest shard (slot
        g at g * maxs: NCCL needs equal sizes), and every x_t index of the
        plan is mapped into it.  Per product: the own slice lands in the
        own slot; then, concurrently, the x all-gather (in place, on its own
        stream) and the forward transform of the own column subtree and the
        near-field blocks with local columns; the x-hat all-gather (in
        place); the coupling blocks with local columns run as soon as the
        forward tiers they read are done, those with remote columns after
        the x-hat all-gather (adding onto the same y-hat rows), likewise the
        remote near-field blocks after the x all-gather; backward transform
        and leaf rows; y_own = y_t + y_t2 over the own rows
        (gc_scatter2_inv).  Over NCCL the whole slice product is one CUDA
        graph."""

        def __init__(self, sh):
            import torch
            import torch.distributed as dist
            from .h2 import _NativeGraph, _Node
            self.sh = sh
            world, g = sh.layout.world, sh.layout.rank
            lo_hi = np.asarray(sh.ranges, np.int64).reshape(-1, 2)
            sizes = lo_hi[:, 1] - lo_hi[:, 0]
            self.maxs = maxs = int(sizes.max())
            self.lo, self.hi = int(lo_hi[g, 0]), int(lo_hi[g, 1])
            n = int(lo_hi[-1, 1])
            owner = np.repeat(np.arange(world), sizes)
            xmap = owner * maxs + (np.arange(n) - lo_hi[owner, 0])      # tree -> padded position
            super().__init__(sh.h, xt_map=xmap, xt_len=world * maxs, col_local=(self.lo, self.hi))
            dev = self.dev
            d = sh.h.dev
            m_own = self.hi - self.lo
            self.m_own = m_own
            self.xt_own = self.xt[g * maxs:(g + 1) * maxs]
            self.xhat_own = self.xhat[g * sh.slot:(g + 1) * sh.slot]
            self.ypad = torch.zeros(world * maxs, dtype=torch.float64, device=dev)
            self.y_own = self.ypad[g * maxs:(g + 1) * maxs]
            self.x_in = torch.zeros(m_own, dtype=torch.float64, device=dev)
            self.y_out = torch.zeros(m_own, dtype=torch.float64, device=dev)
            self._ident = to_dev(np.arange(m_own, dtype=np.int64), dev)
            self._own_rows = to_dev(np.arange(self.lo, self.hi, dtype=np.int64), dev)
            # external API: own rows of x (external ids) -> own slot; padded y -> external y
            perm_c = d.perm_c.cpu().numpy()
            iperm_r = _inv_np(d.perm_r.cpu().numpy())
            self._ext_own = to_dev(perm_c[self.lo:self.hi].astype(np.int64), dev)
            self._ext_from_pad = to_dev(xmap[iperm_r].astype(np.int64), dev)
            self.nccl = dist.get_backend(sh.group) == "nccl"
            self.comm = None
            if self.nccl:
                # the plan's own NCCL communicator (csrc/nccl.cu): the id
                # travels once over the process group, the collectives are
                # nodes of the native product graph
                uid = (_native_ctypes().c_char * 128)()
                if g == 0:
                    _native_call("gc_nccl_unique_id", uid)
                box = [bytes(uid)]
                dist.broadcast_object_list(box, src=0, group=sh.group)
                uid = (_native_ctypes().c_char * 128).from_buffer_copy(box[0])
                c = _native_ctypes().c_void_p(0)
                _native_call("gc_nccl_comm_init", uid, world, g, _native_ctypes().byref(c))
                self.comm = c
            st = stream_handle

            def ag(name, own, full, count):
                return _Node(name, "chain", fn=lambda: self._all_gather(own, full, count),
                             native=(4, [own.data_ptr(), full.data_ptr(), count, (self.comm.value or 0) if self.comm else 0]))
            gather = _Node("gather", "chain", fn=lambda: _native_call(
                "gc_gather_inv", ptr(self.x_in), ptr(self._ident), m_own, ptr(self.xt_own), st()),
                native=(2, [self.x_in.data_ptr(), self._ident.data_ptr(), m_own, self.xt_own.data_ptr()]),
                launches=1)
            combine = _Node("scatter", "chain", fn=lambda: _native_call(
                "gc_scatter2_inv", ptr(self.yt), ptr(self.yt2), ptr(self._own_rows), m_own, ptr(self.y_out),
                st()), native=(3, [self.yt.data_ptr(), self.yt2.data_ptr(), self._own_rows.data_ptr(), m_own,
                                   self.y_out.data_ptr()]), launches=1)
            self.nodes = self._build_nodes(gather=gather, after_gather=[ag("allgather-x", self.xt_own, self.xt, maxs)],
                                           before_coupling=ag("allgather-xhat", self.xhat_own, self.xhat, sh.slot),
                                           scatter=combine)
            self.graph = None
            if self.nccl:
                # the whole slice product - both all-gathers included - as one
                # native CUDA graph; a capture failure raises
                tab = self._native_table()
                if tab is None:
                    raise StateError("sharded product: node without a native form")
                self._body()
                torch.cuda.synchronize(dev)
                rows, deps, ndeps, prio = tab
                hh = _native_ctypes().c_void_p(0)
                _native_call("gc_plan_create", len(rows), rows.ctypes.data, ndeps, deps.ctypes.data, len(prio),
                             prio.ctypes.data, _native_ctypes().byref(hh))
                self.graph = _NativeGraph(hh)

        def _all_gather(self, own, full, count):
            if self.nccl:
                _native_call("gc_nccl_all_gather", ptr(own), ptr(full), count, self.comm, stream_handle())
            else:
                all_gather_into(full, own, self.sh.group)

        def run_slice(self, x_slice, out=None):
            if x_slice.numel() != self.m_own:
                raise ConfigError("slice of length %d, shard owns %d rows" % (x_slice.numel(), self.m_own))
            import torch
            with self.lock:
                res = torch.empty(self.m_own, dtype=torch.float64, device=self.dev) if out is None else out
                if self.graph is not None and x_slice.is_contiguous() and res.is_contiguous() \
                        and x_slice.dtype == torch.float64 and x_slice.device == self.dev:
                    self.graph.bind(x_slice, res)            # the graph reads / writes the caller's slices
                    self.graph.replay()
                else:
                    self.x_in.copy_(x_slice, non_blocking=True)
                    self._exec(self.nodes)
                    res.copy_(self.y_out, non_blocking=True)
                return res

        def run_external(self, x):
            import torch
            with self.lock:
                if not hasattr(self, "_pin_x"):
                    self._pin_x = torch.empty(self.n_in, dtype=torch.float64, pin_memory=True)
                    self._x_full = torch.empty(self.n_in, dtype=torch.float64, device=self.dev)
                    self._y_full = torch.empty(self.n_out, dtype=torch.float64, device=self.dev)
                self._pin_x.numpy()[:] = x
                self._x_full.copy_(self._pin_x, non_blocking=True)
                # own slice of x in tree order, straight from the external vector
                _native_call("gc_gather", ptr(self._x_full), ptr(self._ext_own), self.m_own, ptr(self.x_in),
                             stream_handle())
            ys = self.run_slice(self.x_in, self.y_own[:self.m_own])
            with self.lock:
                self._all_gather(self.y_own, self.ypad, self.maxs)
                _native_call("gc_gather", ptr(self.ypad), ptr(self._ext_from_pad), self.n_out, ptr(self._y_full),
                             stream_handle())
                y = torch.empty(self.n_out, dtype=torch.float64, pin_memory=True)
                y.copy_(self._y_full, non_blocking=True)
                torch.cuda.current_stream().synchronize()
                del ys
                return y.numpy()

        def __del__(self):
            if getattr(self, "comm", None) is not None and self.comm.value:
                try:
                    self.graph = None
                    _native_call("gc_nccl_comm_destroy", self.comm)
                except Exception:        # pragma: no cover - interpreter shutdown
                    pass

    return ShardPlan


def _native_call(name, *args):
    from . import _native
    _native.call(name, *args)


def _native_ctypes():
    import ctypes
    return ctypes


def _inv_np(perm):
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(perm), dtype=perm.dtype)
    return inv


def ShardPlan(sh):
    return _shard_plan_class()(sh)


def bench_distributed(args, rank, world, local, metric, workload, clock_sampler=None, peaks=None):
    """bench.py at N > 1: the same workload sharded by block rows, strong
    scaling; time = max over ranks of CUDA-event time per product.  Also
    reports the end-to-end product through ``ShardedH2.mvm`` (host slice in,
    host slice out), the own-kernel launch count, clocks sampled during the
    timed region (rank 0's GPU) and rank 0's dominant launch roofline."""
    import json
    import time

    import numpy as np
    import torch
    import torch.distributed as dist

    from . import _native, cli, geometry, h2
    from .device import stream_handle
    mesh = (geometry.build_sphere_mesh(args.level) if args.geometry == "sphere"
            else geometry.build_cube_mesh(args.level))
    cfg = cli.default_config(level=args.level, eps=args.eps)
    build_sharded_operator(mesh, cfg)             # warm-up
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    timings = {}
    sh = build_sharded_operator(mesh, cfg, timings=timings)
    torch.cuda.synchronize()
    asm = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
    dist.all_reduce(asm, op=dist.ReduceOp.MAX)
    rep = h2.storage_report(sh.h)
    mine = torch.tensor([rep["couplings"] + rep["nearfield"] + rep["leaf_bases"] + rep["transfers"]],
                        dtype=torch.float64, device="cuda")
    dist.all_reduce(mine)
    n = mesh.nt
    nbytes = float(mine.item()) + 16 * n
    m_own = sh.layout.hi - sh.layout.lo
    x = torch.randn(m_own, dtype=torch.float64, device="cuda")
    for _ in range(args.warmup):
        sh.mvm_local(x)
    torch.cuda.synchronize()
    dist.barrier()
    sampler = clock_sampler(local) if (clock_sampler is not None and rank == 0) else None
    if sampler is not None:
        sampler.__enter__()
    # ~1 s of products under the clock sampler, then the timed steps
    flag = torch.ones(1, dtype=torch.float64, device="cuda")
    w0 = time.perf_counter()
    while True:
        for _ in range(20):
            sh.mvm_local(x)
        torch.cuda.synchronize()
        flag.fill_(1.0 if time.perf_counter() - w0 < 1.0 else 0.0)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)       # every rank stops together
        if flag.item() == 0.0:
            break
    dist.barrier()
    torch.cuda.synchronize()
    l0 = _native.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        sh.mvm_local(x)
    e1.record()
    torch.cuda.synchronize()
    launches = torch.tensor([_native.launch_count() - l0], dtype=torch.float64, device="cuda")
    t = torch.tensor([e0.elapsed_time(e1) * 1e-3 / args.steps], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(launches)
    dist.barrier()
    if sampler is not None:
        sampler.__exit__(None, None, None)
    # end to end through the public sharded API (the reference's mvm(h, x)
    # signature): the full host vector in, the full product back, every rank
    xh = np.random.default_rng(0).standard_normal(n)
    for _ in range(3):
        sh.mvm(xh)
    torch.cuda.synchronize()
    dist.barrier()
    k_e2e = max(10, args.steps // 2)
    w0 = time.perf_counter()
    for _ in range(k_e2e):
        sh.mvm(xh)
    te = torch.tensor([(time.perf_counter() - w0) / k_e2e], dtype=torch.float64, device="cuda")
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    # rank 0: its largest coupling bucket launched alone, L2 flushed
    roof = None
    if rank == 0 and sh.plan is not None:
        p = sh.plan
        buckets = [P for P in p.phases if P.name == "coupling"]
        if buckets:
            big = max(buckets, key=lambda P: P.bytes)
            flush = torch.empty(32 << 20, dtype=torch.float64, device="cuda")
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(5)]
            for a_, b_ in ev:
                flush.zero_()
                a_.record()
                p._launch(big, stream_handle())
                b_.record()
            torch.cuda.synchronize()
            del flush
            sec = float(np.mean([a_.elapsed_time(b_) for a_, b_ in ev])) * 1e-3
            byts = big.bytes + 8 * big.in_elems + 8 * big.out_elems
            hbm = (peaks or {}).get("hbm_gbs", 6650.0)
            roof = {"bound": "hbm", "kernel": "k_panelmv, rank 0's largest coupling bucket",
                    "achieved": round(byts / sec / 1e9, 1), "peak": hbm, "unit": "GB/s",
                    "frac": round(byts / sec / 1e9 / hbm, 4), "traffic": None,
                    "algorithmic_bytes_per_launch": int(byts), "avg_launch_s": sec,
                    "step": {"achieved": round(nbytes / float(t.item()) / 1e9, 1),
                             "frac": round(nbytes / float(t.item()) / 1e9 / hbm, 4)}}
    scale = None
    if getattr(args, "scale_level", 0) > 0:
        sh = None
        torch.cuda.empty_cache()
        scale = _scaling_config(args, world, mesh_level=args.scale_level, eps=args.scale_eps)
    if rank == 0:
        s = float(t.item())
        print(json.dumps({
            "metric": metric, "value": round(nbytes / s / 1e9, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(s * 1e3, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": dict(workload, parallelism="block-row x%d" % world),
            "assembly": {"value": round(float(asm.item()), 4), "unit": "s",
                         "phases_s": {k: round(v, 4) for k, v in timings.items()}},
            "roofline": roof,
            "e2e": {"value": round(nbytes / float(te.item()) / 1e9, 2), "unit": "GB/s",
                    "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                    "ms_per_step": round(float(te.item()) * 1e3, 4),
                    "api": "paper_1810_08429_b200.parallel.ShardedH2.mvm(numpy x, external order) on every "
                           "rank: own rows gathered on the device, x / x-hat / y all-gathered over NCCL"},
            "gpu_launches": int(launches.item()),
            "gpu_launches_note": "own kernels over all ranks in the timed region",
            "clocks": sampler.summary() if sampler is not None else None,
            "scaling_config": scale}))
    dist.destroy_process_group()


def _scaling_config(args, world, mesh_level, eps):
    """The scaling configuration (BASELINE configs[3], C4: sphere level 8,
    eps 1e-8) sharded over the ranks: sharded assembly, then the whole
    sharded product (both NCCL all-gathers included) timed with CUDA events,
    max over ranks.  bench.py's N = 1 line carries the same measurement on
    one GPU, so the per-N lines give C4's strong scaling directly."""
    import time

    import torch
    import torch.distributed as dist

    from . import cli, geometry, h2
    mesh = geometry.build_sphere_mesh(mesh_level)
    cfg = cli.default_config(level=mesh_level, eps=eps)
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sh = build_sharded_operator(mesh, cfg)
    torch.cuda.synchronize()
    asm = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
    dist.all_reduce(asm, op=dist.ReduceOp.MAX)
    rep = h2.storage_report(sh.h)
    mine = torch.tensor([rep["couplings"] + rep["nearfield"] + rep["leaf_bases"] + rep["transfers"]],
                        dtype=torch.float64, device="cuda")
    dist.all_reduce(mine)
    nbytes = float(mine.item()) + 16 * mesh.nt
    x = torch.randn(sh.layout.hi - sh.layout.lo, dtype=torch.float64, device="cuda")
    for _ in range(max(3, args.warmup)):
        sh.mvm_local(x)
    k = max(10, min(args.steps, 50))
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        sh.mvm_local(x)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) * 1e-3 / k], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    s = float(t.item())
    return {"workload": "unit sphere level %d (%d triangles), SLP Galerkin p0, GCA-H2 eps=%g%s"
                        % (mesh_level, mesh.nt, eps,
                           " (BASELINE configs[3], C4)" if (mesh_level, eps) == (8, 1e-8) else ""),
            "n_gpus": world, "value": round(nbytes / s / 1e9, 2), "unit": "GB/s",
            "ms_per_step": round(s * 1e3, 4), "steps": k, "matvec_bytes": int(nbytes),
            "assembly_s": round(float(asm.item()), 3), "parallelism": "block-row x%d" % world,
            "note": "whole sharded product incl. the x and x-hat all-gathers, max over ranks; "
                    "assembly without a warm-up run"}
