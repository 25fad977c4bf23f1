"""C5: near-field quadrature + H2 matvec throughput over sphere levels and
quadrature orders q = q_reg = q_sing (m = 3, eps 1e-6).
Prints one JSON object per (level, q)."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1810_08429_b200 import cli, geometry, h2
from paper_1810_08429_b200.assembly import device_block_assembly
from paper_1810_08429_b200.device import DeviceMesh, DeviceRules, SingularQueue

levels = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else [5, 6, 7, 8]
qs = [int(a) for a in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2, 3, 4, 5, 6]
for L in levels:
    t0 = time.time()
    mesh = geometry.build_sphere_mesh(L)
    tmesh = time.time() - t0
    for q in qs:
        cfg = cli.default_config(eps=1e-6, q_reg=q, q_sing=q)
        try:
            hm, tree, bt = cli.build_h2_operator(mesh, cfg)
            torch.cuda.synchronize()
            tm = {}
            t0 = time.time()
            hm, tree, bt = cli.build_h2_operator(mesh, cfg, timings=tm)
            torch.cuda.synchronize()
            asm = time.time() - t0
            d = hm.dev
            dm, rules, queue = DeviceMesh.get(mesh, q, d.device), DeviceRules.get(q, d.device), SingularQueue.get(mesh, d.device)
            ndesc = np.stack([tree.flat.start[d.n_rows], d.n_nr, tree.flat.start[d.n_cols], d.n_nc, d.n_off], 1)
            scratch = torch.empty_like(d.near)
            from paper_1810_08429_b200.device import to_dev
            d_desc = to_dev(ndesc.astype(np.int64), d.device)      # outside the timed region
            ts = []
            for _ in range(3):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                counts = device_block_assembly(dm, rules, queue, d.perm_r, d.perm_c, ndesc, scratch, d_desc=d_desc)
                e1.record(); e1.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e-3)
            tq = float(np.median(ts))
            per_pt = [0, 33, 27, 21]
            flops = counts[0] * (12 * q ** 4 + 24 * q ** 2 + 3) + sum(counts[k] * (per_pt[k] * rules.npts[k] + 3) for k in (1, 2, 3))
            P_full = [0, 2 * q ** 4, 10 * q ** 4, 6 * q ** 4]
            flops_ref = counts[0] * (12 * q ** 4 + 24 * q ** 2 + 3) + sum(counts[k] * (33 * P_full[k] + 3) for k in (1, 2, 3))
            rep = h2.storage_report(hm)
            nbytes = rep["total"] + 16 * mesh.nt
            p = h2.plan(hm)
            x = torch.randn(mesh.nt, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
            for _ in range(3): p.run(x, y)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10): p.run(x, y)
            b.record(); torch.cuda.synchronize()
            mv = a.elapsed_time(b) / 10 * 1e-3
            print(json.dumps({"level": L, "triangles": mesh.nt, "q": q, "assembly_s": round(asm, 4),
                              "phases": {k: round(v, 4) for k, v in tm.items()},
                              "near_quad_s": round(tq, 6), "near_tflops": round(flops / tq / 1e12, 3),
                              "near_ref_rule_tflops": round(flops_ref / tq / 1e12, 3),
                              "near_tasks": counts, "matvec_us": round(mv * 1e6, 1),
                              "matvec_gbs": round(nbytes / mv / 1e9, 1), "h2_bytes": int(nbytes),
                              "mesh_s": round(tmesh, 2)}), flush=True)
            del hm, p, scratch
            torch.cuda.empty_cache()
        except Exception as exc:  # report and continue the sweep
            print(json.dumps({"level": L, "q": q, "error": repr(exc)[:300]}), flush=True)
