"""Measurement of the SURVEY 8f rank-2 discretisations (the widened rows):
for each (kernel, basis, discretisation, geometry) variant, the device
assembly time and matvec throughput next to the reference CPU path on the
same host (bench.reference_baseline with the same parameters: trees and
bases in full, quadrature on a block sample extrapolated, matvec on the
reference-built structure).  One JSON object per variant.

    python scripts/bench_variants.py [--level 5] [--eps 1e-4] [--steps 20]
"""
import argparse, json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1810_08429_b200 import cli, geometry, h2

VARIANTS = [  # (kernel, basis, disc, curved)
    ("slp", "constant", "galerkin", False), ("dlp", "constant", "galerkin", False),
    ("slp", "linear", "galerkin", False), ("dlp", "linear", "galerkin", False),
    ("slp", "linear", "collocation", False), ("slp", "constant", "galerkin", True),
    ("slp", "linear", "galerkin", True), ("dlp", "linear", "galerkin", True),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--level", type=int, default=5)
    ap.add_argument("--eps", type=float, default=1e-4)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--cpu-sample", type=float, default=0.01)
    ap.add_argument("--no-cpu", action="store_true")
    a = ap.parse_args()
    base = geometry.build_sphere_mesh(a.level)
    for kernel, basis, disc, curved in VARIANTS:
        mesh = geometry.to_curved(base, project_to_unit_sphere=True) if curved else base
        cfg = cli.default_config(level=a.level, eps=a.eps, basis=basis, disc=disc)
        hm, _, _ = cli.build_h2_operator(mesh, cfg, kind=kernel)          # warm-up
        h2.plan(hm)
        del hm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tm = {}
        hm, _, _ = cli.build_h2_operator(mesh, cfg, kind=kernel, timings=tm)
        p = h2.plan(hm)
        torch.cuda.synchronize()
        asm = time.perf_counter() - t0
        n = mesh.nt if basis == "constant" else mesh.nv
        rep = h2.storage_report(hm)
        nbytes = rep["total"] + 16 * n
        x = torch.randn(n, dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)
        for _ in range(3):
            p.run(x, y)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.steps):
            p.run(x, y)
        e1.record()
        torch.cuda.synchronize()
        mv = e0.elapsed_time(e1) * 1e-3 / a.steps
        line = {"kernel": kernel, "basis": basis, "disc": disc, "curved": curved, "level": a.level,
                "eps": a.eps, "dofs": n, "assembly_s": round(asm, 4),
                "phases_s": {k: round(v, 4) for k, v in tm.items()},
                "exec_tasks": [s["tasks"] for s in hm.exec_stats], "h2_bytes": int(nbytes),
                "matvec_us": round(mv * 1e6, 1), "matvec_gbs": round(nbytes / mv / 1e9, 1)}
        if not a.no_cpu:
            args = argparse.Namespace(level=a.level, eps=a.eps, geometry="sphere")
            rb = bench.reference_baseline(args, 3, a.cpu_sample, basis=basis, disc=disc, kernel=kernel,
                                          curved=curved)
            line["cpu_reference"] = {"assembly_s_extrapolated": round(rb["assembly_s_extrapolated"], 2),
                                     "matvec_gbs": round(rb["matvec_gbs"], 3), "cores": rb["cores"],
                                     "kind": rb["kind"], "sample": rb["sample"]}
            line["speedup"] = {"assembly": round(rb["assembly_s_extrapolated"] / asm, 1),
                               "matvec": round(nbytes / mv / 1e9 / rb["matvec_gbs"], 1)}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
