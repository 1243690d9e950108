"""BASELINE.json configs 2, 3 and 5 (single GPU): CB-GMRES(100) time to
solution per basis format, iterations, convergence delay vs the fp64 basis,
final explicit RRN and the explicit RRN at the first restart boundaries.

  python scripts/config_sweep.py [--configs 2,3,5] [--reps 2]
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_15468_b200 as cbg  # noqa: E402

CONFIGS = {
    2: ("poisson128", 0, 128, 0.0, ["f64", "frsz2-32", "f32", "frsz2-21", "frsz2-16"]),
    3: ("convdiff192", 1, 192, 1.0, ["f64", "frsz2-32", "frsz2-21", "frsz2-16", "f32"]),
    5: ("p27-512", 2, 512, 0.0, ["f64", "frsz2-32"]),
}

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="2,3,5")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--formats", default=None)
args = ap.parse_args()

for c in [int(x) for x in args.configs.split(",")]:
    name, kind, nx, pe, fmts = CONFIGS[c]
    if args.formats:
        fmts = args.formats.split(",")
    t0 = time.time()
    A = cbg.stencil(kind, nx, pe=pe)
    n = nx ** 3
    xs = torch.from_numpy(cbg.sin_problem_host(n)).cuda()
    b = cbg.spmv(A, xs)
    del xs
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    ref_its = None
    for f in fmts:
        # timed solves without per-phase events (those serialise the
        # programmatic dependent launches), then one phase-timed solve
        S = cbg.Solver(A, cbg.GmresConfig(storage_format=cbg.StorageFormat.parse(f)))
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        r = S.solve(b, x=x)  # warm-up
        ms = []
        for _ in range(args.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = S.solve(b, x=x)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        del S
        S = cbg.Solver(A, cbg.GmresConfig(storage_format=cbg.StorageFormat.parse(f), phase_timing_deferred=True))
        S.solve(b, x=x)
        S.phase_times()
        S.solve(b, x=x)
        ph = {k: round(v, 3) for k, v in S.phase_times().items() if v}
        explicit = [(h.iteration, h.rrn) for h in r.residual_history if h.is_explicit]
        if f == "f64":
            ref_its = r.total_iterations
        line = {"config": c, "workload": name, "n": n, "nnz": A.desc.nnz, "format": f,
                "converged": r.converged, "iterations": r.total_iterations, "restarts": r.restarts,
                "delay_vs_f64": round(r.total_iterations / ref_its, 4) if ref_its else None,
                "final_rrn": r.final_rrn, "explicit_rrn_at_restarts": explicit[1:4],
                "reorth_passes": r.stats.reorth_passes,
                "ms_per_solve": round(min(ms), 3), "ms_each": [round(v, 3) for v in ms],
                "phase_ms": ph, "setup_s": round(setup_s, 2)}
        print(json.dumps(line), flush=True)
        del S, x
        torch.cuda.empty_cache()
    del A, b
    torch.cuda.empty_cache()
