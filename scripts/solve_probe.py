"""Development probe: time repeated solves (fused vs split) with host/GPU splits."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2409_15468_b200 as cbg  # noqa: E402
from paper_2409_15468_b200 import _lib  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 128
kind = int(sys.argv[2]) if len(sys.argv) > 2 else 0
A = cbg.stencil(kind, nx, pe=1.0 if kind == 1 else 0.0)
b = cbg.spmv(A, torch.from_numpy(cbg.sin_problem_host(nx ** 3)).cuda())
for fmt in ("frsz2-32", "f64"):
    for fusion in (True, False):
        S = cbg.Solver(A, cbg.GmresConfig(storage_format=cbg.StorageFormat.parse(fmt), fusion=fusion,
                                          phase_timing_deferred=True))
        for _ in range(2):
            S.solve(b)
        S.phase_times()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        K = 5
        for _ in range(K):
            r = S.solve(b)
        e1.record()
        torch.cuda.synchronize()
        ph = {k: round(v / K, 3) for k, v in S.phase_times().items() if v}
        st = r.stats
        print(json.dumps({"fmt": fmt, "fusion": fusion, "ms": round(e0.elapsed_time(e1) / K, 3),
                          "its": r.total_iterations, "reorth": st.reorth_passes, "phases": ph,
                          "phase_sum": round(sum(ph.values()), 3),
                          "enqueue_ms": round(st.host_enqueue_ms, 3), "wait_ms": round(st.host_wait_ms, 3),
                          "wall_ms": round(st.wall_seconds * 1e3, 3)}), flush=True)

# same loop with the bench's NVML clock sampler running
sys.path.insert(0, ".")
import bench  # noqa: E402

S = cbg.Solver(A, cbg.GmresConfig(storage_format=cbg.StorageFormat.parse("frsz2-32"), phase_timing_deferred=True))
for _ in range(2):
    S.solve(b)
for period in (0.005, 0.05, 0.2):
    smp = bench.ClockSampler(0, period)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with smp:
        e0.record()
        for _ in range(5):
            r = S.solve(b)
        e1.record()
        torch.cuda.synchronize()
    print("sampler period", period, "ms/solve", round(e0.elapsed_time(e1) / 5, 3), smp.summary(), flush=True)
