"""Benchmark: CB-GMRES(100) time-to-solution with an FRSZ2-32 Krylov basis.

Headline workload (BASELINE.json configs[1]): 7-point Poisson 128^3
(n = 2,097,152, nnz = 14,581,760), generate_problem's sin right-hand side,
x0 = 0, restart 100, target explicit RRN 1e-10, eta = 1/sqrt(2). A "step" is
one complete solve. value = device time per solve (CUDA events on the solve
stream, max over ranks), lower is better. The same solve with an fp64 basis
on the same GPU is reported beside it (north_star: FRSZ2-32 must beat the
fp64-basis GMRES at equal final residual).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload poisson128|convdiff192|p27-512] [--format frsz2-32]

N > 1 (torchrun, one process per GPU): the same solve row-partitioned over N
GPUs (strong scaling) with libcbgx's own NCCL communicator.
--impl reference: the reference's CPU implementation of the same solve
(oracle/_ref: /root/reference/proj/src compiled unmodified by build()), on
the host, bounded to a few minutes.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (stencil kind, nx, peclet)
    "poisson128": (0, 128, 0.0),
    "convdiff192": (1, 192, 1.0),
    "p27-512": (2, 512, 0.0),
    "p27-128": (2, 128, 0.0),
    "poisson64": (0, 64, 0.0),
}
FMT_BYTES = {"f64": 8.0, "f32": 4.0, "f16": 2.0, "frsz2-16": 17 / 8, "frsz2-21": 22 / 8, "frsz2-32": 33 / 8}


def traffic_for(kernel):
    """Measured DRAM bytes per launch of `kernel` from the committed ncu
    launch list of one solve (profiles/traffic.json, scripts/
    traffic_from_launches.py); None when absent."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None, None
    with open(p) as f:
        d = json.load(f)
    e = d.get(kernel)
    return (e["bytes_per_launch"], d.get("_source")) if e else (None, None)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
    }

    def __init__(self, device_index: int, period_s: float = 0.002):
        self.samples, self.reasons = [], set()
        self.period = period_s
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self.nv = None
            self.err = str(e)

    def _sample(self):
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for name, bit in self.REASONS.items():
                if r & bit and name != "gpu_idle":
                    self.reasons.add(name)
        except Exception:  # noqa: BLE001
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()
            # one more reading at the end of the timed region (the work is
            # still queued/finishing): at least two samples per region even
            # when the host thread starves the sampler
            self._sample()

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "")}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def read_peak_gbs(torch):
    """Measured read-only streaming bandwidth (torch sum over 4 GiB of fp64,
    best of 5, CUDA events): the second roofline denominator BASELINE.md asks
    for beside the copy-based MEASURED_PEAKS.json figure."""
    x = torch.ones(1 << 29, dtype=torch.float64, device="cuda")
    best = None
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        x.sum()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    del x
    torch.cuda.empty_cache()
    return round((8 << 29) / best / 1e6, 1)


def shared_config(workload, fmt, n, nnz, ours, world=1, l2="", spmv=""):
    """The config dict both arms print (same keys; values describe each arm)."""
    return {
        "workload": f"CB-GMRES(100) {fmt} basis, {workload}: n={n}, nnz={nnz}",
        "format": fmt, "restart": 100, "target_rrn": 1e-10, "eta": 0.70710678118654752, "x0": "zeros",
        "reduction": "tree (deterministic, fixed shape)" if ours else "sequential (the reference's order)",
        "l2": l2, "spmv": spmv,
        "parallelism": (f"row-partition x{world}" if world > 1 else "single GPU") if ours
        else "single host thread (the reference has no threading)",
    }


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# --------------------------------------------------------------- our arm
def run_ours(args):
    import torch

    import paper_2409_15468_b200 as cbg
    from paper_2409_15468_b200 import _lib

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    _lib.check(_lib.lib().cbgx_set_device(local))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    kind, nx, pe = WORKLOADS[args.workload]
    n = nx ** 3
    fmt = args.format
    peak, peak_kind = peaks()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- problem setup (not timed): matrix generated on the device, sin RHS
    if world == 1:
        A = cbg.stencil(kind, nx, pe=pe)
        xs = torch.from_numpy(cbg.sin_problem_host(n)).cuda()
        b = cbg.spmv(A, xs)
        nnz = A.desc.nnz
        rows = n

        def make_solver(f, phases=False):
            return cbg.Solver(A, cbg.GmresConfig(storage_format=cbg.StorageFormat.parse(f),
                                                 phase_timing_deferred=phases))
    else:
        from paper_2409_15468_b200 import dist as cdist
        comm = cdist.NcclComm(rank, world)
        prob = cdist.DistStencil(comm, kind, nx, nx, nx, pe)
        b, xs = prob.sin_rhs()
        nnz = prob.A.desc.nnz
        rows = prob.re - prob.rb

        def make_solver(f, phases=False):
            return cdist.DistSolver(prob, cbg.GmresConfig(storage_format=cbg.StorageFormat.parse(f),
                                                           phase_timing_deferred=phases))
        A = prob.A
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()

    xbuf = torch.empty(rows, dtype=torch.float64, device="cuda")  # solution buffer reused by every solve

    def timed_solves(solver, steps, warmup, sampler=None):
        # W warm-up solves, and at least ~1.5 s of GPU work so the SM clock
        # has left its idle state before the timed region
        t_w = time.perf_counter()
        done = 0
        while done < warmup or time.perf_counter() - t_w < 1.5:
            solver.solve(b, x=xbuf)
            done += 1
        solver.phase_times()  # drop warm-up phase events
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        l0 = _lib.lib().cbgx_launch_count()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        results = []
        ctx = sampler if sampler is not None else _Null()
        import gc
        gc.collect()
        gc.disable()   # keep the Python collector out of the timed region
        t_host = time.perf_counter()
        with ctx:
            ev0.record(stream)
            for _ in range(steps):
                results.append(solver.solve(b, x=xbuf))
            ev1.record(stream)
            torch.cuda.synchronize()
        t_host = (time.perf_counter() - t_host) * 1e3 / steps
        gc.enable()
        results[-1].host_ms = t_host
        barrier()
        launches = _lib.lib().cbgx_launch_count() - l0
        ms = ev0.elapsed_time(ev1) / steps
        return max_over_ranks(ms), results, launches, solver.phase_times()

    # ---- headline: FRSZ2 basis. The timed solves run without per-phase
    # events (they would serialise the programmatic dependent launches); a
    # second, phase-timed set of solves gives the per-kernel breakdown.
    solver = make_solver(fmt)
    sampler = ClockSampler(local)
    ms, results, launches, _ = timed_solves(solver, args.steps, args.warmup, sampler)
    del solver
    solver = make_solver(fmt, phases=True)
    ms_phased, _, _, phases = timed_solves(solver, args.steps, 1)
    last = results[-1]
    st = last.stats
    # per-solve bytes by phase (identical for every step of the same solve)
    ph_bytes = {p: st.phase_bytes[i] for i, p in enumerate(_lib.PHASES)}
    ph_launch = {p: int(st.phase_launches[i]) for i, p in enumerate(_lib.PHASES)}
    ph_ms = {p: phases[p] / args.steps for p in _lib.PHASES}
    dominant = max(("dot", "update", "spmv", "ortho"), key=lambda p: ph_ms[p])
    kernel_name = {"dot": "cgs_dot_kernel", "update": "cgs_update_kernel", "spmv": "spmv_kernel",
                   "ortho": "arnoldi_fused_kernel"}[dominant]
    achieved = ph_bytes[dominant] / (ph_ms[dominant] * 1e-3) / 1e9 if ph_ms[dominant] > 0 else None
    del solver
    torch.cuda.empty_cache()

    # ---- fp64-basis GMRES on the same GPU(s) (comparison baseline)
    ref64 = None
    if fmt != "f64" and not args.no_fp64:
        s64 = make_solver("f64")
        ms64, r64, _, _ = timed_solves(s64, max(1, args.steps // 2), 1)
        del s64
        s64 = make_solver("f64", phases=True)
        _, _, _, ph64 = timed_solves(s64, max(1, args.steps // 2), 1)
        ref64 = {"ms_per_solve": ms64, "wall_each": [round(r.stats.wall_seconds * 1e3, 2) for r in r64],
                 "python_loop_ms_per_solve": round(r64[-1].host_ms, 3), "iterations": r64[-1].total_iterations,
                 "restarts": r64[-1].restarts, "final_rrn": r64[-1].final_rrn,
                 "converged": r64[-1].converged, "speedup_frsz2_vs_fp64": ms64 / ms,
                 "phase_ms_per_solve": {p: round(v / max(1, args.steps // 2), 4) for p, v in ph64.items() if v}}
        del s64
        torch.cuda.empty_cache()

    # ---- the same solve with the general CSR SpMV path (no dictionary copy):
    # what a matrix outside the dictionary pattern (> 255 distinct values or
    # column offsets, e.g. SuiteSparse systems) gets
    csr_path = None
    if world == 1 and not args.no_fp64:
        sc = cbg.Solver(A, cbg.GmresConfig(storage_format=cbg.StorageFormat.parse(fmt), dict_spmv=False))
        ms_csr, r_csr, _, _ = timed_solves(sc, max(1, args.steps // 2), 1)
        csr_path = {"ms_per_solve": round(ms_csr, 4), "iterations": r_csr[-1].total_iterations,
                    "final_rrn": r_csr[-1].final_rrn,
                    "spmv": "staged (bulk-copy) CSR kernel, 12 B per entry"}
        del sc
        torch.cuda.empty_cache()

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        if world == 1:
            rp = A.row_ptr.cpu().numpy().astype(np.uint64)
            ci = A.col_idx.cpu().numpy().astype(np.uint64)
            va = A.values.cpu().numpy()
            bh = b.cpu().numpy()
            pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
            rp, ci, va, bh = pin(rp), pin(ci), pin(va), pin(bh)
            x0 = pin(np.zeros(n))
            xo = pin(np.zeros(n))
            a_host = cbg.CsrMatrix(n, n, rp, ci, va)
            cfg = cbg.GmresConfig(storage_format=cbg.StorageFormat.parse(fmt))
            cbg.gmres_solve(a_host, bh, x0, cfg, out=xo)  # warm (allocator pools)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            k = max(1, args.steps // 2)
            for _ in range(k):
                r = cbg.gmres_solve(a_host, bh, x0, cfg, out=xo)
            t1 = time.perf_counter()
            e2e = {"value": (t1 - t0) * 1e3 / k, "unit": "ms",
                   "h2d_bytes_per_step": int(rp.nbytes + ci.nbytes + va.nbytes + bh.nbytes + x0.nbytes),
                   "d2h_bytes_per_step": int(8 * n),
                   "api": "paper_2409_15468_b200.gmres_solve (cbgx_gmres_solve_host): host size_t CSR + b + x0 "
                          "in pinned memory, solution back into a pinned host array, every step",
                   "iterations": r.total_iterations, "final_rrn": r.final_rrn}
        else:
            from paper_2409_15468_b200 import dist as cdist  # noqa: F401
            s2 = make_solver(fmt)
            bh = torch.empty(rows, dtype=torch.float64).pin_memory()
            bh.copy_(b.cpu())
            xh = torch.empty(rows, dtype=torch.float64).pin_memory()
            x0h = torch.zeros(rows, dtype=torch.float64).pin_memory()
            bd = torch.empty_like(b)
            x0d = torch.empty_like(b)
            s2.solve(b)
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            k = max(1, args.steps // 2)
            for _ in range(k):
                bd.copy_(bh, non_blocking=True)
                x0d.copy_(x0h, non_blocking=True)
                r = s2.solve(bd, x0d)
                xh.copy_(r.solution[:rows], non_blocking=True)
                torch.cuda.synchronize()
            barrier()
            t1 = time.perf_counter()
            e2e = {"value": max_over_ranks((t1 - t0) * 1e3 / k), "unit": "ms",
                   "h2d_bytes_per_step": int(16 * rows), "d2h_bytes_per_step": int(8 * rows),
                   "api": "paper_2409_15468_b200.dist.DistSolver.solve with pinned host b/x0/x per rank "
                          "(matrix generated on each rank's GPU once)"}
            del s2

    # ---- codec (config 1) and CGS micro numbers on rank 0
    codec = None
    if rank == 0 and not args.no_codec:
        codec = codec_bench(cbg, torch, peak)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(kind, nx, pe, fmt)

    clocks = sampler.summary()
    read_peak = read_peak_gbs(torch) if rank == 0 else None
    if rank == 0:
        bpv = FMT_BYTES[fmt]
        line = {
            "metric": f"cbgmres_{fmt.replace('-', '_')}_time_to_solution",
            "value": round(ms, 4),
            "unit": "ms",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms, 4),
            "higher_is_better": False,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic: device-generated 3-D stencil, generate_problem sin RHS (glibc sin, sequential norm)",
            "config": shared_config(
                args.workload, fmt, n, nnz if world == 1 else "partitioned", True, world,
                l2="inputs larger than L2: per solve the basis grows to %.0f MB (up to %.0f MB at m=100) "
                   "plus the matrix (%s) vs 126 MB L2; no explicit flush"
                   % (last.total_iterations * bpv * rows / 1e6, 101 * bpv * rows / 1e6,
                      "1-byte row-pattern ids, ~%.0f MB" % (rows / 1e6) if world == 1
                      else "1-byte dictionary codes per rank"),
                spmv=("row-pattern coded dictionary copy of the CSR (one byte per row into <=255 distinct rows "
                      "of (value, column offset) pairs -- 27 for a 7-point box stencil; bit-identical to the CSR "
                      "SpMV), built at setup" if world == 1
                      else "pair-coded dictionary copy of each rank's rows in the window halo layout "
                           "[lower ghost planes | own rows | upper ghost planes]; interior rows overlap the "
                           "NCCL halo exchange")),
            "iterations": last.total_iterations,
            "restarts": last.restarts,
            "final_rrn": last.final_rrn,
            "converged": last.converged,
            "fp64_basis": ref64,
            "csr_spmv_path": csr_path,
            "phase_ms_per_solve": {p: round(v, 4) for p, v in ph_ms.items() if v},
            "ms_per_solve_phase_timed": round(ms_phased, 4),
            "phase_gbs": {p: round(ph_bytes[p] / (ph_ms[p] * 1e-3) / 1e9, 1) for p in ph_ms if ph_ms[p] > 0},
            "roofline": {
                "kernel": kernel_name,
                "bound": "hbm",
                "achieved": round(achieved, 1) if achieved else None,
                "peak": peak,
                "peak_source": peak_kind,
                "unit": "GB/s",
                "frac": round(achieved / peak, 4) if achieved else None,
                "frac_datasheet_8000": round(achieved / 8000.0, 4) if achieved else None,
                "read_peak_gbs": read_peak,
                "frac_read_peak": round(achieved / read_peak, 4) if achieved and read_peak else None,
                "traffic": traffic_for(kernel_name)[0],
                "traffic_source": "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch, averaged over one "
                                  "solve's launches of this kernel (%s); compare with algorithmic_bytes_per_launch"
                                  % traffic_for(kernel_name)[1],
                "algorithmic_bytes_per_launch": round(ph_bytes[dominant] / max(1, ph_launch[dominant])),
                "algorithmic_bytes_per_solve": ph_bytes[dominant],
                "launches_per_solve": ph_launch[dominant],
                "note": "achieved = algorithmic bytes of the %s phase (sum over its launches in a solve; basis "
                        "%.4f B/value per column per pass, w/v 8 B/row per read or write; the fused 'ortho' kernel "
                        "counts 2 or 4 basis passes + w read + v and column write) / its CUDA-event time, "
                        "averaged over the timed solves" % (dominant, bpv),
            },
            "codec": codec,
            "e2e": e2e,
            "host_ms_per_solve": {"enqueue": round(st.host_enqueue_ms, 3), "wait": round(st.host_wait_ms, 3),
                                  "wall": round(st.wall_seconds * 1e3, 3),
                                  "wall_each": [round(r.stats.wall_seconds * 1e3, 2) for r in results],
                                  "python_loop_ms_per_solve": round(results[-1].host_ms, 3)},
            "gpu_launches": int(launches),
            "gpu_launches_per_solve": round(launches / args.steps, 1),
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def codec_bench(cbg, torch, peak):
    """Config 1: 2^24 uniform[-1,1) round trip, l = 32 (kernel time, L2 flushed)."""
    from paper_2409_15468_b200 import _lib
    L = _lib.lib()
    n = 1 << 24
    x = (torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1)
    flush = torch.empty(512 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream()
    out = {}
    for l in (32, 21, 16):
        cv = cbg.compress(x, cbg.Frsz2Params(32, l))
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        bad = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        tc, td = [], []
        for _ in range(8):
            flush.fill_(0.0)
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(st)
            L.cbgx_frsz2_compress_async(x.data_ptr(), n, 32, l, cv.exps.data_ptr(), cv.payload.data_ptr(),
                                        bad.data_ptr(), st.cuda_stream)
            e1.record(st)
            flush.fill_(1.0)
            e2.record(st)
            L.cbgx_frsz2_decompress(cv.exps.data_ptr(), cv.payload.data_ptr(), n, 32, l, y.data_ptr(),
                                    st.cuda_stream)
            e3 = torch.cuda.Event(enable_timing=True)
            e3.record(st)
            torch.cuda.synchronize()
            tc.append(e0.elapsed_time(e1))
            td.append(e2.elapsed_time(e3))
        assert torch.equal(y, cbg.decompress(cv))
        byt = n * (8 + (l + 1) / 8)
        out[f"l{l}"] = {"compress_gbs": round(byt / min(tc) / 1e6, 1), "decompress_gbs": round(byt / min(td) / 1e6, 1),
                        "decompress_frac": round(byt / min(td) / 1e6 / peak, 4),
                        "bytes_per_value": 8 + (l + 1) / 8}
    out["n"] = n
    out["note"] = "best of 8, L2 flushed (512 MiB write) before each kernel; bytes = 8 + (l+1)/8 per value"
    del flush
    torch.cuda.empty_cache()
    return out


def cpu_baseline(kind, nx, pe, fmt, budget_s=60.0):
    """The reference's own gmres_solve (oracle/_ref, single-threaded as the
    reference is) on the same problem: a bounded sample of full solves."""
    from oracle import pyoracle as po
    P = po.Port()
    rp, ci, va = P.stencil(kind, nx, pe=pe)
    if po.Ref.available():
        R = po.Ref()
        b = np.zeros(rp.size - 1)
        xs = np.zeros(rp.size - 1)
        R.lib.ref_generate_problem(rp.size - 1, rp, ci, va, b, xs)
        impl, kindname = R, "reference"
    else:
        b, _ = P.generate_problem(rp, ci, va)
        impl, kindname = P, "port"
    t0 = time.perf_counter()
    solves, its = 0, None
    while True:
        r = impl.gmres(rp, ci, va, b, fmt=fmt, restart=100, target=1e-10)
        solves += 1
        its = r["iterations"]
        if time.perf_counter() - t0 > budget_s / 2 or solves >= 1:
            break
    dt = (time.perf_counter() - t0) / solves
    out = {"value": round(dt * 1e3, 1), "unit": "ms", "cores": 1, "kind": kindname,
           "sample": f"{solves} full gmres_solve(s) of the same workload ({its} iterations), "
                     f"single thread (the reference has no threading), 1 thread of {os.cpu_count()} cores, "
                     f"{cpu_model()}; AVX2 kernel table (CBG_KERNELS unset)",
           "cpu_model": cpu_model(), "host_cores": os.cpu_count(), "iterations": its}
    if kindname == "reference":
        out["scalar_kernels_ms"] = reference_scalar_ms(kind, nx, pe, fmt)
    return out


def reference_scalar_ms(kind, nx, pe, fmt):
    """The same reference solve once with CBG_KERNELS=scalar (kernels.cpp:22-36
    selects the table once per process, so it runs in a child process)."""
    import subprocess
    code = ("import sys,time,numpy as np; sys.path.insert(0, %r); from oracle import pyoracle as po; "
            "P=po.Port(); R=po.Ref(); rp,ci,va=P.stencil(%d,%d,pe=%r); n=rp.size-1; b=np.zeros(n); xs=np.zeros(n); "
            "R.lib.ref_generate_problem(n,rp,ci,va,b,xs); t=time.perf_counter(); "
            "R.gmres(rp,ci,va,b,fmt=%r,restart=100,target=1e-10); print((time.perf_counter()-t)*1e3)"
            % (ROOT, kind, nx, pe, fmt))
    try:
        r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, CBG_KERNELS="scalar"),
                           capture_output=True, text=True, timeout=300)
        return round(float(r.stdout.strip().splitlines()[-1]), 1)
    except Exception:  # noqa: BLE001
        return None


# ---------------------------------------------------------- reference arm
def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import pyoracle as po
    kind, nx, pe = WORKLOADS[args.workload]
    if nx > 192:
        print(json.dumps({"impl": "reference", "unavailable":
                          f"{args.workload} needs >150 GB host RAM and hours on the single-threaded CPU reference"}))
        return
    P = po.Port()
    rp, ci, va = P.stencil(kind, nx, pe=pe)
    n = rp.size - 1
    if po.Ref.available():
        impl, kindname = po.Ref(), "reference"
        b = np.zeros(n)
        xs = np.zeros(n)
        impl.lib.ref_generate_problem(n, rp, ci, va, b, xs)
    else:
        impl, kindname = P, "port"
        b, _ = P.generate_problem(rp, ci, va)
    budget = float(os.environ.get("CBG_REF_BUDGET_S", "150"))
    times, its, fr = [], None, None
    t_all = time.perf_counter()
    warm = min(args.warmup, 1)
    for _ in range(warm):
        if time.perf_counter() - t_all > budget / 3:
            break
        impl.gmres(rp, ci, va, b, fmt=args.format, restart=100, target=1e-10)
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r = impl.gmres(rp, ci, va, b, fmt=args.format, restart=100, target=1e-10)
        times.append(time.perf_counter() - t0)
        its, fr = r["iterations"], r["final_rrn"]
        if time.perf_counter() - t_all > budget:
            break
    ms = statistics.mean(times) * 1e3
    sample = (f"{len(times)} of {args.steps} requested full solves (+{warm} warm-up) of CB-GMRES(100) "
              f"{args.format} on {args.workload} (n={n}), {its} iterations, final RRN {fr:.6e}; bounded to "
              f"~{budget:.0f}s; single thread (the reference has no threading): 1 thread of {os.cpu_count()} cores, "
              f"{cpu_model()}")
    print(json.dumps({
        "impl": "reference",
        "metric": f"cbgmres_{args.format.replace('-', '_')}_time_to_solution",
        "value": round(ms, 2), "unit": "ms", "n_gpus": world, "steps": len(times), "warmup": warm,
        "ms_per_step": round(ms, 2), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (same stencil + sin RHS)",
        "config": shared_config(args.workload, args.format, n, int(rp[-1]), False,
                                l2="host memory (CPU reference)",
                                spmv="CSR sparse.cpp:43-56 (size_t indices), host"),
        "iterations": its, "final_rrn": fr,
        "cpu_baseline": {"value": round(ms, 2), "unit": "ms", "cores": 1, "kind": kindname, "sample": sample,
                         "cpu_model": cpu_model(), "host_cores": os.cpu_count()},
        "e2e": {"value": round(ms, 2), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="poisson128", choices=sorted(WORKLOADS))
    ap.add_argument("--format", default="frsz2-32", choices=sorted(FMT_BYTES))
    ap.add_argument("--no-fp64", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-codec", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
