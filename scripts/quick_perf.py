"""Quick kernel timings (CUDA events) -- development aid, not the bench."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2409_15468_b200 as cbg  # noqa: E402
from paper_2409_15468_b200 import _lib  # noqa: E402

peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if __import__("os").path.exists("MEASURED_PEAKS.json") else 6535.4
flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")


def timeit(fn, reps=5):
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts), float(np.median(ts))


out = {}
n = 1 << 24
x = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
for l in (32, 21, 16):
    cv = cbg.compress(x, cbg.Frsz2Params(32, l))
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    L = _lib.lib()
    bad = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    tc = timeit(lambda: L.cbgx_frsz2_compress_async(x.data_ptr(), n, 32, l, cv.exps.data_ptr(), cv.payload.data_ptr(), bad.data_ptr(), st))
    td = timeit(lambda: L.cbgx_frsz2_decompress(cv.exps.data_ptr(), cv.payload.data_ptr(), n, 32, l, y.data_ptr(), st))
    byt = n * (8 + (l + 1) / 8)
    out[f"codec_l{l}"] = dict(compress_ms=tc[0], compress_gbs=byt / tc[0] / 1e6, decompress_ms=td[0],
                              decompress_gbs=byt / td[0] / 1e6)
print(json.dumps(out, indent=1), flush=True)

n = 1 << 26
for fmt in ("frsz2-32", "f64", "frsz2-16", "frsz2-21", "f32"):
    kmax = 100 if fmt != "f64" else 60
    B = cbg.KrylovBasis(n, kmax, cbg.StorageFormat.parse(fmt))
    col = torch.randn(n, dtype=torch.float64, device="cuda")
    for j in range(kmax):
        B.write_vector(j, col)
    w = torch.randn(n, dtype=torch.float64, device="cuda")
    h = torch.randn(kmax + 1, dtype=torch.float64, device="cuda") * 1e-3
    bpv = {"f64": 8, "f32": 4, "f16": 2, "frsz2-16": 17 / 8, "frsz2-21": 22 / 8, "frsz2-32": 33 / 8}[fmt]
    res = {}
    for k in (10, 50, kmax):
        td = timeit(lambda: B.cgs_dot(k, w, out=h))
        tu = timeit(lambda: B.cgs_update(k, h, w))
        bd = k * n * bpv + 8 * n
        bu = k * n * bpv + 16 * n
        res[k] = dict(dot_ms=td[0], dot_gbs=bd / td[0] / 1e6, dot_frac=bd / td[0] / 1e6 / peak,
                      upd_ms=tu[0], upd_gbs=bu / tu[0] / 1e6, upd_frac=bu / tu[0] / 1e6 / peak)
    print(fmt, json.dumps(res), flush=True)
    del B
    torch.cuda.empty_cache()

for fmt in ("frsz2-32", "f64"):
    A = cbg.stencil(0, 128)
    xs = torch.from_numpy(cbg.sin_problem_host(128 ** 3)).cuda()
    b = cbg.spmv(A, xs)
    S = cbg.Solver(A, cbg.GmresConfig(storage_format=cbg.StorageFormat.parse(fmt), phase_timing=True))
    S.solve(b)
    t0 = time.time()
    r = S.solve(b)
    t1 = time.time()
    st = r.stats
    print(fmt, "iters", r.total_iterations, "final", r.final_rrn, "wall_ms", (t1 - t0) * 1e3,
          {p: round(st.phase_ms[i], 3) for i, p in enumerate(_lib.PHASES)},
          {p: round(st.phase_bytes[i] / max(st.phase_ms[i], 1e-9) / 1e6, 1) for i, p in enumerate(_lib.PHASES)}, flush=True)
    S2 = cbg.Solver(A, cbg.GmresConfig(storage_format=cbg.StorageFormat.parse(fmt), phase_timing=False))
    S2.solve(b)
    torch.cuda.synchronize()
    t0 = time.time()
    r = S2.solve(b)
    torch.cuda.synchronize()
    print(fmt, "no-timing wall_ms", (time.time() - t0) * 1e3)
