"""Small end-to-end exercise of every kernel family for compute-sanitizer:
codec (3 fast formats + generic), basis write/read (+ exponent ranges),
split CGS, fused orthogonalisation (fast and exact columns, one fused step
through the C-ABI), staged / plain / SELL / dictionary SpMV (2-byte ELL4,
ragged SELL, 1-byte pair codes, slice ranges), read sweep, host drop-in
solve, partitioned solve on in-process ranks (window halo, overlapped
interior SpMV, merged collectives)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2409_15468_b200 as cbg  # noqa: E402

rng = np.random.default_rng(0)
v = rng.standard_normal(5000)
for l in (16, 21, 32):
    cv = cbg.compress(v, cbg.Frsz2Params(32, l))
    cbg.decompress(cv)
cv = cbg.compress(v, cbg.Frsz2Params(8, 7))
cbg.decompress(cv)
for fmt in ("f64", "f32", "f16", "frsz2-16", "frsz2-21", "frsz2-32"):
    B = cbg.KrylovBasis(5000, 4, cbg.StorageFormat.parse(fmt))
    for j in range(4):
        B.write_vector(j, rng.standard_normal(5000))
    w = torch.from_numpy(rng.standard_normal(5000)).cuda()
    h = B.cgs_dot(4, w)
    B.cgs_update(4, h, w)
    cbg.read_sweep(B, 1, 4992, 2, 1.0, 0.0)
for kind, nx in ((0, 20), (2, 14), (1, 18)):
    A = cbg.stencil(kind, nx, pe=1.0 if kind == 1 else 0.0)
    n = nx ** 3
    x = torch.from_numpy(rng.standard_normal(n)).cuda()
    cbg.spmv(A, x)
    t = cbg.spmv_plan(A)
    if t:
        cbg.spmv_staged(A, x, t, want_norm=True)
    D = cbg.DictCsr(A)
    D.spmv(x, want_norm=True)
    D.spmv(x, b=x)
    b = cbg.spmv(A, torch.from_numpy(cbg.sin_problem_host(n)).cuda())
    for fmt in ("frsz2-32", "f64"):
        for dic in (True, False):
            S = cbg.Solver(A, cbg.GmresConfig(restart=20, storage_format=cbg.StorageFormat.parse(fmt), 
                                              dict_spmv=dic, max_total_iterations=60))
            r = S.solve(b)
            print(kind, fmt, dic, r.total_iterations, r.final_rrn, flush=True)
    rp = A.row_ptr.cpu().numpy().astype(np.uint64)
    ci = A.col_idx.cpu().numpy().astype(np.uint64)
    va = A.values.cpu().numpy()
    r = cbg.gmres_solve(cbg.CsrMatrix(n, n, rp, ci, va), b.cpu().numpy(), np.zeros(n),
                        cbg.GmresConfig(restart=20, storage_format=cbg.StorageFormat.parse("frsz2-32"),
                                        max_total_iterations=60))
    print("host", kind, r.total_iterations, flush=True)
# ragged few-valued matrix: dictionary SELL layout (per-slice offsets)
nr = 3001
lens = rng.integers(0, 12, size=nr)
lens[rng.random(nr) < 0.1] = 0
rp = np.zeros(nr + 1, dtype=np.uint64)
rp[1:] = np.cumsum(lens)
rows = [sorted({min(nr - 1, max(0, r + int(o))) for o in rng.choice(np.arange(-40, 41), size=int(L))}) for r, L in
        enumerate(lens)]
rp[1:] = np.cumsum([len(c) for c in rows])
ci = np.array([c for cs in rows for c in cs], dtype=np.uint64)
va = rng.choice([1.0, -2.0, 0.5], size=ci.size)
Ar = cbg.DeviceCsr.from_host(cbg.CsrMatrix(nr, nr, rp, ci, va))
try:
    Dr = cbg.DictCsr(Ar)
    Dr.spmv(torch.from_numpy(rng.standard_normal(nr)).cuda(), want_norm=True)
except Exception as e:  # many distinct offsets: refused (still exercises the scan kernel)
    print("dict refused:", e)
# one fused Arnoldi step with a tiny-block column (exact decoder) and an
# all-zero block (clamped fast scale)
n5 = 40000
B5 = cbg.KrylovBasis(n5, 8, cbg.StorageFormat.parse("frsz2-32"))
cols = rng.standard_normal((4, n5))
cols[1, 32:64] *= 1e-300
cols[2, 64:96] = 0.0
for j in range(4):
    B5.write_vector(j, cols[j])
w5 = torch.from_numpy(rng.standard_normal(n5)).cuda()
B5.arnoldi_fused_step(4, w5, float((w5 * w5).sum()), 7)
# partitioned solve: P ranks as threads (halo, pell slice ranges, merged collectives)
import ctypes  # noqa: E402
from paper_2409_15468_b200 import _lib  # noqa: E402
from oracle import pyoracle as po  # noqa: E402
P = po.Port()
rp, ci, va = P.stencil(0, 16, 16, 16)
bb, _ = P.generate_problem(rp, ci, va)
nn = rp.size - 1
cfg = cbg.GmresConfig(restart=20, storage_format=cbg.StorageFormat.parse("frsz2-32"), max_total_iterations=40)
xx = np.zeros(nn)
h, bufs = cbg._history_buffers(2 * cfg.max_total_iterations + 4)
st = _lib.SolveStats()
c = cfg.c()
_lib.check(_lib.lib().cbgx_gmres_solve_partitioned_local(nn, rp.ctypes.data, ci.ctypes.data, va.ctypes.data,
                                                         bb.ctypes.data, np.zeros(nn).ctypes.data, ctypes.byref(c),
                                                         3, xx.ctypes.data, ctypes.byref(h), ctypes.byref(st)))
print("partitioned", st.total_iterations, flush=True)
torch.cuda.synchronize()
print("sanitize_small done")
