"""Small end-to-end exercise of every kernel family for compute-sanitizer:
codec (3 fast formats + generic), basis write/read, split CGS, fused
orthogonalisation (+ folded SpMV variant), staged / plain / SELL SpMV, read
sweep, host drop-in solve."""
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
    b = cbg.spmv(A, torch.from_numpy(cbg.sin_problem_host(n)).cuda())
    for fmt in ("frsz2-32", "f64"):
        for fold in (False, True):
            S = cbg.Solver(A, cbg.GmresConfig(restart=20, storage_format=cbg.StorageFormat.parse(fmt), fold=fold,
                                              max_total_iterations=60))
            r = S.solve(b)
            print(kind, fmt, fold, r.total_iterations, r.final_rrn, flush=True)
    rp = A.row_ptr.cpu().numpy().astype(np.uint64)
    ci = A.col_idx.cpu().numpy().astype(np.uint64)
    va = A.values.cpu().numpy()
    r = cbg.gmres_solve(cbg.CsrMatrix(n, n, rp, ci, va), b.cpu().numpy(), np.zeros(n),
                        cbg.GmresConfig(restart=20, storage_format=cbg.StorageFormat.parse("frsz2-32"),
                                        max_total_iterations=60))
    print("host", kind, r.total_iterations, flush=True)
torch.cuda.synchronize()
print("sanitize_small done")
