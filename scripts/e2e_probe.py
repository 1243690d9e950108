"""Breakdown of the host drop-in solve (CBGX_PROFILE_HOST_SOLVE=1)."""
import os
import sys
import time

os.environ["CBGX_PROFILE_HOST_SOLVE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, ".")
import paper_2409_15468_b200 as cbg  # noqa: E402

A = cbg.stencil(0, 128)
n = 128 ** 3
xs = torch.from_numpy(cbg.sin_problem_host(n)).cuda()
b = cbg.spmv(A, xs)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
rp = pin(A.row_ptr.cpu().numpy().astype(np.uint64))
ci = pin(A.col_idx.cpu().numpy().astype(np.uint64))
va = pin(A.values.cpu().numpy())
bh = pin(b.cpu().numpy())
x0 = pin(np.zeros(n))
xo = pin(np.zeros(n))
cfg = cbg.GmresConfig(storage_format=cbg.StorageFormat.parse("frsz2-32"))
a = cbg.CsrMatrix(n, n, rp, ci, va)
for i in range(4):
    t = time.perf_counter()
    cbg.gmres_solve(a, bh, x0, cfg, out=xo)
    print("total %.3f ms" % ((time.perf_counter() - t) * 1e3), flush=True)
