import os, sys
os.environ["CBGX_TRACE_FUSED"] = "1"
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2409_15468_b200 as cbg
from paper_2409_15468_b200 import _lib
A = cbg.stencil(0, 128)
b = cbg.spmv(A, torch.from_numpy(cbg.sin_problem_host(128 ** 3)).cuda())
for its in (10, 20):
    acc = None
    for rep in range(5):
        S = cbg.Solver(A, cbg.GmresConfig(storage_format=cbg.StorageFormat.parse("frsz2-32"), max_total_iterations=its))
        S.solve(b)
        t = np.zeros(32 + 3 * 1024, np.uint64)
        _lib.check(_lib.lib().cbgx_debug_fused_trace(t.ctypes.data, t.size))
        st = t[32 + 2048:32 + 3072].astype(np.int64)
        d0 = t[32:32 + 1024].astype(np.int64)
        d1 = t[32 + 1024:32 + 2048].astype(np.int64)
        g = int((st > 0).sum())
        dur = np.stack([(d0[:g] - st[:g]) / 1e3, (d1[:g] - d0[:g]) / 1e3])
        acc = dur if acc is None else acc + dur
    acc /= 5
    print("cols", its, "grid", g)
    for name, row in (("dot1", acc[0]), ("upd1", acc[1])):
        q = row.reshape(-1, 8).mean(axis=1)
        print(" ", name, "by 8-CTA bucket:", " ".join("%.1f" % v for v in q))
        print("   even/odd blockIdx:", row[0::2].mean().round(2), row[1::2].mean().round(2), " first/second half:", row[:g//2].mean().round(2), row[g//2:].mean().round(2))
