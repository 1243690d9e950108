"""Per-CTA duration of the first dot pass in the last fused launch of solves
capped at 20, 21, 22 iterations: is the CTA-to-CTA skew persistent?"""
import os
import sys

os.environ["CBGX_TRACE_FUSED"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, ".")
import paper_2409_15468_b200 as cbg  # noqa: E402
from paper_2409_15468_b200 import _lib  # noqa: E402

A = cbg.stencil(0, 128)
b = cbg.spmv(A, torch.from_numpy(cbg.sin_problem_host(128 ** 3)).cuda())
rot = int(sys.argv[1]) if len(sys.argv) > 1 else 0
_lib.check(_lib.lib().cbgx_debug_fused_rotation(rot))
print("rotation", rot)
runs = []
for its in (20, 21, 22, 20, 21):
    S = cbg.Solver(A, cbg.GmresConfig(storage_format=cbg.StorageFormat.parse("frsz2-32"), max_total_iterations=its))
    S.solve(b)
    t = np.zeros(32 + 3 * 1024, np.uint64)
    _lib.check(_lib.lib().cbgx_debug_fused_trace(t.ctypes.data, t.size))
    st = t[32 + 2048:32 + 3072].astype(np.int64)
    d0 = t[32:32 + 1024].astype(np.int64)
    d1 = t[32 + 1024:32 + 2048].astype(np.int64)
    g = int((st > 0).sum())
    runs.append(((d0[:g] - st[:g]) / 1e3, (d1[:g] - d0[:g]) / 1e3))
    del S
for i in range(1, len(runs)):
    a, b2 = runs[0][0], runs[i][0]
    print(f"run {i}: dot1 corr {np.corrcoef(a, b2)[0,1]:.3f}  upd1 corr {np.corrcoef(runs[0][1], runs[i][1])[0,1]:.3f}")
a = runs[0][0]
print("dot1 per-CTA us: min %.1f med %.1f max %.1f" % (a.min(), np.median(a), a.max()))
order = np.argsort(-a)
print("slowest CTAs", order[:12].tolist(), "fastest", order[-8:].tolist())
G = len(a)
slots = [(int(c) + rot) % G for c in order[:12]]
print("slowest slots (row ranges)", slots)
u = runs[0][1]
ou = np.argsort(-u)
print("upd1 slowest CTAs", ou[:12].tolist(), "slots", [(int(c) + rot) % G for c in ou[:12]])
# by SM pair (c, c+148) and by index parity
G = len(a)
print("mean dot1 by CTA half: first %.2f second %.2f" % (a[:G // 2].mean(), a[G // 2:].mean()))
