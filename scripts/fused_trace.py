"""Timeline of one fused orthogonalisation launch (CTA 0, globaltimer)."""
import os
import sys

os.environ["CBGX_TRACE_FUSED"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, ".")
import paper_2409_15468_b200 as cbg  # noqa: E402
from paper_2409_15468_b200 import _lib  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 128
fmt = sys.argv[2] if len(sys.argv) > 2 else "frsz2-32"
A = cbg.stencil(0, nx)
b = cbg.spmv(A, torch.from_numpy(cbg.sin_problem_host(nx ** 3)).cuda())
names = ["start", "w loaded", "dot1 done", "R0[h]", "upd1 done", "dot2 done", "R1[u,hn1]", "gate",
         "upd2 done", "R2[hn2]", "written"]
for its in (2, 10, 20, 40):
    S = cbg.Solver(A, cbg.GmresConfig(storage_format=cbg.StorageFormat.parse(fmt), max_total_iterations=its))
    for _ in range(3):
        S.solve(b)
    t = np.zeros(32 + 3 * 1024, np.uint64)
    _lib.check(_lib.lib().cbgx_debug_fused_trace(t.ctypes.data, t.size))
    st = t[32 + 2048:32 + 3072].astype(np.int64)
    t0c = 0
    d0 = t[32:32 + 1024].astype(np.int64)
    d1 = t[32 + 1024:32 + 2048].astype(np.int64)
    g = int((st > 0).sum())
    st, d0, d1 = st[:g], d0[:g], d1[:g]
    if g:
        t0c = st.min()
        print(f"  grid {g}: start spread {(st.max()-t0c)/1e3:.1f} us; dot1 end min/med/max "
              f"{(d0.min()-t0c)/1e3:.1f}/{(np.median(d0)-t0c)/1e3:.1f}/{(d0.max()-t0c)/1e3:.1f} us; "
              f"upd1 end min/med/max {(d1.min()-t0c)/1e3:.1f}/{(np.median(d1)-t0c)/1e3:.1f}/{(d1.max()-t0c)/1e3:.1f}")
        order = np.argsort(d0)[-5:]
        print("  slowest dot1 CTAs:", [(int(i), round((d0[i]-st[i])/1e3, 1)) for i in order],
              "fastest:", [(int(i), round((d0[i]-st[i])/1e3, 1)) for i in np.argsort(d0)[:3]])
    t0 = int(t[0])
    parts = []
    prev = t0
    for i, nm in enumerate(names):
        if t[i] and int(t[i]) >= t0:
            parts.append(f"{nm}:{(int(t[i]) - prev) / 1e3:.1f}")
            prev = int(t[i])
    print(f"cols={its}: total {(prev - t0) / 1e3:.1f} us | " + " ".join(parts), flush=True)
    for bi in range(3):
        a_, r_ = int(t[11 + 2 * bi]), int(t[12 + 2 * bi])
        if a_ and r_ >= a_:
            print(f"   barrier {bi}: CTA0 arrive at {(a_ - t0) / 1e3:.1f}, released after {(r_ - a_) / 1e3:.1f} us", flush=True)
    if g:
        print(f"   R0: last CTA dot1 end {(d0.max() - t0) / 1e3:.1f} us after CTA0 start (CTA0 start vs grid min {(t0 - t0c) / 1e3:.1f})")
