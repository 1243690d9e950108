"""Per-CTA phase timeline of one fused orthogonalisation launch (globaltimer,
every CTA): where the launch time goes -- column passes vs waiting at the
grid all-reduces -- and how the pass times spread over the CTAs.

    CBGX_NVFLAGS_EXTRA=-DCBGX_FUSED_TRACE=1 python -c "from paper_2409_15468_b200 import build as b; b.build(force=True)"
    python scripts/fused_phases.py [edge] [fmt] [its,...]
(the trace points are compiled out of production builds)
"""
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
its_list = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [2, 10, 20, 40]
NAMES = {0: "start", 1: "w loaded", 2: "dot1", 3: "R0", 4: "upd1", 5: "dot2", 6: "R1", 7: "u out",
         8: "upd2", 9: "R2", 10: "write"}
BASE = 32
A = cbg.stencil(0, nx)
b = cbg.spmv(A, torch.from_numpy(cbg.sin_problem_host(nx ** 3)).cuda())
for its in its_list:
    S = cbg.Solver(A, cbg.GmresConfig(storage_format=cbg.StorageFormat.parse(fmt), max_total_iterations=its))
    for _ in range(3):
        S.solve(b)
    torch.cuda.synchronize()
    t = np.zeros(BASE + 24 * 1024, np.uint64)
    _lib.check(_lib.lib().cbgx_debug_fused_trace(t.ctypes.data, t.size))
    T = t[BASE:].reshape(24, 1024).astype(np.int64)
    g = int((T[0] > 0).sum())
    T = T[:, :g]
    t0 = T[0].min()
    present = [p for p in range(11) if (T[p] > 0).all()]
    print(f"=== {fmt} n={nx}^3 last launch of a {its}-iteration solve (cols={its}), grid {g}")
    print(f"  launch span {(T[present[-1]].max() - t0) / 1e3:.1f} us; start spread {(T[0].max() - t0) / 1e3:.2f} us")
    prev = 0
    tot_wait = 0.0
    for p in present[1:]:
        d = (T[p] - T[prev]) / 1e3
        sync = NAMES[p].startswith("R")
        tag = "SYNC" if sync else "pass"
        print(f"  {NAMES[prev]:>8} -> {NAMES[p]:<8} {tag}: min {d.min():6.1f}  med {np.median(d):6.1f}  "
              f"max {d.max():6.1f} us   (grid-wide end spread {(T[p].max() - T[p].min()) / 1e3:5.1f})")
        if sync:
            tot_wait += float(np.median(d))
        prev = p
    # how consistent are the slow CTAs across passes?
    passes = [(1, 2), (3, 4), (4, 5), (7, 8)]
    dur = [((T[b_] - T[a_]) / 1e3) for a_, b_ in passes if a_ in present and b_ in present]
    if len(dur) >= 2:
        c = np.corrcoef(np.stack(dur))
        print(f"  pass-time correlation across CTAs (dot1/upd1/dot2/upd2): "
              + " ".join(f"{c[0, i]:.2f}" for i in range(1, len(dur))))
        tot = np.sum(np.stack(dur), axis=0)
        print(f"  sum of passes per CTA: min {tot.min():.1f} med {np.median(tot):.1f} max {tot.max():.1f} us; "
              f"slowest CTAs {np.argsort(tot)[-6:].tolist()}, fastest {np.argsort(tot)[:4].tolist()}")
        half = g // 2
        print(f"  first-half vs second-half median pass sum: {np.median(tot[:half]):.1f} / {np.median(tot[half:]):.1f} us")
    print(f"  median time in grid syncs: {tot_wait:.1f} us", flush=True)
