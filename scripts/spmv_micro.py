"""SpMV micro-bench: plain CSR kernel vs staged (bulk-copy) kernel, CUDA events."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2409_15468_b200 as cbg  # noqa: E402

peak = 6546.9
for kind, nx in ((0, 128), (2, 128), (1, 192), (0, 256)):
    A = cbg.stencil(kind, nx, pe=1.0 if kind == 1 else 0.0)
    n = nx ** 3
    nnz = A.desc.nnz
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    byt = nnz * 12 + (n + 1) * 4 + 16 * n
    t = cbg.spmv_plan(A)
    res = {"kind": kind, "nx": nx, "nnz": nnz, "tile": t}
    ref = cbg.spmv(A, x)
    variants = {"csr": lambda: cbg.spmv(A, x, want_norm=True)}
    if t:
        assert torch.equal(cbg.spmv_staged(A, x, t), ref)
        variants["staged"] = lambda: cbg.spmv_staged(A, x, t, want_norm=True)
    for name, fn in variants.items():
        for _ in range(3):
            fn()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[len(ts) // 2]
        res[name + "_us"] = round(ms * 1e3, 1)
        res[name + "_gbs"] = round(byt / ms / 1e6, 1)
        res[name + "_frac"] = round(byt / ms / 1e6 / peak, 3)
    print(json.dumps(res), flush=True)
