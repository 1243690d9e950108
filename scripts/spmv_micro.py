"""SpMV micro-bench: plain CSR kernel vs staged (bulk-copy) kernel vs the dictionary-coded
SELL-32 copy, CUDA events. *_frac: own bytes / time / HBM peak; dict_speedup: staged time / dict time."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2409_15468_b200 as cbg  # noqa: E402

peak = 6546.9
flush = "--flush" in sys.argv  # evict L2 (512 MiB write) before every timed call
scratch = torch.empty(64 << 20, dtype=torch.float64, device="cuda") if flush else None
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
    D = cbg.DictCsr(A)
    no, nv, ne = D.info()
    assert torch.equal(D.spmv(x), ref)
    variants["dict"] = lambda: D.spmv(x, want_norm=True)
    own = {"dict": ne * 2 + ((n + 31) // 32 + 1) * 8 + 16 * n}
    res["dict_entries"] = ne
    for name, fn in variants.items():
        for _ in range(3):
            fn()
        ts = []
        for _ in range(10):
            if flush:
                scratch.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[len(ts) // 2]
        res[name + "_us"] = round(ms * 1e3, 1)
        bb = own.get(name, byt)
        res[name + "_gbs"] = round(bb / ms / 1e6, 1)
        res[name + "_frac"] = round(bb / ms / 1e6 / peak, 3)
    if "staged_us" in res:
        res["dict_speedup"] = round(res["staged_us"] / res["dict_us"], 2)
    res["l2_flushed"] = flush
    print(json.dumps(res), flush=True)
