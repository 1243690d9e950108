"""One read-benchmark sweep per format at 2^28 values, intensity 1 (ncu target)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2409_15468_b200 as cbg  # noqa: E402

fmts = sys.argv[1].split(",") if len(sys.argv) > 1 else ["frsz2-32"]
n = 1 << 28
data = torch.rand(n, dtype=torch.float64, device="cuda") * 2 - 1
for f in fmts:
    basis = cbg.KrylovBasis(n, 1, cbg.StorageFormat.parse(f))
    basis.write_vector(0, data)
    print(f, cbg.read_sweep(basis, 0, n, 1, 1.0, 0.0))
    torch.cuda.synchronize()
    del basis
