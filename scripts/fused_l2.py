"""One solve with max_total_iterations=K (ncu target: the fused launches)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2409_15468_b200 as cbg  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 128
its = int(sys.argv[2]) if len(sys.argv) > 2 else 12
A = cbg.stencil(0, nx)
b = cbg.spmv(A, torch.from_numpy(cbg.sin_problem_host(nx ** 3)).cuda())
S = cbg.Solver(A, cbg.GmresConfig(storage_format=cbg.StorageFormat.parse(sys.argv[3] if len(sys.argv) > 3 else "frsz2-32"),
                                  max_total_iterations=its))
r = S.solve(b)
torch.cuda.synchronize()
print("its", r.total_iterations)
