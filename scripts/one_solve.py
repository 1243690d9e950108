"""Exactly one CB-GMRES(100) solve of a BASELINE workload after one untimed
warm-up solve (ncu target: the launch list of a solve, cold-cache)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2409_15468_b200 as cbg  # noqa: E402

kind, nx = {"poisson128": (0, 128), "convdiff192": (1, 192), "p27-128": (2, 128)}[sys.argv[1] if len(sys.argv) > 1 else "poisson128"]
fmt = sys.argv[2] if len(sys.argv) > 2 else "frsz2-32"
A = cbg.stencil(kind, nx, pe=1.0 if kind == 1 else 0.0)
b = cbg.spmv(A, torch.from_numpy(cbg.sin_problem_host(nx ** 3)).cuda())
S = cbg.Solver(A, cbg.GmresConfig(storage_format=cbg.StorageFormat.parse(fmt)))
S.solve(b)
torch.cuda.synchronize()
r = S.solve(b)
torch.cuda.synchronize()
print("its", r.total_iterations, "rrn", r.final_rrn)
