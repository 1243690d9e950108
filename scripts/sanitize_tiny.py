"""Tiny fused-kernel + staged-SpMV + codec run for racecheck/synccheck."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2409_15468_b200 as cbg  # noqa: E402

v = np.random.default_rng(0).standard_normal(3000)
for l in (16, 21, 32):
    cbg.decompress(cbg.compress(v, cbg.Frsz2Params(32, l)))
A = cbg.stencil(0, 12)
n = 12 ** 3
b = cbg.spmv(A, torch.from_numpy(cbg.sin_problem_host(n)).cuda())
cbg.spmv_staged(A, b, cbg.spmv_plan(A), want_norm=True)
S = cbg.Solver(A, cbg.GmresConfig(restart=8, storage_format=cbg.StorageFormat.parse(sys.argv[1] if len(sys.argv) > 1 else "frsz2-21"),
                                  max_total_iterations=10))
print(S.solve(b).total_iterations, flush=True)
torch.cuda.synchronize()
print("tiny done")
