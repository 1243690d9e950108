"""The Python multi-GPU path of bench.py --gpus N (paper_2409_15468_b200.dist:
DistStencil / DistSolver over cbgx_halo_create and cbgx_solver_create_dist)
run end to end on ONE GPU: P ranks as P host threads with in-process
communicators (cbgx_comm_create_local_group) instead of NCCL -- the same
halo planning (window layout), device stencil rows, sin right-hand side,
overlapped halo SpMV and rank-ordered collectives. The assembled solution
matches the single-GPU solve of the same problem."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cbg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2409_15468_b200 as m
    return m


@pytest.mark.parametrize("kind,edge,parts,fmt", [(0, 32, 2, "frsz2-32"), (1, 24, 3, "frsz2-32"),
                                                 (2, 24, 4, "f64"), (0, 64, 8, "frsz2-32")])
def test_dist_stencil_solver_on_local_ranks(cbg, kind, edge, parts, fmt):
    import torch
    from paper_2409_15468_b200 import dist
    pe = 1.0 if kind == 1 else 0.0
    group = dist.LocalComms(parts)
    out = [None] * parts
    errs = []

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            prob = dist.DistStencil(group.comms[r], kind, edge, edge, edge, pe)
            b, _ = prob.sin_rhs()
            S = dist.DistSolver(prob, cbg.GmresConfig(restart=40, storage_format=cbg.StorageFormat.parse(fmt)))
            res = S.solve(b)
            torch.cuda.synchronize()
            out[r] = (prob.rb, prob.re, prob.own_off, res.total_iterations, res.converged,
                      res.solution[:prob.re - prob.rb].cpu().numpy().copy(), b.cpu().numpy().copy())
            del S, prob
        except Exception as e:  # noqa: BLE001
            errs.append((r, repr(e)))

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(parts)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    # every rank but the first has a lower ghost plane: window layout
    assert all(o[2] > 0 for o in out[1:])
    n = edge ** 3
    x = np.concatenate([o[5] for o in out])
    b = np.concatenate([o[6] for o in out])
    assert x.size == n and all(o[0] == sum(p[1] - p[0] for p in out[:i]) for i, o in enumerate(out))
    # the same problem on one GPU: b bit-identical, the solve within the contract
    A = cbg.stencil(kind, edge, pe=pe)
    b1 = cbg.spmv(A, torch.from_numpy(cbg.sin_problem_host(n)).cuda())
    assert b1.cpu().numpy().tobytes() == b.tobytes()
    r1 = cbg.Solver(A, cbg.GmresConfig(restart=40, storage_format=cbg.StorageFormat.parse(fmt))).solve(b1)
    its = {o[3] for o in out}
    assert len(its) == 1 and all(o[4] for o in out)   # ranks agree (replicated Givens)
    assert abs(its.pop() - r1.total_iterations) <= max(2, 0.02 * r1.total_iterations)
    x1 = r1.solution.cpu().numpy()
    assert np.allclose(x, x1, rtol=1e-7, atol=1e-9 * np.abs(x1).max())
