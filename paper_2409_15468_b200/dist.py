"""Row-partitioned multi-GPU CB-GMRES (one process per GPU).

torch.distributed is plumbing only: it carries the 128-byte NCCL unique id
from rank 0 to the other ranks. Every collective on the solve path is issued
by libcbgx itself (cbgx_comm_* / cbgx_halo_* / cbgx_solver_create_dist):
rank-ordered sums of all-gathered partials for the Hessenberg dot products
and norms, grouped ncclSend/ncclRecv for the SpMV halo.

Rows are split into contiguous blocks whose boundaries are multiples of 32
(and, for 3-D grids, of whole z-planes when possible), so every FRSZ2 block is
rank-local and the compressed columns are bit-identical to the single-GPU
ones for identical input vectors.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import DeviceCsr, GmresConfig, _history_buffers, _lib, _ptr, _result, _stream, _torch
from ._lib import check, lib


def row_blocks(n: int, parts: int, plane: int = 0):
    """Contiguous 32-aligned row blocks; whole planes of `plane` rows when
    that keeps the split balanced (z-slabs for a 3-D grid)."""
    if plane and plane % 32 == 0 and (n // plane) >= parts:
        planes = n // plane
        cuts = [plane * ((planes * r) // parts) for r in range(parts + 1)]
    else:
        per = ((n + parts - 1) // parts + 31) // 32 * 32
        cuts = [min(n, per * r) for r in range(parts + 1)]
    return [(cuts[r], cuts[r + 1]) for r in range(parts)]


class NcclComm:
    def __init__(self, rank: int, world: int):
        import torch.distributed as dist
        uid = (ctypes.c_uint8 * 128)()
        if rank == 0:
            check(lib().cbgx_nccl_unique_id(uid))
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0)
        uid = (ctypes.c_uint8 * 128).from_buffer_copy(obj[0])
        h = ctypes.c_void_p()
        check(lib().cbgx_comm_create_nccl(uid, world, rank, ctypes.byref(h)))
        self.h = h
        self.rank, self.world = rank, world

    def __del__(self):
        try:
            lib().cbgx_comm_destroy(self.h)
        except Exception:
            pass


class LocalComms:
    """P in-process communicators (cbgx_comm_create_local_group): rank r is
    driven by its own host thread on the current device -- exercises the
    NCCL path's halo / overlap / collective code on one GPU."""

    class _One:
        def __init__(self, h, rank, world):
            self.h, self.rank, self.world = h, rank, world

        def __del__(self):
            try:
                lib().cbgx_comm_destroy(self.h)
            except Exception:
                pass

    def __init__(self, world: int):
        arr = (ctypes.c_void_p * world)()
        check(lib().cbgx_comm_create_local_group(world, arr))
        self.comms = [LocalComms._One(ctypes.c_void_p(arr[r]), r, world) for r in range(world)]


class DistStencil:
    """This rank's rows of a 3-D stencil (generated on the device), columns
    remapped by a collective halo plan to the window layout [lower ghost
    planes | own rows | upper ghost planes] (column offsets preserved, so the
    dictionary SpMV applies) or, for other partitions, [own rows | ghosts]."""

    def __init__(self, comm: NcclComm, kind: int, nx: int, ny: int, nz: int, pe: float = 0.0):
        torch = _torch()
        self.n = nx * ny * nz
        self.rb, self.re = row_blocks(self.n, comm.world, nx * ny)[comm.rank]
        L = lib()
        nnz = L.cbgx_stencil_nnz(kind, nx, ny, nz, self.rb, self.re)
        rows = self.re - self.rb
        wide = nnz > 0x7FFFFFFF
        rp = torch.empty(rows + 1, dtype=torch.int64 if wide else torch.int32, device="cuda")
        gci = torch.empty(max(nnz, 1), dtype=torch.int32, device="cuda")
        va = torch.empty(max(nnz, 1), dtype=torch.float64, device="cuda")
        check(L.cbgx_stencil_generate(kind, nx, ny, nz, pe, self.rb, self.re, 0, _ptr(rp),
                                      64 if wide else 32, _ptr(gci), _ptr(va), _stream()))
        g64 = gci.to(torch.int64)
        del gci
        lci = torch.empty(max(nnz, 1), dtype=torch.int32, device="cuda")
        torch.cuda.synchronize()
        h = ctypes.c_void_p()
        check(L.cbgx_halo_create(comm.h, self.rb, self.re, self.n, _ptr(g64), nnz, _ptr(lci), ctypes.byref(h)))
        del g64
        self.halo = h
        self.ghosts = L.cbgx_halo_ghosts(h)
        # own rows' position in a local vector (window layout: after the
        # lower ghost rows, cbgx_halo_own_offset)
        self.own_off = L.cbgx_halo_own_offset(h)
        self.A = DeviceCsr(rows, rows + self.ghosts, rp, lci, va)
        self.comm = comm

    def halo_exchange(self, vec):
        check(lib().cbgx_halo_exchange(self.halo, _ptr(vec), _stream()))

    def sin_rhs(self):
        """b = A x_sol for this rank's rows (x_sol from generate_problem)."""
        torch = _torch()
        rows = self.re - self.rb
        xs = np.empty(rows, np.float64)
        check(lib().cbgx_sin_solution(self.n, self.rb, rows, xs.ctypes.data, 0))
        xe = torch.zeros(rows + self.ghosts, dtype=torch.float64, device="cuda")
        o = self.own_off
        xe[o:o + rows] = torch.from_numpy(xs).cuda()
        self.halo_exchange(xe)
        b = torch.empty(max(rows, 1), dtype=torch.float64, device="cuda")
        check(lib().cbgx_csr_spmv(ctypes.byref(self.A.desc), _ptr(xe), _ptr(b), None, 0, None, _stream()))
        return b[:rows], xe[o:o + rows]

    def __del__(self):
        try:
            lib().cbgx_halo_destroy(self.halo)
        except Exception:
            pass


class DistSolver:
    def __init__(self, prob: DistStencil, cfg: GmresConfig = GmresConfig()):
        self.prob = prob
        self.cfg = cfg
        self._c = cfg.c()
        h = ctypes.c_void_p()
        check(lib().cbgx_solver_create_dist(ctypes.byref(prob.A.desc), prob.halo, ctypes.byref(self._c),
                                            prob.comm.h, ctypes.byref(h)))
        self.h = h

    def solve(self, b, x0=None, x=None):
        torch = _torch()
        rows = self.prob.re - self.prob.rb
        if x0 is None:
            if getattr(self, "_zeros", None) is None:
                self._zeros = torch.zeros(rows, dtype=torch.float64, device="cuda")
            x0 = self._zeros
        if x is None:
            x = torch.empty(rows, dtype=torch.float64, device="cuda")
        if getattr(self, "_hbufs", None) is None:
            self._hbufs = _history_buffers(2 * self.cfg.max_total_iterations + 4)
        hist, bufs = self._hbufs
        hist.length = 0
        st = _lib.SolveStats()
        check(lib().cbgx_solver_solve(self.h, _ptr(b), _ptr(x0), _ptr(x), ctypes.byref(hist), ctypes.byref(st),
                                      _stream()))
        return _result(st, hist, bufs, x)

    def phase_times(self):
        ms = np.zeros(8, np.float64)
        check(lib().cbgx_solver_phase_times(self.h, ms.ctypes.data, 8))
        return dict(zip(_lib.PHASES, ms.tolist()))

    def __del__(self):
        try:
            lib().cbgx_solver_destroy(self.h)
        except Exception:
            pass
