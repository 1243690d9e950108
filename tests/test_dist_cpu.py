"""Row-partitioned (multi-GPU) host logic on CPU: two real processes over a
gloo process group run the production halo-planning code of libcbgx
(cbgx_halo_plan / cbgx_halo_send_index / cbgx_sum_ranks_host, the same
functions cbgx_halo_create calls between its NCCL collectives), exchange
requests and ghost values through gloo, and check

* the distributed SpMV on [own rows | ghosts] with remapped columns is
  bit-identical to the global SpMV rows (per-row order preserved);
* every ghost value is the owner's value of that global row;
* the rank-ordered combine of per-rank partial sums is identical on every
  rank (the determinism contract of the NCCL reduction).
"""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, kind, dims, out_q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import pyoracle as po
        from paper_2409_15468_b200 import _lib
        from paper_2409_15468_b200.dist import row_blocks
        L = _lib.lib()
        P = po.Port()
        nx, ny, nz = dims
        rp, ci, va = P.stencil(kind, nx, ny, nz, pe=1.0)
        n = rp.size - 1
        blocks = row_blocks(n, world, nx * ny)
        assert all(b % 32 == 0 for b, _ in blocks), blocks
        rb, re_ = blocks[rank]
        ranges = np.array([x for b in blocks for x in b], np.uint64)
        k0, k1 = int(rp[rb]), int(rp[re_])
        gcols = ci[k0:k1].astype(np.int64)
        nnz = k1 - k0
        lcols = np.zeros(max(nnz, 1), np.int32)
        ghosts = np.zeros(max(nnz, 1), np.int64)
        ng = ctypes.c_uint64()
        need = np.zeros(world, np.uint64)
        own = ctypes.c_uint64()
        _lib.check(L.cbgx_halo_plan(world, rank, ranges.ctypes.data, n, gcols.ctypes.data, nnz,
                                    lcols.ctypes.data, ghosts.ctypes.data, ctypes.byref(ng), need.ctypes.data,
                                    ctypes.byref(own)))
        ghosts = ghosts[:ng.value]
        # requests grouped by owner (ghosts are sorted by global index)
        owner = np.searchsorted(ranges[0::2].astype(np.int64), ghosts, side="right") - 1
        reqs = {o: ghosts[owner == o] for o in range(world) if o != rank}
        assert all(len(reqs[o]) == int(need[o]) for o in reqs)
        all_reqs = [None] * world
        dist.all_gather_object(all_reqs, reqs)
        # owner side: rows every peer asked me for
        x = np.random.default_rng(123).standard_normal(n)       # same x on every rank
        x_local = x[rb:re_]
        sends = {}
        for r in range(world):
            if r == rank:
                continue
            ask = np.ascontiguousarray(all_reqs[r].get(rank, np.zeros(0, np.int64)), np.int64)
            idx = np.zeros(max(ask.size, 1), np.int32)
            if ask.size:
                _lib.check(L.cbgx_halo_send_index(rb, re_, ask.ctypes.data, ask.size, idx.ctypes.data))
            sends[r] = x_local[idx[:ask.size]]
        all_sends = [None] * world
        dist.all_gather_object(all_sends, sends)
        ghost_vals = np.concatenate([all_sends[o][rank] for o in range(world) if o != rank and o in reqs
                                     and len(reqs[o])] or [np.zeros(0)])
        assert np.array_equal(ghost_vals, x[ghosts])
        o = own.value
        if o:
            # window layout: the local vector is the global rows [rb - o, re + ...),
            # so every column offset survives the remap (shifted by o)
            x_ext = np.concatenate([ghost_vals[:o], x_local, ghost_vals[o:]])
            assert np.array_equal(x_ext, x[rb - o:rb - o + x_ext.size])
            lr = np.repeat(np.arange(re_ - rb), np.diff(rp[rb:re_ + 1]).astype(np.int64))
            assert np.array_equal(lcols[:nnz].astype(np.int64) - lr - o, gcols - (lr + rb))
        else:
            x_ext = np.concatenate([x_local, ghost_vals])
        # local SpMV with the oracle's row-sequential kernel on remapped columns
        lrp = (rp[rb:re_ + 1] - rp[rb]).astype(np.uint64)
        y_local = P.spmv(lrp, lcols[:nnz].astype(np.uint64), np.ascontiguousarray(va[k0:k1]), x_ext)
        y_global = P.spmv(rp, ci, va, x)
        assert y_local.tobytes() == y_global[rb:re_].tobytes()
        # rank-ordered combine of partial dot products
        part = np.array([P.dot(y_local, y_local), P.dot(x_local, y_local)])
        parts = [None] * world
        dist.all_gather_object(parts, part)
        g = np.ascontiguousarray(np.concatenate(parts))
        out = np.zeros(2)
        _lib.check(L.cbgx_sum_ranks_host(world, 2, g.ctypes.data, out.ctypes.data))
        combined = [None] * world
        dist.all_gather_object(combined, out.tobytes())
        assert len(set(combined)) == 1
        ref = P.dot(y_global, y_global)
        assert abs(out[0] - ref) <= 1e-12 * abs(ref)
        out_q.put((rank, "ok", int(ng.value), int(o)))
    except Exception as e:  # noqa: BLE001
        out_q.put((rank, repr(e), 0, 0))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,dims,world", [(1, (8, 8, 6), 2), (2, (8, 4, 10), 2), (0, (16, 8, 6), 3)])
def test_partitioned_halo_and_reduction(kind, dims, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, dims, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    res = [q.get(timeout=10) for _ in range(world)]
    assert all(r[1] == "ok" for r in res), res
    assert all(p.exitcode == 0 for p in procs)
    assert sum(r[2] for r in res) > 0   # some ghosts actually crossed ranks
    # z-slab partitions of 3-D stencils take the window layout on every rank
    # that has a lower neighbour
    assert all(r[3] > 0 for r in res if r[0] > 0), res


def test_row_blocks():
    from paper_2409_15468_b200.dist import row_blocks
    assert row_blocks(512 ** 3, 8, 512 * 512) == [(r * 64 * 512 * 512, (r + 1) * 64 * 512 * 512) for r in range(8)]
    b = row_blocks(1000, 3)
    assert b[0][0] == 0 and b[-1][1] == 1000 and all(x % 32 == 0 for x, _ in b)
    assert all(b[i][1] == b[i + 1][0] for i in range(2))
