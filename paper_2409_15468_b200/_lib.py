"""ctypes binding of libcbgx.so (include/cbgx.h). Fails loudly if the
extension is missing: there is no CPU fallback anywhere in this package."""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libcbgx.so")

OK, EINVAL, ENONFINITE, ERANGE, EBREAKDOWN, ECUDA, ENOMEM, ECOMM, EINTERNAL = range(9)
F64, F32, F16, FRSZ2 = 0, 1, 2, 3
REDUCE_TREE, REDUCE_REFERENCE = 0, 1
PHASE_TIMING = 1
PHASE_TIMING_DEFERRED = 2
NO_FUSION = 4
NO_SELL = 8
NO_TMA_SPMV = 16
NO_DICT_SPMV = 64
PHASES = ["spmv", "dot", "update", "write", "residual", "solution", "comm", "ortho"]

u32, u64, i32, i64, dbl, vp = C.c_uint32, C.c_uint64, C.c_int32, C.c_int64, C.c_double, C.c_void_p


class Basis(C.Structure):
    _fields_ = [("kind", u32), ("bit_length", u32), ("n", u64), ("n_pad", u64),
                ("capacity", u64), ("d_data", vp), ("d_exp", vp),
                ("col_stride_bytes", u64), ("exp_col_stride", u64), ("d_erange", vp)]


class Csr(C.Structure):
    _fields_ = [("n_rows", u64), ("n_cols", u64), ("nnz", u64), ("d_row_ptr", vp),
                ("row_ptr_bits", u32), ("d_col_idx", vp), ("d_values", vp), ("max_row_nnz", u32)]


class GmresConfig(C.Structure):
    _fields_ = [("restart", u64), ("target_rrn", dbl), ("max_total_iterations", u64),
                ("eta", dbl), ("format_kind", u32), ("bit_length", u32),
                ("reduction", u32), ("flags", u32)]


class History(C.Structure):
    _fields_ = [("iteration", vp), ("rrn", vp), ("is_explicit", vp),
                ("capacity", u64), ("length", u64)]


class SolveStats(C.Structure):
    _fields_ = [("converged", C.c_int), ("total_iterations", u64), ("restarts", u64),
                ("final_rrn", dbl), ("wall_seconds", dbl), ("reorth_passes", u64),
                ("phase_ms", dbl * 8), ("phase_bytes", dbl * 8), ("phase_launches", u64 * 8),
                ("kernel_launches", u64), ("host_enqueue_ms", dbl), ("host_wait_ms", dbl)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run python -c 'import __graft_entry__ as g; g.build()'")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        sigs = {
            "cbgx_last_error": ([], C.c_char_p),
            "cbgx_last_error_index": ([], u64),
            "cbgx_version": ([], C.c_int),
            "cbgx_launch_count": ([], u64),
            "cbgx_set_device": ([C.c_int], C.c_int),
            "cbgx_sin_solution": ([u64, u64, u64, vp, C.c_int], C.c_int),
            "cbgx_halo_exchange": ([vp, vp, vp], C.c_int),
            "cbgx_debug_fused_trace": ([vp, C.c_int], C.c_int),
            "cbgx_debug_fused_rotation": ([u32], C.c_int),
            "cbgx_device_info": ([P(C.c_int), P(C.c_int), P(i64)], C.c_int),
            "cbgx_frsz2_num_blocks": ([u64, u32], u64),
            "cbgx_frsz2_words_per_block": ([u32, u32], u64),
            "cbgx_frsz2_storage_bytes": ([u64, u32, u32], u64),
            "cbgx_frsz2_max_abs_error_bound": ([u32, u32], dbl),
            "cbgx_frsz2_compress": ([vp, u64, u32, u32, vp, vp, vp], C.c_int),
            "cbgx_frsz2_compress_async": ([vp, u64, u32, u32, vp, vp, vp, vp], C.c_int),
            "cbgx_frsz2_decompress": ([vp, vp, u64, u32, u32, vp, vp], C.c_int),
            "cbgx_frsz2_decompress_range": ([vp, vp, u64, u32, u32, u64, u64, vp, vp], C.c_int),
            "cbgx_frsz2_encode_block": ([vp, u32, u32, vp, vp, vp], C.c_int),
            "cbgx_basis_layout": ([u32, u32, u64, u64, P(Basis), P(u64), P(u64)], C.c_int),
            "cbgx_workspace_create": ([P(vp)], C.c_int),
            "cbgx_workspace_destroy": ([vp], C.c_int),
            "cbgx_basis_write": ([P(Basis), u64, vp, vp, C.c_int, vp, vp, vp], C.c_int),
            "cbgx_basis_read": ([P(Basis), u64, u64, u64, vp, vp], C.c_int),
            "cbgx_cgs_dot": ([P(Basis), u64, u32, vp, C.c_int, C.c_int, vp, vp, vp], C.c_int),
            "cbgx_cgs_update": ([P(Basis), u64, u32, vp, C.c_int, vp, vp, C.c_int, vp, vp], C.c_int),
            "cbgx_arnoldi_fused_step": ([P(Basis), u32, u32, vp, vp, vp, dbl, C.c_int, vp, vp], C.c_int),
            "cbgx_csr_spmv": ([P(Csr), vp, vp, vp, C.c_int, vp, vp], C.c_int),
            "cbgx_csr_residual": ([P(Csr), vp, vp, vp, vp, C.c_int, vp, vp], C.c_int),
            "cbgx_csr_spmv_plan": ([P(Csr), P(C.c_uint32), vp], C.c_int),
            "cbgx_csr_spmv_staged": ([P(Csr), C.c_uint32, vp, vp, vp, vp, C.c_int, vp, vp], C.c_int),
            "cbgx_csr_dict_create": ([P(Csr), P(vp), vp], C.c_int),
            "cbgx_csr_dict_info": ([vp, P(C.c_uint32), P(C.c_uint32), P(C.c_uint64)], C.c_int),
            "cbgx_csr_dict_create2": ([P(Csr), C.c_uint32, P(vp), vp], C.c_int),
            "cbgx_csr_dict_layout": ([vp, P(C.c_uint32), P(C.c_uint32), P(C.c_uint32)], C.c_int),
            "cbgx_csr_dict_spmv": ([P(Csr), vp, vp, vp, vp, vp, C.c_int, vp, vp], C.c_int),
            "cbgx_csr_dict_destroy": ([vp], None),
            "cbgx_dot": ([vp, vp, u64, C.c_int, vp, vp, vp], C.c_int),
            "cbgx_scale": ([dbl, vp, u64, vp], C.c_int),
            "cbgx_axpy": ([dbl, vp, vp, u64, vp], C.c_int),
            "cbgx_stencil_nnz": ([C.c_int, u64, u64, u64, u64, u64], u64),
            "cbgx_stencil_generate": ([C.c_int, u64, u64, u64, dbl, u64, u64, i64, vp, u32, vp, vp, vp], C.c_int),
            "cbgx_solver_create": ([P(Csr), P(GmresConfig), vp, P(vp)], C.c_int),
            "cbgx_solver_destroy": ([vp], C.c_int),
            "cbgx_solver_phase_times": ([vp, vp, u64], C.c_int),
            "cbgx_solver_solve": ([vp, vp, vp, vp, P(History), P(SolveStats), vp], C.c_int),
            "cbgx_host_cache_release": ([], C.c_int),
            "cbgx_read_sweep": ([P(Basis), u64, u64, C.c_int, C.c_double, C.c_double, vp, vp, vp], C.c_int),
            "cbgx_read_sweep_timed": ([P(Basis), u64, u64, C.c_int, C.c_double, C.c_double, C.c_int, P(C.c_double),
                                       P(C.c_double)], C.c_int),
            "cbgx_gmres_solve_host": ([u64, vp, vp, vp, vp, vp, P(GmresConfig), vp, P(History), P(SolveStats)], C.c_int),
            "cbgx_nccl_unique_id": ([vp], C.c_int),
            "cbgx_comm_create_nccl": ([vp, C.c_int, C.c_int, P(vp)], C.c_int),
            "cbgx_comm_create_local_group": ([C.c_int, vp], C.c_int),
            "cbgx_comm_destroy": ([vp], C.c_int),
            "cbgx_comm_rank": ([vp, P(C.c_int), P(C.c_int)], C.c_int),
            "cbgx_halo_create": ([vp, u64, u64, u64, vp, u64, vp, P(vp)], C.c_int),
            "cbgx_halo_destroy": ([vp], C.c_int),
            "cbgx_halo_ghosts": ([vp], u64),
            "cbgx_halo_own_offset": ([vp], u64),
            "cbgx_halo_plan": ([C.c_int, C.c_int, vp, u64, vp, u64, vp, vp, P(u64), vp, P(u64)], C.c_int),
            "cbgx_halo_send_index": ([u64, u64, vp, u64, vp], C.c_int),
            "cbgx_sum_ranks_host": ([C.c_int, u64, vp, vp], C.c_int),
            "cbgx_malloc": ([P(vp), u64], C.c_int),
            "cbgx_free": ([vp], C.c_int),
            "cbgx_memcpy": ([vp, vp, u64, C.c_int], C.c_int),
            "cbgx_memset": ([vp, C.c_int, u64], C.c_int),
            "cbgx_solver_create_dist": ([P(Csr), vp, P(GmresConfig), vp, P(vp)], C.c_int),
            "cbgx_gmres_solve_partitioned_local": ([u64, vp, vp, vp, vp, vp, P(GmresConfig), C.c_int, vp,
                                                    P(History), P(SolveStats)], C.c_int),
        }
        for name, (args, res) in sigs.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        L.cbgx_signatures = frozenset(sigs)
        _lib = L
    return _lib


class CbgxError(RuntimeError):
    def __init__(self, status, msg, index):
        super().__init__(msg)
        self.status = status
        self.index = index


def check(status: int) -> None:
    """Map a C-ABI status onto the reference's exception types."""
    if status == OK:
        return
    L = lib()
    msg = L.cbgx_last_error().decode()
    idx = L.cbgx_last_error_index()
    if status in (EINVAL, ENONFINITE):
        e = ValueError(msg)            # std::invalid_argument
    elif status == ERANGE:
        e = IndexError(msg)            # std::out_of_range
    elif status == EBREAKDOWN:
        from . import SolverBreakdown
        e = SolverBreakdown(msg, idx)
    else:
        e = CbgxError(status, msg, idx)
    e.index = idx
    raise e
