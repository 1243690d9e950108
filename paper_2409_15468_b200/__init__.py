"""B200-native FRSZ2-compressed-basis GMRES (arXiv 2409.15468).

Python mirror of the reference's public interface (proj/include/cbg:
frsz2.hpp, basis.hpp, sparse.hpp, gmres.hpp) over the C-ABI in
include/cbgx.h (libcbgx.so, sm_100a). Same names, argument meaning and
error behaviour as the reference: ValueError for std::invalid_argument
(including "frsz2: non-finite value at index N"), IndexError for
std::out_of_range, SolverBreakdown for cbg::SolverBreakdown.

Device buffers are torch CUDA tensors (torch is plumbing only: allocation,
streams, events). Every compute call goes to the CUDA extension; if it is
missing the import of the binding raises -- there is no CPU fallback.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check, lib

__all__ = [
    "Frsz2Params", "CompressedVector", "compress", "compress_block", "decompress",
    "decompress_block", "decompress_value", "storage_bytes", "max_abs_error_bound",
    "StorageFormat", "KrylovBasis", "Workspace", "CsrMatrix", "DeviceCsr", "spmv", "dot",
    "norm2", "GmresConfig", "ResidualRecord", "SolveResult", "SolverBreakdown", "gmres_solve",
    "Solver", "stencil", "sin_problem_host",
]


def _torch():
    import torch
    return torch


def _dev(x, dtype=None):
    """Return a contiguous CUDA tensor view/copy of x (numpy, list or tensor)."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        t = x if x.is_cuda else x.cuda()
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).cuda()
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    return t.contiguous()


def _ptr(t):
    return C_void(t.data_ptr()) if t is not None else None


def C_void(p):
    import ctypes
    return ctypes.c_void_p(p)


def _stream():
    torch = _torch()
    return C_void(torch.cuda.current_stream().cuda_stream)


class SolverBreakdown(RuntimeError):
    """cbg::SolverBreakdown (gmres.hpp:48-53)."""

    def __init__(self, what, iteration):
        super().__init__(what)
        self.iteration = iteration


# ------------------------------------------------------------------ codec
@dataclasses.dataclass(frozen=True)
class Frsz2Params:
    """frsz2.hpp:16-22."""
    block_size: int = 32
    bit_length: int = 32

    def validate(self):
        if self.block_size < 1:
            raise ValueError("frsz2: block_size must be >= 1")
        if self.bit_length < 2 or self.bit_length > 64:
            raise ValueError("frsz2: bit_length must be in [2, 64]")

    def words_per_block(self):
        return (self.block_size * self.bit_length + 31) // 32


class CompressedVector:
    """frsz2.hpp:29-48, device resident: `exps` and `payload` are uint32
    CUDA tensors in exactly the reference layout (separate exponent and
    LSB-first payload arrays)."""

    def __init__(self, params: Frsz2Params, n: int, exps=None, payload=None):
        params.validate()
        torch = _torch()
        self.params = params
        self.n = n
        nb = self.num_blocks()
        self.exps = exps if exps is not None else torch.zeros(max(nb, 1), dtype=torch.int32, device="cuda")
        self.payload = payload if payload is not None else torch.zeros(
            max(nb * params.words_per_block(), 1), dtype=torch.int32, device="cuda")

    def size(self):
        return self.n

    def num_blocks(self):
        return (self.n + self.params.block_size - 1) // self.params.block_size

    def exponents(self) -> np.ndarray:
        return self.exps[:self.num_blocks()].cpu().numpy().view(np.uint32)

    def payload_words(self) -> np.ndarray:
        return self.payload[:self.num_blocks() * self.params.words_per_block()].cpu().numpy().view(np.uint32)

    def container_bytes(self) -> bytes:
        """write_frsz2_file (frsz2.cpp:297-311): "FRSZ2\\0", u16 1, u32 bs,
        u32 l, u64 n, exponents, payload (little endian)."""
        import struct
        hdr = b"FRSZ2\x00" + struct.pack("<HIIQ", 1, self.params.block_size, self.params.bit_length, self.n)
        return hdr + self.exponents().astype("<u4").tobytes() + self.payload_words().astype("<u4").tobytes()

    @staticmethod
    def from_container(data: bytes) -> "CompressedVector":
        """read_frsz2_file (frsz2.cpp:313-343) with the same error texts."""
        import struct
        torch = _torch()
        if len(data) < 6 or data[:6] != b"FRSZ2\x00":
            raise RuntimeError("frsz2 container: bad magic")
        if len(data) < 8:
            raise RuntimeError("frsz2 container: truncated file")
        (ver,) = struct.unpack_from("<H", data, 6)
        if ver != 1:
            raise RuntimeError(f"frsz2 container: unsupported version {ver}")
        if len(data) < 24:
            raise RuntimeError("frsz2 container: truncated file")
        bs, l, n = struct.unpack_from("<IIQ", data, 8)
        try:
            Frsz2Params(bs, l).validate()
        except ValueError as e:
            raise RuntimeError(f"frsz2 container: {e}") from None
        p = Frsz2Params(bs, l)
        nb = (n + bs - 1) // bs
        need = 24 + 4 * nb + 4 * nb * p.words_per_block()
        if len(data) < need:
            raise RuntimeError("frsz2 container: truncated file")
        if len(data) > need:
            raise RuntimeError("frsz2 container: trailing data")
        e = np.frombuffer(data, "<u4", nb, 24).astype(np.uint32)
        w = np.frombuffer(data, "<u4", nb * p.words_per_block(), 24 + 4 * nb).astype(np.uint32)
        ex = torch.from_numpy(np.concatenate([e, np.zeros(1, np.uint32)]).view(np.int32)).cuda()
        pw = torch.from_numpy(np.concatenate([w, np.zeros(1, np.uint32)]).view(np.int32)).cuda()
        return CompressedVector(p, n, ex, pw)


def storage_bytes(n: int, params: Frsz2Params = Frsz2Params()) -> int:
    params.validate()
    return lib().cbgx_frsz2_storage_bytes(n, params.block_size, params.bit_length)


def max_abs_error_bound(e_max_biased: int, bit_length: int) -> float:
    return lib().cbgx_frsz2_max_abs_error_bound(e_max_biased, bit_length)


def compress(values, params: Frsz2Params = Frsz2Params()) -> CompressedVector:
    """frsz2.hpp:70-71 on the GPU (warp-per-block codec for bs=32,
    l in {16,21,32}; generic codec otherwise). Raises ValueError
    "frsz2: non-finite value at index N" like the reference."""
    params.validate()
    x = _dev(values)
    n = x.numel()
    cv = CompressedVector(params, n)
    if n:
        check(lib().cbgx_frsz2_compress(_ptr(x), n, params.block_size, params.bit_length,
                                        _ptr(cv.exps), _ptr(cv.payload), _stream()))
    return cv


def compress_block(values, bit_length: int):
    """frsz2.hpp:64-65 -> (e_max, codes as uint64 numpy)."""
    torch = _torch()
    x = _dev(values)
    Frsz2Params(max(x.numel(), 0), bit_length).validate()
    em = torch.zeros(1, dtype=torch.int32, device="cuda")
    codes = torch.zeros(max(x.numel(), 1), dtype=torch.int64, device="cuda")
    check(lib().cbgx_frsz2_encode_block(_ptr(x), x.numel(), bit_length, _ptr(em), _ptr(codes), _stream()))
    return int(em.cpu().numpy().view(np.uint32)[0]), codes[:x.numel()].cpu().numpy().view(np.uint64)


def decompress(cv: CompressedVector, out=None):
    """frsz2.hpp:79-80 -> CUDA float64 tensor."""
    torch = _torch()
    if out is None:
        out = torch.empty(max(cv.n, 1), dtype=torch.float64, device="cuda")
    elif out.numel() != cv.n:
        raise ValueError("frsz2: output length mismatch")
    if cv.n:
        check(lib().cbgx_frsz2_decompress(_ptr(cv.exps), _ptr(cv.payload), cv.n, cv.params.block_size,
                                          cv.params.bit_length, _ptr(out), _stream()))
    return out[:cv.n]


def decompress_block(cv: CompressedVector, block: int):
    torch = _torch()
    if block < 0 or block >= cv.num_blocks():
        raise IndexError("frsz2: block index out of range")
    bs = cv.params.block_size
    out = torch.empty(bs, dtype=torch.float64, device="cuda")
    check(lib().cbgx_frsz2_decompress_range(_ptr(cv.exps), _ptr(cv.payload), cv.n, bs, cv.params.bit_length,
                                            block * bs, bs, _ptr(out), _stream()))
    return out


def decompress_value(cv: CompressedVector, i: int) -> float:
    torch = _torch()
    if i < 0 or i >= cv.n:
        raise IndexError("frsz2: index out of range")
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    check(lib().cbgx_frsz2_decompress_range(_ptr(cv.exps), _ptr(cv.payload), cv.n, cv.params.block_size,
                                            cv.params.bit_length, i, 1, _ptr(out), _stream()))
    return float(out.item())


# ------------------------------------------------------------ workspace
class Workspace:
    def __init__(self):
        import ctypes
        h = ctypes.c_void_p()
        check(lib().cbgx_workspace_create(ctypes.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if self.h:
                lib().cbgx_workspace_destroy(self.h)
        except Exception:
            pass


_default_ws = None


def _ws():
    global _default_ws
    if _default_ws is None:
        _default_ws = Workspace()
    return _default_ws.h


# ------------------------------------------------------------ basis
@dataclasses.dataclass(frozen=True)
class StorageFormat:
    """basis.hpp:23-38."""
    kind: int = _lib.F64
    bit_length: int = 0

    @staticmethod
    def f64():
        return StorageFormat(_lib.F64, 0)

    @staticmethod
    def f32():
        return StorageFormat(_lib.F32, 0)

    @staticmethod
    def f16():
        return StorageFormat(_lib.F16, 0)

    @staticmethod
    def frsz2_format(bit_length: int):
        if bit_length not in (16, 21, 32):
            raise ValueError("storage format: frsz2 bit length must be 16, 21 or 32")
        return StorageFormat(_lib.FRSZ2, bit_length)

    @staticmethod
    def parse(name: str) -> Optional["StorageFormat"]:
        table = {"f64": StorageFormat.f64(), "f32": StorageFormat.f32(), "f16": StorageFormat.f16(),
                 "frsz2-16": StorageFormat(_lib.FRSZ2, 16), "frsz2-21": StorageFormat(_lib.FRSZ2, 21),
                 "frsz2-32": StorageFormat(_lib.FRSZ2, 32)}
        return table.get(name)

    def name(self) -> str:
        return {_lib.F64: "f64", _lib.F32: "f32", _lib.F16: "f16"}.get(self.kind, f"frsz2-{self.bit_length}")

    def column_bytes(self, n: int) -> int:
        if self.kind == _lib.F64:
            return 8 * n
        if self.kind == _lib.F32:
            return 4 * n
        if self.kind == _lib.F16:
            return 2 * n
        return storage_bytes(n, Frsz2Params(32, self.bit_length))


class KrylovBasis:
    """basis.hpp:43-83 on the device: a padded column-major panel."""
    kBlock = 32

    def __init__(self, length: int, capacity: int, fmt: StorageFormat = StorageFormat.f64()):
        import ctypes
        torch = _torch()
        self.fmt = fmt
        self.desc = _lib.Basis()
        db, eb = ctypes.c_uint64(), ctypes.c_uint64()
        check(lib().cbgx_basis_layout(fmt.kind, fmt.bit_length, length, capacity, ctypes.byref(self.desc),
                                      ctypes.byref(db), ctypes.byref(eb)))
        self._data = torch.zeros((db.value + 7) // 8, dtype=torch.float64, device="cuda")
        self._exp = torch.zeros(max((eb.value + 3) // 4, 1), dtype=torch.int32, device="cuda")
        self.desc.d_data = self._data.data_ptr()
        self.desc.d_exp = self._exp.data_ptr() if eb.value else None
        # per-column exponent range (cbgx_basis.d_erange): lets the CGS
        # kernels take the fast decode per column
        self._erange = torch.zeros(max(2 * capacity, 1), dtype=torch.int32, device="cuda")
        self.desc.d_erange = self._erange.data_ptr() if eb.value else None
        self.n = length
        self.capacity_ = capacity
        self.count_ = 0

    def length(self):
        return self.n

    def capacity(self):
        return self.capacity_

    def count(self):
        return self.count_

    def num_blocks(self):
        return (self.n + 31) // 32

    def write_vector(self, j: int, values, scale=None, scale_mode=0, v_out=None):
        """basis.cpp:85-115 (+ optional fused scale, see cbgx_basis_write)."""
        import ctypes
        torch = _torch()
        if j > self.count_ or j >= self.capacity_:
            raise IndexError("basis: cannot write column")
        x = _dev(values)
        if x.numel() != self.n:
            raise ValueError("basis: length mismatch")
        bad = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        check(lib().cbgx_basis_write(ctypes.byref(self.desc), j, _ptr(x), _ptr(scale), scale_mode,
                                     _ptr(v_out), _ptr(bad), _stream()))
        b = int(bad.item())
        if b != -1:
            raise ValueError(f"frsz2: non-finite value at index {b}")
        self.count_ = max(self.count_, j + 1)

    def _check(self, j):
        if j >= self.count_:
            raise IndexError("basis: column index out of range")

    def read_block(self, j: int, blk: int):
        import ctypes
        torch = _torch()
        self._check(j)
        if blk >= self.num_blocks():
            raise IndexError("basis: block index out of range")
        out = torch.empty(32, dtype=torch.float64, device="cuda")
        check(lib().cbgx_basis_read(ctypes.byref(self.desc), j, blk * 32, 32, _ptr(out), _stream()))
        return out

    def read_column(self, j: int):
        import ctypes
        torch = _torch()
        self._check(j)
        out = torch.empty(max(self.n, 1), dtype=torch.float64, device="cuda")
        check(lib().cbgx_basis_read(ctypes.byref(self.desc), j, 0, self.n, _ptr(out), _stream()))
        return out[:self.n]

    def read_element(self, j: int, i: int) -> float:
        import ctypes
        torch = _torch()
        self._check(j)
        if i >= self.n:
            raise IndexError("basis: element index out of range")
        out = torch.empty(1, dtype=torch.float64, device="cuda")
        check(lib().cbgx_basis_read(ctypes.byref(self.desc), j, i, 1, _ptr(out), _stream()))
        return float(out.item())

    def cgs_dot(self, cols: int, w, first: int = 0, with_wnorm=False, reduction=_lib.REDUCE_TREE, out=None):
        """h[i] = <V_{first+i}, w> for i < cols (+ <w,w>): one fused pass."""
        import ctypes
        torch = _torch()
        if first + cols > self.count_:
            raise IndexError("basis: column index out of range")
        w = _dev(w)
        if w.numel() != self.n:
            raise ValueError("basis: length mismatch")
        if out is None:
            out = torch.empty(cols + 1, dtype=torch.float64, device="cuda")
        check(lib().cbgx_cgs_dot(ctypes.byref(self.desc), first, cols, _ptr(w), int(with_wnorm), reduction,
                                 _ptr(out), _ws(), _stream()))
        return out[:cols + (1 if with_wnorm else 0)]

    def cgs_update(self, cols: int, h, w, first: int = 0, sign=1, want_norm=False,
                   reduction=_lib.REDUCE_TREE, norm_out=None):
        """w -= sum_i h[i] V_{first+i} in place (bit-identical to
        subtract_scaled in column order); returns <w,w> tensor if asked."""
        import ctypes
        torch = _torch()
        if first + cols > self.count_:
            raise IndexError("basis: column index out of range")
        h = _dev(h)
        if want_norm and norm_out is None:
            norm_out = torch.empty(1, dtype=torch.float64, device="cuda")
        check(lib().cbgx_cgs_update(ctypes.byref(self.desc), first, cols, _ptr(h), sign, _ptr(w),
                                    _ptr(norm_out) if want_norm else None, reduction, _ws(), _stream()))
        return norm_out

    def arnoldi_fused_step(self, cols: int, w, omega2, max_cols: int, eta=0.70710678118654752,
                           speculate=True):
        """One fused Arnoldi step (cbgx_arnoldi_fused_step: gmres.cpp:36-71
        + the scaled write of column `cols`, :230-234). Returns (slot, v):
        slot = [hn1, hn2, omega2, h[0..max_cols], u[0..max_cols]] (CUDA
        float64), v = the written column's fp64 values."""
        import ctypes
        torch = _torch()
        if cols > self.count_ or cols + 1 > self.capacity_:
            raise IndexError("basis: column index out of range")
        w = _dev(w)
        if w.numel() != self.n:
            raise ValueError("basis: length mismatch")
        slot = torch.zeros(3 + 2 * (max_cols + 1), dtype=torch.float64, device="cuda")
        slot[2] = omega2
        v = torch.empty(max(self.n, 1), dtype=torch.float64, device="cuda")
        check(lib().cbgx_arnoldi_fused_step(ctypes.byref(self.desc), cols, max_cols, _ptr(w), _ptr(v), _ptr(slot),
                                            eta, int(bool(speculate)), _ws(), _stream()))
        self.count_ = max(self.count_, cols + 1)
        return slot, v[:self.n]

    def dot(self, j: int, w) -> float:
        """basis.cpp:168-187 (single column; syncs)."""
        self._check(j)
        return float(self.cgs_dot(1, w, first=j)[0].item())

    def subtract_scaled(self, j: int, alpha: float, y):
        """basis.cpp:189-205: y -= alpha * column j (y: CUDA tensor, in place)."""
        torch = _torch()
        self._check(j)
        if y.numel() != self.n:
            raise ValueError("basis: length mismatch")
        self.cgs_update(1, torch.tensor([alpha], dtype=torch.float64, device="cuda"), y, first=j)


# ------------------------------------------------------------ sparse
@dataclasses.dataclass
class CsrMatrix:
    """sparse.hpp:17-26 (host arrays, size_t row_ptrs / col_idx)."""
    n_rows: int
    n_cols: int
    row_ptrs: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    def nnz(self):
        return int(self.values.size)


class DeviceCsr:
    """CSR resident on the device (int32 col_idx; int32/int64 row_ptr)."""

    def __init__(self, n_rows, n_cols, row_ptr, col_idx, values):
        torch = _torch()
        self.row_ptr = row_ptr
        self.col_idx = col_idx
        self.values = values
        bits = 64 if row_ptr.dtype == torch.int64 else 32
        self.desc = _lib.Csr(n_rows, n_cols, values.numel(), row_ptr.data_ptr(), bits,
                             col_idx.data_ptr(), values.data_ptr())

    @staticmethod
    def from_host(a: CsrMatrix) -> "DeviceCsr":
        torch = _torch()
        nnz = int(a.row_ptrs[-1])
        rp_dtype = np.int64 if nnz > 0x7FFFFFFF else np.int32
        rp = torch.from_numpy(np.asarray(a.row_ptrs).astype(rp_dtype)).cuda()
        ci = torch.from_numpy(np.asarray(a.col_idx).astype(np.int32)).cuda()
        va = torch.from_numpy(np.ascontiguousarray(a.values, dtype=np.float64)).cuda()
        return DeviceCsr(a.n_rows, a.n_cols, rp, ci, va)


def stencil(kind: int, nx: int, ny: int = None, nz: int = None, pe: float = 0.0,
            row_begin: int = 0, row_end: int = None, col_offset: int = 0) -> DeviceCsr:
    """3-D stencil generated on the device (cbgx_stencil_generate).
    kind 0 = 7-pt Poisson, 1 = 7-pt upwind convdiff, 2 = 27-pt."""
    torch = _torch()
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    n = nx * ny * nz
    row_end = n if row_end is None else row_end
    L = lib()
    nnz = L.cbgx_stencil_nnz(kind, nx, ny, nz, row_begin, row_end)
    rows = row_end - row_begin
    wide = nnz > 0x7FFFFFFF
    rp = torch.empty(rows + 1, dtype=torch.int64 if wide else torch.int32, device="cuda")
    ci = torch.empty(max(nnz, 1), dtype=torch.int32, device="cuda")
    va = torch.empty(max(nnz, 1), dtype=torch.float64, device="cuda")
    check(L.cbgx_stencil_generate(kind, nx, ny, nz, pe, row_begin, row_end, col_offset, _ptr(rp),
                                  64 if wide else 32, _ptr(ci), _ptr(va), _stream()))
    return DeviceCsr(rows, n, rp, ci, va)


def spmv(a: DeviceCsr, x, y=None, want_norm=False, reduction=_lib.REDUCE_TREE):
    import ctypes
    torch = _torch()
    x = _dev(x)
    if y is None:
        y = torch.empty(max(a.desc.n_rows, 1), dtype=torch.float64, device="cuda")
    nrm = torch.empty(1, dtype=torch.float64, device="cuda") if want_norm else None
    check(lib().cbgx_csr_spmv(ctypes.byref(a.desc), _ptr(x), _ptr(y), _ptr(nrm), reduction, _ws(), _stream()))
    return (y[:a.desc.n_rows], nrm) if want_norm else y[:a.desc.n_rows]


@dataclasses.dataclass
class BenchResult:
    """bench.hpp:15-24."""
    format: str
    intensity: int
    elements: int
    stored_bytes: int
    seconds: float       # minimum over trials (CUDA events)
    stored_gbps: float   # stored bytes / time
    logical_gbps: float  # 8 * elements / time


def _read_sweep_launch(basis, col, n, intensity, mul, add, out):
    import ctypes
    check(lib().cbgx_read_sweep(ctypes.byref(basis.desc), col, n, intensity, mul, add, _ptr(out), _ws(), _stream()))


def read_sweep(basis: "KrylovBasis", col: int, n: int, intensity: int, mul: float, add: float) -> float:
    """One device sweep (cbgx_read_sweep): checksum of decode + intensity FMAs."""
    torch = _torch()
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    _read_sweep_launch(basis, col, n, intensity, mul, add, out)
    return float(out.item())


def read_benchmark(elements: int, formats, intensities, trials: int = 10, seed: int = 0) -> List[BenchResult]:
    """run_read_benchmark (bench.hpp:28-30, bench.cpp:100-152) on the device:
    uniform[-1, 1) data of `elements` (rounded down to whole 32-blocks),
    stored in each format, decoded and swept with `intensity` multiply-adds
    per value; the minimum kernel time over `trials` runs (after a warm-up
    run) per (format, intensity)."""
    torch = _torch()
    if elements < 32:
        raise ValueError("bench: need at least one block")
    if trials < 1:
        raise ValueError("bench: trials must be >= 1")
    if any(i < 1 for i in intensities):
        raise ValueError("bench: intensity must be >= 1")
    n = elements // 32 * 32
    g = torch.Generator(device="cuda").manual_seed(seed)
    data = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    u = (torch.rand(2, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).tolist()
    mul, add = 1.0 + u[0] * 1e-7, u[1] * 1e-9
    out = []
    for f in formats:
        fmt = StorageFormat.parse(f) if isinstance(f, str) else f
        basis = KrylovBasis(n, 1, fmt)
        basis.write_vector(0, data)
        stored = fmt.column_bytes(n)
        chk = torch.empty(1, dtype=torch.float64, device="cuda")
        for inten in intensities:
            _read_sweep_launch(basis, 0, n, inten, mul, add, chk)  # warm-up
            best = float("inf")
            for _ in range(trials):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                _read_sweep_launch(basis, 0, n, inten, mul, add, chk)
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1) * 1e-3)
            out.append(BenchResult(fmt.name(), inten, n, stored, best, stored / best / 1e9, 8.0 * n / best / 1e9))
        del basis
    return out


def spmv_plan(a: DeviceCsr) -> int:
    """Tile height of the staged SpMV for this matrix (0: not stageable)."""
    import ctypes
    t = ctypes.c_uint32(0)
    check(lib().cbgx_csr_spmv_plan(ctypes.byref(a.desc), ctypes.byref(t), _stream()))
    return t.value


def spmv_staged(a: DeviceCsr, x, tile_rows: int, b=None, want_norm=False, reduction=_lib.REDUCE_TREE):
    """Staged (bulk-copy) CSR SpMV: y = A x, or r = b - A x when b is given."""
    import ctypes
    torch = _torch()
    x = _dev(x)
    bb = _dev(b) if b is not None else None
    y = torch.empty(max(a.desc.n_rows, 1), dtype=torch.float64, device="cuda")
    nrm = torch.empty(1, dtype=torch.float64, device="cuda") if want_norm else None
    check(lib().cbgx_csr_spmv_staged(ctypes.byref(a.desc), tile_rows, _ptr(x), _ptr(bb), _ptr(y), _ptr(nrm),
                                     reduction, _ws(), _stream()))
    return (y[:a.desc.n_rows], nrm) if want_norm else y[:a.desc.n_rows]


class DictCsr:
    """Dictionary-coded SELL-32 copy of a device CSR matrix (cbgx_csr_dict_*):
    2-byte codes into <= 255 distinct values and column offsets. Raises
    CbgxError for matrices outside that pattern."""

    def __init__(self, a: DeviceCsr, max_level: int = 3):
        """max_level: 0 = 2-byte codes, 1 = up to 1-byte pair codes,
        2 = up to one pattern byte per row, 3 = up to uniform slots
        (cbgx_csr_dict_create2)."""
        import ctypes
        self.a = a
        self.h = ctypes.c_void_p()
        check(lib().cbgx_csr_dict_create2(ctypes.byref(a.desc), max_level, ctypes.byref(self.h), _stream()))

    def layout(self):
        """(level, pairs, patterns): level 0 SELL / 1 ELL4 2-byte codes /
        2 pair-coded ELL8 / 3 row patterns / 4 uniform slots."""
        import ctypes
        lv, npr, npt = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32()
        check(lib().cbgx_csr_dict_layout(self.h, ctypes.byref(lv), ctypes.byref(npr), ctypes.byref(npt)))
        return lv.value, npr.value, npt.value

    def info(self):
        import ctypes
        no, nv, ne = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint64()
        check(lib().cbgx_csr_dict_info(self.h, ctypes.byref(no), ctypes.byref(nv), ctypes.byref(ne)))
        return no.value, nv.value, ne.value

    def spmv(self, x, b=None, want_norm=False, reduction=_lib.REDUCE_TREE):
        """y = A x, or r = b - A x when b is given."""
        import ctypes
        torch = _torch()
        x = _dev(x)
        bb = _dev(b) if b is not None else None
        y = torch.empty(max(self.a.desc.n_rows, 1), dtype=torch.float64, device="cuda")
        nrm = torch.empty(1, dtype=torch.float64, device="cuda") if want_norm else None
        check(lib().cbgx_csr_dict_spmv(ctypes.byref(self.a.desc), self.h, _ptr(x), _ptr(bb), _ptr(y), _ptr(nrm),
                                       reduction, _ws(), _stream()))
        return (y[:self.a.desc.n_rows], nrm) if want_norm else y[:self.a.desc.n_rows]

    def __del__(self):
        try:
            if self.h:
                lib().cbgx_csr_dict_destroy(self.h)
                self.h = None
        except Exception:
            pass


def dot(x, y, reduction=_lib.REDUCE_TREE) -> float:
    torch = _torch()
    x, y = _dev(x), _dev(y)
    if x.numel() != y.numel():
        raise ValueError("dot: length mismatch")
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    check(lib().cbgx_dot(_ptr(x), _ptr(y), x.numel(), reduction, _ptr(out), _ws(), _stream()))
    return float(out.item())


def norm2(x, reduction=_lib.REDUCE_TREE) -> float:
    return float(np.sqrt(dot(x, x, reduction)))


def sin_problem_host(n: int, first: int = 0, count: int = None) -> np.ndarray:
    """x_sol = s/||s||, s[i] = sin(i): generate_problem's recipe
    (sparse.cpp:233-247) with the C library sin and a sequential norm over
    all n; rows [first, first+count). b is then A x_sol on the device
    (bit-identical SpMV)."""
    count = n - first if count is None else count
    out = np.empty(max(count, 1), np.float64)
    check(lib().cbgx_sin_solution(n, first, count, out.ctypes.data, 0))
    return out[:count]


# ------------------------------------------------------------ solver
@dataclasses.dataclass
class GmresConfig:
    """gmres.hpp:17-27 plus the device options."""
    restart: int = 100
    target_rrn: float = 1e-10
    max_total_iterations: int = 20000
    eta: float = 0.70710678118654752
    storage_format: StorageFormat = StorageFormat.f64()
    reduction: int = _lib.REDUCE_TREE
    phase_timing: bool = False
    phase_timing_deferred: bool = False
    fusion: bool = True   # fused single-GPU orthogonalisation kernel when eligible
    sell: bool = True     # SELL-32 copy of A for the SpMV when memory allows
    tma_spmv: bool = True  # staged (bulk-copy) CSR SpMV when every row tile fits
    dict_spmv: bool = True  # dictionary-coded SELL-32 SpMV when A has <= 255 distinct values/offsets

    def c(self):
        flags = (_lib.PHASE_TIMING if self.phase_timing else 0) | \
            (_lib.PHASE_TIMING_DEFERRED if self.phase_timing_deferred else 0) | \
            (0 if self.fusion else _lib.NO_FUSION) | (0 if self.sell else _lib.NO_SELL) | \
            (0 if self.tma_spmv else _lib.NO_TMA_SPMV) | \
            (0 if self.dict_spmv else _lib.NO_DICT_SPMV)
        return _lib.GmresConfig(self.restart, self.target_rrn, self.max_total_iterations, self.eta,
                                self.storage_format.kind, self.storage_format.bit_length,
                                self.reduction, flags)


@dataclasses.dataclass
class ResidualRecord:
    iteration: int
    rrn: float
    is_explicit: bool


class SolveResult:
    """gmres.hpp:37-45 (+ device statistics). The residual history is
    materialised lazily from the raw arrays the C-ABI filled."""

    def __init__(self, converged, total_iterations, restarts, final_rrn, history_arrays, wall_seconds, solution,
                 stats=None):
        self.converged = converged
        self.total_iterations = total_iterations
        self.restarts = restarts
        self.final_rrn = final_rrn
        self.wall_seconds = wall_seconds
        self.solution = solution
        self.stats = stats
        self._hist = history_arrays
        self._records = None

    @property
    def residual_history(self) -> List[ResidualRecord]:
        if self._records is None:
            hi, hr, he, k = self._hist
            self._records = [ResidualRecord(int(hi[i]), float(hr[i]), bool(he[i])) for i in range(k)]
        return self._records


def _history_buffers(cap):
    hi = np.zeros(cap, np.uint64)
    hr = np.zeros(cap, np.float64)
    he = np.zeros(cap, np.uint8)
    h = _lib.History(hi.ctypes.data, hr.ctypes.data, he.ctypes.data, cap, 0)
    return h, (hi, hr, he)


def _result(st: "_lib.SolveStats", hist, bufs, x) -> SolveResult:
    hi, hr, he = bufs
    k = min(hist.length, hist.capacity)
    return SolveResult(bool(st.converged), int(st.total_iterations), int(st.restarts), float(st.final_rrn),
                       (hi[:k].copy(), hr[:k].copy(), he[:k].copy(), k), float(st.wall_seconds), x, st)


def gmres_solve(a: CsrMatrix, b, x0, cfg: GmresConfig = GmresConfig(), out=None) -> SolveResult:
    """gmres.hpp:113-115 drop-in: host CSR / host vectors in, host solution out.
    `out` (optional, float64[n], e.g. pinned) receives the solution instead of
    a fresh array."""
    import ctypes
    n = a.n_rows
    if a.n_rows != a.n_cols:
        raise ValueError("gmres: matrix must be square")
    b = np.ascontiguousarray(b, np.float64)
    x0 = np.ascontiguousarray(x0, np.float64)
    if b.size != n or x0.size != n:
        raise ValueError("gmres: dimension mismatch")
    rp = np.ascontiguousarray(a.row_ptrs, np.uint64)
    ci = np.ascontiguousarray(a.col_idx, np.uint64)
    va = np.ascontiguousarray(a.values, np.float64)
    if out is not None:
        x = out
        if not (isinstance(x, np.ndarray) and x.dtype == np.float64 and x.flags.c_contiguous and x.size >= max(n, 1)):
            raise ValueError("gmres: out must be a contiguous float64 array of n values")
    else:
        x = np.zeros(max(n, 1), np.float64)
    hist, bufs = _history_buffers(2 * cfg.max_total_iterations + 4)
    st = _lib.SolveStats()
    c = cfg.c()
    check(lib().cbgx_gmres_solve_host(n, rp.ctypes.data, ci.ctypes.data, va.ctypes.data, b.ctypes.data,
                                      x0.ctypes.data, ctypes.byref(c), x.ctypes.data, ctypes.byref(hist),
                                      ctypes.byref(st)))
    return _result(st, hist, bufs, x[:n])


class Solver:
    """Device-resident solver (setup once, solve many) -- cbgx_solver_*."""

    def __init__(self, a: DeviceCsr, cfg: GmresConfig = GmresConfig()):
        import ctypes
        self.a = a
        self.cfg = cfg
        self._c = cfg.c()
        h = ctypes.c_void_p()
        check(lib().cbgx_solver_create(ctypes.byref(a.desc), ctypes.byref(self._c), None, ctypes.byref(h)))
        self.h = h

    def solve(self, b, x0=None, x=None) -> SolveResult:
        import ctypes
        torch = _torch()
        n = self.a.desc.n_rows
        b = _dev(b)
        if x0 is None:
            if getattr(self, "_zeros", None) is None:
                self._zeros = torch.zeros(n, dtype=torch.float64, device="cuda")
            x0 = self._zeros
        if x is None:
            x = torch.empty(n, dtype=torch.float64, device="cuda")
        if getattr(self, "_hbufs", None) is None:
            self._hbufs = _history_buffers(2 * self.cfg.max_total_iterations + 4)
        hist, bufs = self._hbufs
        hist.length = 0
        st = _lib.SolveStats()
        check(lib().cbgx_solver_solve(self.h, _ptr(b), _ptr(_dev(x0)), _ptr(x), ctypes.byref(hist),
                                      ctypes.byref(st), _stream()))
        return _result(st, hist, bufs, x)

    def phase_times(self):
        """{phase: device ms} over the deferred-timing solves since last call."""
        ms = np.zeros(8, np.float64)
        check(lib().cbgx_solver_phase_times(self.h, ms.ctypes.data, 8))
        return dict(zip(_lib.PHASES, ms.tolist()))

    def __del__(self):
        try:
            lib().cbgx_solver_destroy(self.h)
        except Exception:
            pass
