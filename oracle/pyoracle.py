"""ctypes front-end for the CPU oracles -- TEST INFRASTRUCTURE ONLY.

Two checkers live behind this module:

* ``Port`` -- oracle/_port/liboracle.so, the plain-C restatement of the
  reference algorithm (oracle/cbg_oracle.c).
* ``Ref``  -- oracle/_ref/libcbgref.so, the unmodified reference sources
  (/root/reference/proj/src) compiled in place by oracle/Makefile, reached
  through oracle/ref_shim.cpp. Present wherever ``build()`` ran with the
  reference mounted; its .so travels to the GPU box with the snapshot.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline /
``--impl reference`` legs may import this. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_port", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcbgref.so")

F64, F32, F16, FRSZ2 = 0, 1, 2, 3
FORMATS = {"f64": (F64, 32), "f32": (F32, 32), "f16": (F16, 32),
           "frsz2-16": (FRSZ2, 16), "frsz2-21": (FRSZ2, 21), "frsz2-32": (FRSZ2, 32)}

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


def build(ref: bool = True) -> None:
    """Compile the checkers (make -C oracle [ref])."""
    targets = ["all"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


class OracleError(RuntimeError):
    pass


class NonFinite(ValueError):
    def __init__(self, index):
        super().__init__(f"frsz2: non-finite value at index {index}")
        self.index = index


class Breakdown(RuntimeError):
    def __init__(self, iteration):
        super().__init__(f"solver breakdown at iteration {iteration}")
        self.iteration = iteration


class _GmresCfg(C.Structure):
    _fields_ = [("restart", C.c_size_t), ("target_rrn", C.c_double),
                ("max_total_iterations", C.c_size_t), ("eta", C.c_double),
                ("fmt", C.c_int), ("bit_length", C.c_uint32)]


class _GmresRes(C.Structure):
    _fields_ = [("converged", C.c_int), ("total_iterations", C.c_size_t),
                ("restarts", C.c_size_t), ("final_rrn", C.c_double),
                ("history_len", C.c_size_t)]


def _nb(n, bs=32):
    return (n + bs - 1) // bs


def _wpb(bs, l):
    return (bs * l + 31) // 32


class Port:
    """The plain-C restatement (oracle/cbg_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        sz, u32, u64, dbl = C.c_size_t, C.c_uint32, C.c_uint64, C.c_double
        L.orc_encode_one.argtypes = [dbl, u32, u32]; L.orc_encode_one.restype = u64
        L.orc_decode_one.argtypes = [u64, u32, u32]; L.orc_decode_one.restype = dbl
        L.orc_max_biased_exp.argtypes = [_dp, sz]; L.orc_max_biased_exp.restype = u32
        L.orc_storage_bytes.argtypes = [sz, u32, u32]; L.orc_storage_bytes.restype = sz
        L.orc_max_abs_error_bound.argtypes = [u32, u32]; L.orc_max_abs_error_bound.restype = dbl
        L.orc_compress.argtypes = [_dp, sz, u32, u32, _u32p, _u32p, C.POINTER(u64)]
        L.orc_compress_block.argtypes = [_dp, sz, u32, C.POINTER(u32), _u64p, C.POINTER(u64)]
        L.orc_decompress.argtypes = [_u32p, _u32p, sz, u32, u32, _dp]
        L.orc_decompress_block.argtypes = [_u32p, _u32p, sz, u32, u32, sz, _dp]
        L.orc_decompress_value.argtypes = [_u32p, _u32p, sz, u32, u32, sz, C.POINTER(dbl)]
        L.orc_container_size.argtypes = [sz, u32, u32]; L.orc_container_size.restype = sz
        L.orc_container_write.argtypes = [_u32p, _u32p, sz, u32, u32, _u8p]
        L.orc_container_write.restype = sz
        L.orc_container_read.argtypes = [_u8p, sz, C.POINTER(u32), C.POINTER(u32),
                                         C.POINTER(u64), C.c_void_p, C.c_void_p,
                                         C.c_char_p, sz]
        L.orc_oracle_biased_exp.argtypes = [dbl]; L.orc_oracle_biased_exp.restype = u32
        L.orc_truncate_exact.argtypes = [dbl, u32, u32, C.POINTER(u64), C.POINTER(dbl)]
        L.orc_brute_force_code.argtypes = [dbl, u32, u32]; L.orc_brute_force_code.restype = u64
        L.orc_half_from_double.argtypes = [dbl]; L.orc_half_from_double.restype = C.c_uint16
        L.orc_half_to_double.argtypes = [C.c_uint16]; L.orc_half_to_double.restype = dbl
        L.orc_spmv.argtypes = [sz, _u64p, _u64p, _dp, _dp, _dp]
        L.orc_dot.argtypes = [_dp, _dp, sz]; L.orc_dot.restype = dbl
        L.orc_norm2.argtypes = [_dp, sz]; L.orc_norm2.restype = dbl
        L.orc_generate_problem.argtypes = [sz, _u64p, _u64p, _dp, _dp, _dp]
        L.orc_convdiff_nnz.argtypes = [sz, sz]; L.orc_convdiff_nnz.restype = sz
        L.orc_gen_convdiff.argtypes = [sz, sz, dbl, _u64p, _u64p, _dp]
        L.orc_rescale_rows_geometric.argtypes = [sz, _u64p, _dp, dbl]
        L.orc_stencil_nnz.argtypes = [C.c_int, sz, sz, sz]; L.orc_stencil_nnz.restype = sz
        L.orc_gen_stencil.argtypes = [C.c_int, sz, sz, sz, dbl, _u64p, _u64p, _dp]
        L.orc_arnoldi_orthogonalize.argtypes = [C.c_int, u32, sz, sz, _dp, _dp, _dp, dbl, _dp]
        L.orc_basis_dot.argtypes = [C.c_int, u32, sz, _dp, _dp, C.POINTER(dbl)]
        L.orc_basis_subtract_scaled.argtypes = [C.c_int, u32, sz, _dp, dbl, _dp]
        L.orc_basis_roundtrip.argtypes = [C.c_int, u32, sz, _dp, _dp]
        L.orc_gmres_solve.argtypes = [sz, _u64p, _u64p, _dp, _dp, _dp,
                                      C.POINTER(_GmresCfg), C.POINTER(_GmresRes), _dp,
                                      _u64p, _dp, _u8p, sz, C.POINTER(u64)]

    # -- codec
    def compress(self, v, l=32, bs=32):
        v = np.ascontiguousarray(v, dtype=np.float64)
        n = v.size
        exps = np.zeros(max(_nb(n, bs), 1), np.uint32)
        pay = np.zeros(max(_nb(n, bs) * _wpb(bs, l), 1), np.uint32)
        bad = C.c_uint64(0)
        st = self.lib.orc_compress(v, n, bs, l, exps, pay, C.byref(bad))
        if st == 2:
            raise NonFinite(bad.value)
        if st:
            raise ValueError(f"compress status {st}")
        return exps[:_nb(n, bs)], pay[:_nb(n, bs) * _wpb(bs, l)]

    def compress_block(self, v, l):
        v = np.ascontiguousarray(v, dtype=np.float64)
        codes = np.zeros(max(v.size, 1), np.uint64)
        e = C.c_uint32(0)
        bad = C.c_uint64(0)
        st = self.lib.orc_compress_block(v, v.size, l, C.byref(e), codes, C.byref(bad))
        if st == 2:
            raise NonFinite(bad.value)
        if st:
            raise ValueError(f"compress_block status {st}")
        return e.value, codes[:v.size]

    def decompress(self, exps, pay, n, l=32, bs=32):
        out = np.zeros(max(n, 1), np.float64)
        st = self.lib.orc_decompress(np.ascontiguousarray(exps, np.uint32) if exps.size else np.zeros(1, np.uint32),
                                     np.ascontiguousarray(pay, np.uint32) if pay.size else np.zeros(1, np.uint32),
                                     n, bs, l, out)
        if st:
            raise ValueError(f"decompress status {st}")
        return out[:n]

    def container(self, exps, pay, n, l=32, bs=32) -> bytes:
        size = self.lib.orc_container_size(n, bs, l)
        out = np.zeros(size, np.uint8)
        e = np.ascontiguousarray(exps, np.uint32) if exps.size else np.zeros(1, np.uint32)
        p = np.ascontiguousarray(pay, np.uint32) if pay.size else np.zeros(1, np.uint32)
        w = self.lib.orc_container_write(e, p, n, bs, l, out)
        assert w == size
        return out.tobytes()

    def read_container(self, data: bytes):
        buf = np.frombuffer(data, np.uint8).copy() if data else np.zeros(1, np.uint8)
        bs, l, n = C.c_uint32(), C.c_uint32(), C.c_uint64()
        msg = C.create_string_buffer(128)
        st = self.lib.orc_container_read(buf, len(data), C.byref(bs), C.byref(l), C.byref(n),
                                         None, None, msg, 128)
        if st:
            raise OracleError(msg.value.decode())
        nb = _nb(n.value, bs.value)
        exps = np.zeros(max(nb, 1), np.uint32)
        pay = np.zeros(max(nb * _wpb(bs.value, l.value), 1), np.uint32)
        self.lib.orc_container_read(buf, len(data), C.byref(bs), C.byref(l), C.byref(n),
                                    exps.ctypes.data, pay.ctypes.data, msg, 128)
        return bs.value, l.value, n.value, exps[:nb], pay[:nb * _wpb(bs.value, l.value)]

    def truncate_exact(self, x, e_max, l):
        code, val = C.c_uint64(), C.c_double()
        self.lib.orc_truncate_exact(float(x), e_max, l, C.byref(code), C.byref(val))
        return code.value, val.value

    # -- sparse
    def stencil(self, kind, nx, ny=None, nz=None, pe=0.0):
        ny = nx if ny is None else ny
        nz = nx if nz is None else nz
        n = nx * ny * nz
        nnz = self.lib.orc_stencil_nnz(kind, nx, ny, nz)
        rp = np.zeros(n + 1, np.uint64)
        ci = np.zeros(nnz, np.uint64)
        va = np.zeros(nnz, np.float64)
        assert self.lib.orc_gen_stencil(kind, nx, ny, nz, pe, rp, ci, va) == 0
        return rp, ci, va

    def convdiff(self, nx, ny, pe, decades=0.0):
        nnz = self.lib.orc_convdiff_nnz(nx, ny)
        rp = np.zeros(nx * ny + 1, np.uint64)
        ci = np.zeros(nnz, np.uint64)
        va = np.zeros(nnz, np.float64)
        assert self.lib.orc_gen_convdiff(nx, ny, pe, rp, ci, va) == 0
        if decades:
            self.lib.orc_rescale_rows_geometric(nx * ny, rp, va, decades)
        return rp, ci, va

    def spmv(self, rp, ci, va, x):
        n = rp.size - 1
        y = np.zeros(n, np.float64)
        self.lib.orc_spmv(n, rp, ci, va, np.ascontiguousarray(x, np.float64), y)
        return y

    def generate_problem(self, rp, ci, va):
        n = rp.size - 1
        b = np.zeros(n, np.float64)
        x = np.zeros(n, np.float64)
        assert self.lib.orc_generate_problem(n, rp, ci, va, b, x) == 0
        return b, x

    def norm2(self, x):
        x = np.ascontiguousarray(x, np.float64)
        return self.lib.orc_norm2(x, x.size)

    def dot(self, x, y):
        return self.lib.orc_dot(np.ascontiguousarray(x, np.float64),
                                np.ascontiguousarray(y, np.float64), len(x))

    # -- basis / solver
    def arnoldi(self, fmt, cols, w, eta=0.70710678118654752):
        kind, l = FORMATS[fmt]
        cols = np.ascontiguousarray(cols, np.float64)
        k, n = cols.shape
        w = np.array(w, np.float64, copy=True)
        h = np.zeros(max(k, 1), np.float64)
        out = np.zeros(4, np.float64)
        assert self.lib.orc_arnoldi_orthogonalize(kind, l, n, k, cols.reshape(-1) if k else np.zeros(1),
                                                  w, h, eta, out) == 0
        return h[:k], w, dict(omega=out[0], h_next=out[1], reorth=bool(out[2]),
                              breakdown=bool(out[3]))

    def basis_roundtrip(self, fmt, col):
        kind, l = FORMATS[fmt]
        col = np.ascontiguousarray(col, np.float64)
        out = np.zeros(col.size, np.float64)
        assert self.lib.orc_basis_roundtrip(kind, l, col.size, col, out) == 0
        return out

    def basis_subtract_scaled(self, fmt, col, alpha, y):
        """y -= alpha * column (through the storage format), in place
        (basis.cpp:189-205)."""
        kind, l = FORMATS[fmt]
        assert y.dtype == np.float64 and y.flags.c_contiguous
        assert self.lib.orc_basis_subtract_scaled(kind, l, y.size, np.ascontiguousarray(col, np.float64),
                                                  float(alpha), y) == 0
        return y

    def basis_dot(self, fmt, col, w):
        kind, l = FORMATS[fmt]
        out = C.c_double()
        assert self.lib.orc_basis_dot(kind, l, len(col), np.ascontiguousarray(col, np.float64),
                                      np.ascontiguousarray(w, np.float64), C.byref(out)) == 0
        return out.value

    def gmres(self, rp, ci, va, b, x0=None, fmt="f64", restart=100, target=1e-10,
              max_it=20000, eta=0.70710678118654752):
        n = rp.size - 1
        kind, l = FORMATS[fmt]
        x0 = np.zeros(n) if x0 is None else np.ascontiguousarray(x0, np.float64)
        cfg = _GmresCfg(restart, target, max_it, eta, kind, l)
        res = _GmresRes()
        cap = 2 * max_it + 4
        hi = np.zeros(cap, np.uint64)
        hr = np.zeros(cap, np.float64)
        he = np.zeros(cap, np.uint8)
        x = np.zeros(n, np.float64)
        bad = C.c_uint64()
        st = self.lib.orc_gmres_solve(n, rp, ci, va, np.ascontiguousarray(b, np.float64), x0,
                                      C.byref(cfg), C.byref(res), x, hi, hr, he, cap,
                                      C.byref(bad))
        if st == 4:
            raise Breakdown(bad.value)
        if st:
            raise ValueError(f"gmres status {st}")
        h = res.history_len
        return dict(converged=bool(res.converged), iterations=res.total_iterations,
                    restarts=res.restarts, final_rrn=res.final_rrn, x=x,
                    history=list(zip(hi[:h].tolist(), hr[:h].tolist(), he[:h].astype(bool).tolist())))


class Ref:
    """The unmodified reference library (oracle/_ref/libcbgref.so)."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self, path: str = REF_SO):
        L = self.lib = C.CDLL(path)
        u32, u64, dbl = C.c_uint32, C.c_uint64, C.c_double
        L.ref_last_error.restype = C.c_char_p
        L.ref_compress.argtypes = [_dp, u64, u32, u32, _u32p, _u32p]
        L.ref_compress_container.argtypes = [_dp, u64, u32, u32, _u8p, u64, C.POINTER(u64)]
        L.ref_decompress_container.argtypes = [_u8p, u64, _dp]
        L.ref_half_from_double.argtypes = [dbl]; L.ref_half_from_double.restype = C.c_uint16
        L.ref_half_to_double.argtypes = [C.c_uint16]; L.ref_half_to_double.restype = dbl
        L.ref_spmv.argtypes = [u64, _u64p, _u64p, _dp, _dp, _dp]
        L.ref_generate_problem.argtypes = [u64, _u64p, _u64p, _dp, _dp, _dp]
        L.ref_gen_convdiff.argtypes = [u64, u64, dbl, dbl, _u64p, _u64p, _dp]
        L.ref_arnoldi.argtypes = [C.c_int, u32, u64, u64, _dp, _dp, _dp, dbl, _dp]
        L.ref_gmres_solve.argtypes = [u64, _u64p, _u64p, _dp, _dp, _dp, u64, dbl, u64, dbl,
                                      C.c_int, u32, C.POINTER(C.c_int), C.POINTER(u64),
                                      C.POINTER(u64), C.POINTER(dbl), _dp, _u64p, _dp, _u8p,
                                      u64, C.POINTER(u64), C.POINTER(dbl)]

    def error(self):
        return self.lib.ref_last_error().decode()

    def container(self, v, l=32, bs=32) -> bytes:
        v = np.ascontiguousarray(v, np.float64)
        cap = 24 + (_nb(v.size, bs) * (_wpb(bs, l) + 1)) * 4
        out = np.zeros(max(cap, 1), np.uint8)
        ln = C.c_uint64()
        st = self.lib.ref_compress_container(v if v.size else np.zeros(1), v.size, bs, l,
                                             out, cap, C.byref(ln))
        if st:
            raise ValueError(self.error())
        return out[:ln.value].tobytes()

    def decompress_container(self, data: bytes, n: int):
        out = np.zeros(max(n, 1), np.float64)
        st = self.lib.ref_decompress_container(np.frombuffer(data, np.uint8).copy(), len(data), out)
        if st:
            raise ValueError(self.error())
        return out[:n]

    def arnoldi(self, fmt, cols, w, eta=0.70710678118654752):
        kind, l = FORMATS[fmt]
        cols = np.ascontiguousarray(cols, np.float64)
        k, n = cols.shape
        w = np.array(w, np.float64, copy=True)
        h = np.zeros(max(k, 1), np.float64)
        out = np.zeros(4, np.float64)
        assert self.lib.ref_arnoldi(kind, l, n, k, cols.reshape(-1) if k else np.zeros(1),
                                    w, h, eta, out) == 0, self.error()
        return h[:k], w, dict(omega=out[0], h_next=out[1], reorth=bool(out[2]),
                              breakdown=bool(out[3]))

    def gmres(self, rp, ci, va, b, x0=None, fmt="f64", restart=100, target=1e-10,
              max_it=20000, eta=0.70710678118654752):
        n = rp.size - 1
        kind, l = FORMATS[fmt]
        x0 = np.zeros(n) if x0 is None else np.ascontiguousarray(x0, np.float64)
        cap = 2 * max_it + 4
        hi = np.zeros(cap, np.uint64)
        hr = np.zeros(cap, np.float64)
        he = np.zeros(cap, np.uint8)
        x = np.zeros(n, np.float64)
        conv, it, rs, fr, hl, wall = (C.c_int(), C.c_uint64(), C.c_uint64(), C.c_double(),
                                      C.c_uint64(), C.c_double())
        st = self.lib.ref_gmres_solve(n, rp, ci, va, np.ascontiguousarray(b, np.float64), x0,
                                      restart, target, max_it, eta, kind, l, C.byref(conv),
                                      C.byref(it), C.byref(rs), C.byref(fr), x, hi, hr, he, cap,
                                      C.byref(hl), C.byref(wall))
        if st == 4:
            raise Breakdown(it.value)
        if st:
            raise ValueError(self.error())
        h = hl.value
        return dict(converged=bool(conv.value), iterations=it.value, restarts=rs.value,
                    final_rrn=fr.value, x=x, wall_seconds=wall.value,
                    history=list(zip(hi[:h].tolist(), hr[:h].tolist(), he[:h].astype(bool).tolist())))


RNG_SO = os.path.join(HERE, "_port", "libstdrng.so")
_rng = None


def _rnglib():
    global _rng
    if _rng is None:
        if not os.path.exists(RNG_SO):
            build(ref=False)
        _rng = C.CDLL(RNG_SO)
        _rng.rng_uniform.argtypes = [C.c_uint64, C.c_double, C.c_double, _dp, C.c_size_t]
        _rng.rng_mixed.argtypes = [C.c_uint64, _dp, C.c_size_t]
        _rng.rng_wide.argtypes = [C.c_uint64, C.c_int, C.c_int, _dp, C.c_size_t]
    return _rng


def uniform_values(n, seed, lo=-1.0, hi=1.0):
    """std::mt19937_64(seed) + uniform_real_distribution(lo, hi) (acceptance.cpp:60-68)."""
    out = np.zeros(max(n, 1), np.float64)
    _rnglib().rng_uniform(seed, lo, hi, out, n)
    return out[:n]


def mixed_values(n, seed):
    """test_kernels.cpp:26-41 corner-case generator."""
    out = np.zeros(max(n, 1), np.float64)
    _rnglib().rng_mixed(seed, out, n)
    return out[:n]


def wide_values(n, seed, lo_e=-60, hi_e=0):
    out = np.zeros(max(n, 1), np.float64)
    _rnglib().rng_wide(seed, lo_e, hi_e, out, n)
    return out[:n]
