"""CPU-side checks of the C-ABI library: it loads, exports every entry point
include/cbgx.h declares, the pure host functions answer like the reference,
and compute entry points fail loudly (no CPU fallback) without a device."""
import ctypes
import os
import re

import pytest

from helpers import ROOT

HEADER = os.path.join(ROOT, "include", "cbgx.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cbgx_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    from paper_2409_15468_b200 import _lib
    return _lib.lib()


def test_exports_every_declared_symbol(L):
    syms = declared_symbols()
    assert len(syms) > 30
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing


def test_every_symbol_has_a_ctypes_signature(L):
    missing = [s for s in declared_symbols() if s not in L.cbgx_signatures]
    assert not missing, missing


def test_pure_host_functions(L):
    assert L.cbgx_frsz2_storage_bytes(64, 32, 32) == 264        # acceptance.cpp:141-149
    assert L.cbgx_frsz2_storage_bytes(32, 32, 21) == 88         # test_frsz2.cpp:301
    assert L.cbgx_frsz2_storage_bytes(0, 32, 32) == 0
    assert L.cbgx_frsz2_words_per_block(32, 21) == 21
    assert L.cbgx_frsz2_max_abs_error_bound(1023, 32) == 2.0 ** -30
    for n in (32, 320, 4096):
        assert L.cbgx_frsz2_storage_bytes(n, 32, 21) * 3 == L.cbgx_frsz2_storage_bytes(n, 32, 32) * 2


def test_stencil_nnz_closed_form(L, port):
    for kind in (0, 1, 2):
        for dims in ((5, 4, 3), (1, 7, 2), (16, 16, 16), (3, 1, 1)):
            rp, ci, va = port.stencil(kind, *dims, pe=1.0)
            n = dims[0] * dims[1] * dims[2]
            assert L.cbgx_stencil_nnz(kind, *dims, 0, n) == int(rp[-1])
            for rb, re_ in ((1, n - 1), (n // 3, n // 2), (7 % n, n)):
                if rb < re_:
                    assert L.cbgx_stencil_nnz(kind, *dims, rb, re_) == int(rp[re_] - rp[rb])
    # configs: 7-pt 128^3 / 192^3 and 27-pt 512^3
    assert L.cbgx_stencil_nnz(0, 128, 128, 128, 0, 128 ** 3) == 14_581_760
    assert L.cbgx_stencil_nnz(1, 192, 192, 192, 0, 192 ** 3) == 49_324_032
    assert L.cbgx_stencil_nnz(2, 512, 512, 512, 0, 512 ** 3) == 3_609_741_304


def test_basis_layout(L):
    from paper_2409_15468_b200 import _lib
    B = _lib.Basis()
    db, eb = ctypes.c_uint64(), ctypes.c_uint64()
    assert L.cbgx_basis_layout(3, 21, 100, 5, ctypes.byref(B), ctypes.byref(db), ctypes.byref(eb)) == 0
    assert B.n_pad % 8192 == 0 and B.n_pad >= 100
    # each column: n_pad rows + a 2048-row zero tail (whole fused steps)
    assert B.col_stride_bytes == (B.n_pad + 2048) // 32 * 21 * 4
    assert B.exp_col_stride == (B.n_pad + 2048) // 32
    assert db.value == B.col_stride_bytes * 5 + 64 and eb.value == B.exp_col_stride * 5 * 4
    assert L.cbgx_basis_layout(3, 24, 100, 5, ctypes.byref(B), None, None) == 1
    assert "bit length" in L.cbgx_last_error().decode()


def test_compute_fails_loudly_without_device(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    buf = (ctypes.c_double * 64)()
    st = L.cbgx_frsz2_compress(buf, 64, 32, 32, buf, buf, None)
    assert st == 5  # CBGX_ECUDA
    assert "cuda" in L.cbgx_last_error().decode()
