"""BLAS-1 entry points of the C-ABI (include/cbgx.h): cbgx_scale (x *= alpha,
sparse.cpp:80-84) and cbgx_axpy (y += alpha x, sparse.cpp:71-78) bit-identical
to the reference's element-wise roundings (one rounding for the scale; a
rounded product then a rounded sum for the axpy -- the reference is built
without FMA contraction), and cbgx_dot in reference order equal to the
oracle's sequential sum (sparse.cpp:58-67). Called through ctypes, device
buffers from torch."""
import ctypes

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


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("n", [1, 31, 4099, 1 << 20])
@pytest.mark.parametrize("alpha", [0.75, -3.0e-7, 1.0 / 3.0])
def test_scale_axpy_bit_exact(cbg, n, alpha):
    import torch
    from paper_2409_15468_b200 import _lib
    L = _lib.lib()
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n) * 10.0 ** rng.integers(-30, 30, n)
    y = rng.standard_normal(n)
    dx, dy = _dev(x), _dev(y)
    st = torch.cuda.current_stream().cuda_stream
    _lib.check(L.cbgx_axpy(alpha, ctypes.c_void_p(dx.data_ptr()), ctypes.c_void_p(dy.data_ptr()), n, st))
    _lib.check(L.cbgx_scale(alpha, ctypes.c_void_p(dx.data_ptr()), n, st))
    torch.cuda.synchronize()
    ref_y = y + alpha * x  # numpy: product rounded, then the sum rounded
    ref_x = x * alpha
    assert dy.cpu().numpy().tobytes() == ref_y.tobytes()
    assert dx.cpu().numpy().tobytes() == ref_x.tobytes()


@pytest.mark.parametrize("n", [1, 1000, 65537])
def test_dot_reference_order(cbg, port, n):
    import torch
    from paper_2409_15468_b200 import _lib
    L = _lib.lib()
    rng = np.random.default_rng(3 * n)
    x, y = rng.standard_normal(n), rng.standard_normal(n)
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    dx, dy = _dev(x), _dev(y)
    st = torch.cuda.current_stream().cuda_stream
    _lib.check(L.cbgx_dot(ctypes.c_void_p(dx.data_ptr()), ctypes.c_void_p(dy.data_ptr()), n, _lib.REDUCE_REFERENCE,
                          ctypes.c_void_p(out.data_ptr()), cbg._ws(), st))
    torch.cuda.synchronize()
    assert out.item() == port.dot(x, y)
