"""GPU parity of the decompress-fused CGS kernels and the basis accessor.

* basis write/read-back: bit-exact vs the oracle's KrylovBasis round trip;
* cgs_update (w -= sum h_j v_j, column order, two roundings): bit-exact vs
  the reference's subtract_scaled sequence;
* cgs_dot: REFERENCE order bit-exact vs KrylovBasis::dot; TREE order
  within 2^-40 relative of a compensated (Kahan) dot of the decoded
  columns (the tolerance of test_basis.cpp:148-177).
"""
import numpy as np
import pytest

from oracle import pyoracle as po

pytestmark = pytest.mark.gpu
FORMATS = ["f64", "f32", "f16", "frsz2-16", "frsz2-21", "frsz2-32"]


@pytest.fixture(scope="module")
def cbg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2409_15468_b200 as m
    return m


def kahan(x, y):
    s = c = 0.0
    for a, b in zip(x.tolist(), y.tolist()):
        t = a * b - c
        u = s + t
        c = (u - s) - t
        s = u
    return s


def make_basis(cbg, fmt, cols):
    k, n = cols.shape
    B = cbg.KrylovBasis(n, k, cbg.StorageFormat.parse(fmt))
    for j in range(k):
        B.write_vector(j, cols[j])
    return B


def columns(n, k, seed):
    rng = np.random.default_rng(seed)
    c = rng.standard_normal((k, n))
    c[:, ::7] *= 1e-3          # exponent variation inside blocks
    if k > 2:
        c[2] *= 1e6
    return c


@pytest.mark.parametrize("fmt", FORMATS)
@pytest.mark.parametrize("n", [77, 4095, 4097, 20000])
def test_write_read_roundtrip(cbg, port, fmt, n):
    cols = columns(n, 3, n)
    B = make_basis(cbg, fmt, cols)
    for j in range(3):
        got = B.read_column(j).cpu().numpy()
        want = port.basis_roundtrip(fmt, cols[j])
        assert got.view(np.uint64).tobytes() == want.view(np.uint64).tobytes()
    blk = B.read_block(0, B.num_blocks() - 1).cpu().numpy()
    tail = n - (B.num_blocks() - 1) * 32
    assert np.all(blk[tail:] == 0.0)


@pytest.mark.parametrize("fmt", FORMATS)
@pytest.mark.parametrize("n,k", [(77, 1), (4096, 7), (12289, 33), (100003, 5)])
def test_update_bit_exact(cbg, port, fmt, n, k):
    import torch
    cols = columns(n, k, 3 * n + k)
    B = make_basis(cbg, fmt, cols)
    rng = np.random.default_rng(k)
    w0 = rng.standard_normal(n)
    h = rng.standard_normal(k)
    w = torch.from_numpy(w0.copy()).cuda()
    nrm = B.cgs_update(k, h, w, want_norm=True)
    # reference: subtract_scaled column by column
    dec = np.stack([port.basis_roundtrip(fmt, cols[j]) for j in range(k)])
    want = w0.copy()
    for j in range(k):
        want = want - h[j] * dec[j]          # numpy: separate mul and sub roundings
    got = w.cpu().numpy()
    assert got.view(np.uint64).tobytes() == want.view(np.uint64).tobytes()
    assert abs(nrm.item() - kahan(want, want)) <= 2.0 ** -40 * kahan(want, want)


@pytest.mark.parametrize("fmt", FORMATS)
@pytest.mark.parametrize("n,k", [(77, 2), (4096, 9), (50001, 17)])
def test_dot_tree_and_reference(cbg, port, fmt, n, k):
    cols = columns(n, k, 5 * n + k)
    B = make_basis(cbg, fmt, cols)
    w = np.random.default_rng(n).standard_normal(n)
    dec = np.stack([port.basis_roundtrip(fmt, cols[j]) for j in range(k)])
    tree = B.cgs_dot(k, w, with_wnorm=True).cpu().numpy()
    for j in range(k):
        ex = kahan(dec[j], w)
        assert abs(tree[j] - ex) <= 2.0 ** -40 * np.abs(dec[j] * w).sum() + 2.0 ** -60
    assert abs(tree[k] - kahan(w, w)) <= 2.0 ** -40 * kahan(w, w)
    refo = B.cgs_dot(k, w, with_wnorm=True, reduction=1).cpu().numpy()
    for j in range(k):
        assert refo[j] == port.basis_dot(fmt, cols[j], w)
    assert refo[k] == port.dot(w, w)


def test_dot_deterministic(cbg):
    n, k = 300000, 40
    cols = columns(n, k, 11)
    B = make_basis(cbg, "frsz2-32", cols)
    w = np.random.default_rng(2).standard_normal(n)
    a = B.cgs_dot(k, w, with_wnorm=True).cpu().numpy()
    b = B.cgs_dot(k, w, with_wnorm=True).cpu().numpy()
    assert a.tobytes() == b.tobytes()


def test_single_column_api(cbg, port):
    import torch
    n = 1000
    cols = columns(n, 2, 1)
    B = make_basis(cbg, "frsz2-32", cols)
    w = np.random.default_rng(3).standard_normal(n)
    assert abs(B.dot(1, w) - port.basis_dot("frsz2-32", cols[1], w)) <= 1e-12 * np.abs(cols[1] * w).sum()
    y = torch.from_numpy(w.copy()).cuda()
    B.subtract_scaled(1, 0.0, y)
    assert np.array_equal(y.cpu().numpy(), w)           # alpha = 0 leaves y unchanged
    with pytest.raises(IndexError):
        B.dot(2, w)
    with pytest.raises(IndexError):
        B.write_vector(3, w)
    with pytest.raises(ValueError):
        B.write_vector(0, w[:-1])
    bad = w.copy()
    bad[17] = np.nan
    C = cbg.KrylovBasis(n, 1, cbg.StorageFormat.frsz2_format(16))
    with pytest.raises(ValueError, match="index 17"):
        C.write_vector(0, bad)


def test_fused_scale_write(cbg):
    import torch
    n = 10000
    x = np.random.default_rng(5).standard_normal(n)
    nrm2 = float(np.dot(x, x))
    B = cbg.KrylovBasis(n, 2, cbg.StorageFormat.frsz2_format(32))
    s = torch.tensor([nrm2], dtype=torch.float64, device="cuda")
    v = torch.empty(n, dtype=torch.float64, device="cuda")
    B.write_vector(0, x, scale=s, scale_mode=1, v_out=v)
    inv = 1.0 / np.sqrt(nrm2)
    want = x * inv
    assert v.cpu().numpy().tobytes() == want.tobytes()
    B.write_vector(1, want)
    assert B.read_column(0).cpu().numpy().tobytes() == B.read_column(1).cpu().numpy().tobytes()


@pytest.mark.parametrize("fmt", ["f64", "f32", "f16", "frsz2-16", "frsz2-21", "frsz2-32"])
def test_read_sweep_checksum(cbg, port, fmt):
    """Read benchmark sweep (bench.cpp:55-96): decoded values after
    `intensity` two-rounding multiply-adds, summed; vs the oracle decode +
    numpy's identical arithmetic (summation order differs: 1e-12 rel.)."""
    import torch
    n = 32 * 1000
    v = np.random.default_rng(5).uniform(-1, 1, n)
    B = cbg.KrylovBasis(n, 2, cbg.StorageFormat.parse(fmt))
    B.write_vector(0, -v)  # columns are written in order (basis.cpp:85-115)
    B.write_vector(1, v)
    dec = port.basis_roundtrip(fmt, v)
    mul, add = 1.0 + 3e-8, -2e-10
    for inten in (1, 3):
        buf = dec.copy()
        for _ in range(inten):
            buf = buf * mul + add
        want = float(np.sum(buf, dtype=np.float64))
        got = cbg.read_sweep(B, 1, n, inten, mul, add)
        assert abs(got - want) <= 1e-12 * np.sum(np.abs(buf)), (fmt, inten, got, want)
    # block exponents near the top of the folded-multiply range (2^52 * scale
    # * mul would overflow): the streamed FMA decode hands those stages to
    # the general path
    if fmt.startswith("frsz2"):
        vb = v * 2.0 ** 500
        Bb = cbg.KrylovBasis(n, 1, cbg.StorageFormat.parse(fmt))
        Bb.write_vector(0, vb)
        decb = port.basis_roundtrip(fmt, vb)
        mulb = 2.0 ** 505
        want = float(np.sum(decb * mulb + add, dtype=np.float64))
        got = cbg.read_sweep(Bb, 0, n, 1, mulb, add)
        assert abs(got - want) <= 1e-12 * np.sum(np.abs(decb * mulb)), (fmt, got, want)
    # partial length (multiple of 32) and argument checks
    got = cbg.read_sweep(B, 1, 64, 1, 1.0, 0.0)
    assert abs(got - float(np.sum(dec[:64]))) <= 1e-14
    with pytest.raises(Exception):
        cbg.read_sweep(B, 1, 33, 1, 1.0, 0.0)


def test_read_benchmark_api(cbg):
    res = cbg.read_benchmark(1 << 16, ["f64", "frsz2-32"], [1, 4], trials=2, seed=3)
    assert [(r.format, r.intensity) for r in res] == [("f64", 1), ("f64", 4), ("frsz2-32", 1), ("frsz2-32", 4)]
    assert res[0].stored_bytes == 8 * 65536 and res[2].stored_bytes == 2048 * 4 * 33
    assert all(r.seconds > 0 and r.logical_gbps > 0 for r in res)


@pytest.mark.parametrize("fmt", ["frsz2-16", "frsz2-21", "frsz2-32"])
def test_column_exponent_ranges(cbg, port, fmt):
    """Every column write folds the column's exponent range (cbgx_basis.
    d_erange: max of 2047 - e over nonzero blocks, max e) in the compress
    kernel; it must equal the range of the oracle's block exponents (the
    CGS kernels choose their decode path from it)."""
    rng = np.random.default_rng(7)
    n = 70_001
    l = int(fmt.split("-")[1])
    cols = [rng.standard_normal(n), np.zeros(n), rng.standard_normal(n) * 1e-300,
            np.where(rng.random(n) < 0.5, 0.0, rng.standard_normal(n) * 10.0 ** rng.integers(-200, 200, n))]
    B = cbg.KrylovBasis(n, len(cols), cbg.StorageFormat.parse(fmt))
    for j, c in enumerate(cols):
        B.write_vector(j, c)
    er = B._erange.cpu().numpy().astype(np.int64)
    for j, c in enumerate(cols):
        e, _ = port.compress(c, l)
        e = np.asarray(e, dtype=np.int64)
        nz = e[e != 0]
        assert er[2 * j] == (int((2047 - nz).max()) if nz.size else 0), j
        assert er[2 * j + 1] == (int(e.max()) if e.size else 0), j
