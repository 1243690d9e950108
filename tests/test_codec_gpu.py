"""GPU parity of the FRSZ2 codec (C-ABI through the Python mirror) against
the oracle and the reference's golden vectors: bit-exact streams and values."""
import hashlib
import os

import numpy as np
import pytest

from helpers import GOLDEN
from oracle import pyoracle as po

pytestmark = pytest.mark.gpu

SHA_2P24 = {
    32: "67e8ca651687a1a5092d43394d72bdd518baa396e57fd547e10792afb22dd258",
    21: "cee77949bb8f2c009206c71047ec9f470d79e116d9dc1f69f50ed091b144ef19",
    16: "383a908bacec7d9d624e75e4e4d0e9d3df0be38aa926c09e8d34d05c31989906",
}
GOLDEN_BS4 = bytes([0x46, 0x52, 0x53, 0x5A, 0x32, 0x00, 0x01, 0x00, 0x04, 0, 0, 0,
                    0x20, 0, 0, 0, 0x04, 0, 0, 0, 0, 0, 0, 0, 0xFF, 0x03, 0, 0,
                    0, 0, 0, 0x40, 0, 0, 0, 0x20, 0, 0, 0, 0, 0, 0, 0, 0x90])


@pytest.fixture(scope="module")
def cbg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2409_15468_b200 as m
    return m


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def test_golden_container_bs4(cbg):
    cv = cbg.compress([1.0, 0.5, 0.0, -0.25], cbg.Frsz2Params(4, 32))
    assert cv.container_bytes() == GOLDEN_BS4
    back = cbg.decompress(cbg.CompressedVector.from_container(GOLDEN_BS4)).cpu().numpy()
    assert list(back) == [1.0, 0.5, 0.0, -0.25]


@pytest.mark.parametrize("l", [32, 21, 16])
def test_sha256_2p24(cbg, port, l):
    v = po.uniform_values(1 << 24, 42)
    cv = cbg.compress(v, cbg.Frsz2Params(32, l))
    assert hashlib.sha256(cv.container_bytes()).hexdigest() == SHA_2P24[l]
    back = cbg.decompress(cv).cpu().numpy()
    e, p = port.compress(v, l)
    assert bits(back).tobytes() == bits(port.decompress(e, p, v.size, l)).tobytes()


@pytest.mark.parametrize("name", ["mixed_4099_s7", "wide_5000_s11", "uniform_1000_s3"])
@pytest.mark.parametrize("l", [16, 21, 32])
def test_reference_golden_containers(cbg, name, l):
    v = np.load(os.path.join(GOLDEN, f"in_{name}.npy"))
    with open(os.path.join(GOLDEN, f"c_{name}_l{l}.frsz2"), "rb") as f:
        want = f.read()
    cv = cbg.compress(v, cbg.Frsz2Params(32, l))
    assert cv.container_bytes() == want
    # decode of the reference's own container
    back = cbg.decompress(cbg.CompressedVector.from_container(want)).cpu().numpy()
    ref = po.Port()
    _, _, n, e, p = ref.read_container(want)
    assert bits(back).tobytes() == bits(ref.decompress(e, p, n, l)).tobytes()


@pytest.mark.parametrize("n", [0, 1, 31, 32, 33, 77, 1000, 65537])
@pytest.mark.parametrize("l", [16, 21, 32])
def test_ragged_lengths(cbg, port, n, l):
    v = po.mixed_values(n, 100 + n)
    cv = cbg.compress(v, cbg.Frsz2Params(32, l))
    e, p = port.compress(v, l)
    assert np.array_equal(cv.exponents(), e) and np.array_equal(cv.payload_words(), p)
    assert bits(cbg.decompress(cv).cpu().numpy()[:n]).tobytes() == bits(port.decompress(e, p, n, l)).tobytes()


@pytest.mark.parametrize("bs", [1, 4, 8, 32, 33])
@pytest.mark.parametrize("l", [2, 3, 5, 7, 8, 12, 16, 21, 31, 32, 47, 50, 53, 64])
def test_generic_codec(cbg, port, bs, l):
    v = po.mixed_values(301, 7 * l + bs)
    cv = cbg.compress(v, cbg.Frsz2Params(bs, l))
    e, p = port.compress(v, l, bs)
    assert np.array_equal(cv.exponents(), e) and np.array_equal(cv.payload_words(), p)
    assert bits(cbg.decompress(cv).cpu().numpy()).tobytes() == bits(port.decompress(e, p, v.size, l, bs)).tobytes()


def test_flush_to_zero_decode(cbg, port):
    # test_kernels.cpp:88-113: random codes at tiny / huge e_max decode like decode_one
    rng = np.random.default_rng(77)
    for l in (16, 21, 32):
        for e_max in (0, 1, 5, 20, 40, 1023, 2046):
            nb = 64
            codes = rng.integers(0, 1 << l, size=nb * 32, dtype=np.uint64)
            # pack through the oracle's stream rule via a container we craft
            words = np.zeros(nb * l, np.uint32)
            for j, c in enumerate(codes.tolist()):
                b, r = divmod(j, 32)
                bit = b * l * 32 + r * l
                for t in range(l):
                    if (c >> t) & 1:
                        q = bit + t
                        words[q >> 5] |= np.uint32(1 << (q & 31))
            exps = np.full(nb, e_max, np.uint32)
            data = port.container(exps, words, nb * 32, l)
            got = cbg.decompress(cbg.CompressedVector.from_container(data)).cpu().numpy()
            want = np.array([port.lib.orc_decode_one(int(c), e_max, l) for c in codes.tolist()])
            assert bits(got).tobytes() == bits(want).tobytes(), (l, e_max)


def test_non_finite_reports_lowest_index(cbg):
    v = np.ones(1000)
    v[733] = np.inf
    v[901] = np.nan
    with pytest.raises(ValueError, match="frsz2: non-finite value at index 733"):
        cbg.compress(v, cbg.Frsz2Params(32, 32))
    with pytest.raises(ValueError, match="index 2"):
        cbg.compress_block([1.0, 2.0, np.inf, 0.5], 16)
    with pytest.raises(ValueError, match="index 5"):
        cbg.compress(np.array([0, 0, 0, 0, 0, np.nan, 1.0]), cbg.Frsz2Params(4, 12))


def test_compress_block_kats(cbg):
    e, codes = cbg.compress_block([1.0, 0.5, 0.0, -0.25], 32)
    assert e == 1023 and list(codes) == [0x40000000, 0x20000000, 0, 0x90000000]
    e, codes = cbg.compress_block([0.0, 0.0], 32)
    assert e == 0 and list(codes) == [0, 0]


def test_block_and_value_access(cbg, port):
    for l in (16, 21, 32, 7, 50):
        v = po.uniform_values(100, 100 + l)
        cv = cbg.compress(v, cbg.Frsz2Params(32, l))
        e, p = port.compress(v, l)
        for b in range(cv.num_blocks()):
            got = cbg.decompress_block(cv, b).cpu().numpy()
            out = np.zeros(32)
            port.lib.orc_decompress_block(e, p, 100, 32, l, b, out)
            assert bits(got).tobytes() == bits(out).tobytes()
        for i in (0, 5, 63, 99):
            assert cbg.decompress_value(cv, i) == port.decompress(e, p, 100, l)[i]
        with pytest.raises(IndexError):
            cbg.decompress_block(cv, cv.num_blocks())
        with pytest.raises(IndexError):
            cbg.decompress_value(cv, 100)


@pytest.mark.parametrize("l", [2, 16, 21, 32, 47, 64])
def test_recompression_idempotent(cbg, l):
    v = po.uniform_values(257, 7000 + l, -100.0, 100.0)
    cv = cbg.compress(v, cbg.Frsz2Params(32, l))
    cv2 = cbg.compress(cbg.decompress(cv), cbg.Frsz2Params(32, l))
    assert np.array_equal(cv.exponents(), cv2.exponents())
    assert np.array_equal(cv.payload_words(), cv2.payload_words())


def test_error_bound_and_truncation_oracle(cbg, port):
    # acceptance.cpp:78-103 on 2^20 values per bit length
    for l in (16, 21, 32):
        v = po.uniform_values(1 << 20, 1000 + l)
        cv = cbg.compress(v, cbg.Frsz2Params(32, l))
        back = cbg.decompress(cv).cpu().numpy()
        e = cv.exponents()
        bound = np.ldexp(1.0, e.astype(np.int64) - 1023 - (l - 2))[np.arange(v.size) // 32]
        assert np.all(np.abs(v - back) < bound)
        assert np.all(np.abs(back) <= np.abs(v))
        for i in range(0, v.size, 4099):
            assert bits(back[i]) == bits(port.truncate_exact(v[i], int(e[i // 32]), l)[1])


@pytest.mark.parametrize("l", [16, 21, 32])
@pytest.mark.parametrize("offset", [1, 2, 3])
def test_unaligned_vectors(cbg, port, l, offset):
    """The fast codec uses 256-bit accesses when the fp64 vector is 32-B
    aligned and 16-B/scalar accesses otherwise: compress from / decompress
    into vectors offset by 8..24 bytes give the same bits."""
    import torch
    n = 4099
    v = port_mixed(port, n)
    big = torch.zeros(n + 8, dtype=torch.float64, device="cuda")
    big[offset:offset + n] = torch.from_numpy(v).cuda()
    src = big[offset:offset + n]
    cv = cbg.compress(src, cbg.Frsz2Params(32, l))
    e, p = port.compress(v, l)
    assert np.array_equal(cv.exponents(), e) and np.array_equal(cv.payload_words(), p)
    out_big = torch.full((n + 8,), 7.0, dtype=torch.float64, device="cuda")
    dst = out_big[offset:offset + n]
    cbg.decompress(cv, out=dst)
    assert dst.cpu().numpy().tobytes() == port.decompress(e, p, n, l).tobytes()
    assert (out_big[:offset] == 7.0).all() and (out_big[offset + n:] == 7.0).all()


def port_mixed(port, n):
    from oracle import pyoracle as po
    return po.mixed_values(n, 7)
