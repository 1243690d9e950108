"""Pins the C restatement (oracle/cbg_oracle.c) before anything trusts it:
against the reference's own golden vectors / KATs and against fixtures the
unmodified reference produced (tests/golden/make_golden.py)."""
import hashlib
import os
import struct

import numpy as np
import pytest

from oracle import pyoracle as po
from helpers import GOLDEN, csv_of, read_golden_text as read_csv

# acceptance.cpp:159-170 (44 bytes)
GOLDEN_BS4 = bytes([0x46, 0x52, 0x53, 0x5A, 0x32, 0x00, 0x01, 0x00, 0x04, 0, 0, 0,
                    0x20, 0, 0, 0, 0x04, 0, 0, 0, 0, 0, 0, 0, 0xFF, 0x03, 0, 0,
                    0, 0, 0, 0x40, 0, 0, 0, 0x20, 0, 0, 0, 0, 0, 0, 0, 0x90])

SHA_2P24 = {  # SURVEY.md 8(c), reproduced from the reference at survey time
    32: "67e8ca651687a1a5092d43394d72bdd518baa396e57fd547e10792afb22dd258",
    21: "cee77949bb8f2c009206c71047ec9f470d79e116d9dc1f69f50ed091b144ef19",
    16: "383a908bacec7d9d624e75e4e4d0e9d3df0be38aa926c09e8d34d05c31989906",
}


def bits(x):
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def test_golden_container_bs4(port):
    e, p = port.compress([1.0, 0.5, 0.0, -0.25], l=32, bs=4)
    assert port.container(e, p, 4, l=32, bs=4) == GOLDEN_BS4
    bs, l, n, e2, p2 = port.read_container(GOLDEN_BS4)
    assert (bs, l, n) == (4, 32, 4)
    assert list(port.decompress(e2, p2, 4, l=32, bs=4)) == [1.0, 0.5, 0.0, -0.25]


def test_layout_kats(port):
    # test_frsz2.cpp:37-64
    e, codes = port.compress_block([1.0, 0.5, 0.0, -0.25], 32)
    assert e == 1023 and list(codes) == [0x40000000, 0x20000000, 0, 0x90000000]
    e, codes = port.compress_block([0.0, 0.0], 32)
    assert e == 0 and list(codes) == [0, 0]
    e, codes = port.compress_block([1.0 + 2.0 ** -40, 1.0], 32)
    assert port.lib.orc_decode_one(int(codes[0]), e, 32) == 1.0
    with pytest.raises(po.NonFinite, match="index 2"):
        port.compress_block([1.0, 2.0, float("inf"), 0.5], 16)
    # -0 keeps its sign, subnormals flush (test_frsz2.cpp:138-155)
    e, p = port.compress([-0.0, 0.0, 1.0, -1.0], l=16, bs=4)
    back = port.decompress(e, p, 4, l=16, bs=4)
    assert bits(back[0]) == bits(-0.0) and bits(back[1]) == 0
    e, p = port.compress([5e-320, -5e-320, 1.0, 2.0], l=32, bs=4)
    back = port.decompress(e, p, 4, l=32, bs=4)
    assert back[0] == 0.0 and bits(back[1]) == bits(-0.0) and back[2] == 1.0


def test_storage_arithmetic(port):
    # acceptance.cpp:141-149, test_frsz2.cpp:299-313
    assert port.lib.orc_storage_bytes(64, 32, 32) == 264
    assert port.lib.orc_storage_bytes(32, 32, 21) == 88
    assert port.lib.orc_storage_bytes(0, 32, 32) == 0
    assert port.lib.orc_max_abs_error_bound(1023, 32) == 2.0 ** -30
    assert port.lib.orc_max_abs_error_bound(1023, 16) == 2.0 ** -14


def test_sha256_2p24(port):
    v = po.uniform_values(1 << 24, 42)
    assert hashlib.sha256(v.tobytes()).hexdigest() == \
        "546caa03c766761bdfe55651cbe0eb1667780127092cbf702d824b29b029a3d2"
    for l, sha in SHA_2P24.items():
        e, p = port.compress(v, l)
        assert hashlib.sha256(port.container(e, p, v.size, l)).hexdigest() == sha


@pytest.mark.parametrize("name", ["mixed_4099_s7", "wide_5000_s11", "uniform_1000_s3"])
@pytest.mark.parametrize("l", [16, 21, 32])
def test_reference_containers(port, golden, name, l):
    v = np.load(os.path.join(GOLDEN, f"in_{name}.npy"))
    with open(os.path.join(GOLDEN, f"c_{name}_l{l}.frsz2"), "rb") as f:
        want = f.read()
    e, p = port.compress(v, l)
    assert port.container(e, p, v.size, l) == want


def test_truncate_exact_1e6(port):
    # acceptance.cpp:78-103 (criterion 1), on a 2^16 sample per bit length
    for l in (16, 21, 32):
        v = po.uniform_values(1 << 16, 1000 + l)
        e, p = port.compress(v, l)
        back = port.decompress(e, p, v.size, l)
        for i in range(0, v.size, 97):
            code, val = port.truncate_exact(v[i], int(e[i // 32]), l)
            assert bits(back[i]) == bits(val)
            assert abs(v[i] - back[i]) < port.lib.orc_max_abs_error_bound(int(e[i // 32]), l)


def test_brute_force_4096(port):
    # acceptance.cpp:106-138 (criterion 2)
    grid = [0.0, -1.0, 0.8125, 2.5, -0.3, 1.75, 0.0625, -3.9]
    import itertools
    for blk in itertools.product(grid, repeat=4):
        e, codes = port.compress_block(list(blk), 8)
        assert e == max(port.lib.orc_oracle_biased_exp(x) for x in blk)
        for x, c in zip(blk, codes):
            assert c == port.lib.orc_brute_force_code(x, e, 8)


@pytest.mark.parametrize("l", [2, 16, 21, 32, 47, 64])
def test_idempotent_recompression(port, l):
    # test_frsz2.cpp:157-173
    v = po.uniform_values(257, 7000 + l, -100.0, 100.0)
    e, p = port.compress(v, l)
    d = port.decompress(e, p, v.size, l)
    e2, p2 = port.compress(d, l)
    assert np.array_equal(e, e2) and np.array_equal(p, p2)


def test_half_matches_reference(port, ref):
    for h in range(0, 0x10000, 7):
        assert bits(port.lib.orc_half_to_double(h)) == bits(ref.lib.ref_half_to_double(h))
    for x in np.concatenate([po.mixed_values(3000, 5), po.uniform_values(3000, 9, -7e4, 7e4),
                             [65504.0, 65520.0, 1e300, -1e300, 2.0 ** -24, 2.0 ** -25, -0.0]]):
        assert port.lib.orc_half_from_double(x) == ref.lib.ref_half_from_double(x)


@pytest.mark.parametrize("case", ["convdiff100_pe1/f64", "convdiff100_pe1/f32",
                                  "convdiff8_pe1_rs12/frsz2-32", "convdiff12_pe1_m20/frsz2-32",
                                  "p7_16/frsz2-32", "p7_16/frsz2-21", "cd7_12_pe1/frsz2-32",
                                  "p27_10/f64"])
def test_solver_histories_byte_identical(port, golden, case):
    s = golden["solves"][case]
    a = s["args"]
    if s["kind"] == "convdiff":
        rp, ci, va = port.convdiff(a[0], a[1], a[2], decades=a[3])
    else:
        rp, ci, va = port.stencil(a[0], a[1], a[2], a[3], pe=a[4])
    b, _ = port.generate_problem(rp, ci, va)
    r = port.gmres(rp, ci, va, b, fmt=s["fmt"], restart=s["restart"])
    assert r["iterations"] == s["iterations"]
    assert csv_of(r["history"]) == read_csv(s["residuals"])
    assert hashlib.sha256(r["x"].tobytes()).hexdigest() == s["solution_sha256"]


def test_pinned_counts(golden):
    # acceptance.cpp:278-280 criterion 7
    sv = golden["solves"]
    assert sv["convdiff100_pe1/f64"]["iterations"] == 626
    assert sv["convdiff100_pe1/frsz2-32"]["iterations"] == 627
    assert sv["convdiff100_pe1/f32"]["iterations"] == 658
    assert sv["convdiff8_pe1_rs12/frsz2-32"]["converged"]


def test_arnoldi_port_vs_ref(port, ref):
    rng = np.random.default_rng(3)
    n = 301
    cols = np.linalg.qr(rng.standard_normal((n, 7)))[0].T.copy()
    for fmt in ("f64", "f32", "f16", "frsz2-16", "frsz2-21", "frsz2-32"):
        w = rng.standard_normal(n)
        w2 = w.copy()
        w2[:] = cols[:5].T @ np.arange(1, 6) + 1e-9 * w   # forces the re-orth pass
        for vec in (w, w2):
            h1, wo1, f1 = port.arnoldi(fmt, cols, vec)
            h2, wo2, f2 = ref.arnoldi(fmt, cols, vec)
            assert h1.tobytes() == h2.tobytes() and wo1.tobytes() == wo2.tobytes() and f1 == f2


def test_ref_matches_port_containers(port, ref):
    v = po.mixed_values(1000, 99)
    for l in (2, 5, 16, 21, 32, 53, 64):
        e, p = port.compress(v, l)
        assert port.container(e, p, v.size, l) == ref.container(v, l)
