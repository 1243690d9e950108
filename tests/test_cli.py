"""The `cbgmres` tool (reference proj/tools/cbgmres_main.cpp + proj/src/cli.cpp)
over the B200 drop-in: option parsing, exit codes, host-only subcommands on
CPU; solve / codec / bench against the reference's golden files on the GPU."""
import json
import os
import subprocess

import numpy as np
import pytest

from helpers import ROOT

PKG = os.path.join(ROOT, "paper_2409_15468_b200")
BIN = os.path.join(PKG, "cbgmres")
GOLD = os.path.join(ROOT, "tests", "golden")


def run(*args, cwd=None, timeout=600):
    return subprocess.run([BIN, *map(str, args)], capture_output=True, text=True, cwd=cwd, timeout=timeout)


@pytest.fixture(scope="module", autouse=True)
def built():
    if not os.path.exists(BIN):
        from paper_2409_15468_b200 import build as b
        b.build()
    assert os.path.exists(BIN)


def need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


# ------------------------------------------------------------------ CPU
def test_usage_and_parse_errors():
    r = run()
    assert r.returncode == 1 and "usage: cbgmres" in r.stderr
    r = run("--help")
    assert r.returncode == 0 and "gen-convdiff" in r.stdout
    assert run("frobnicate").returncode == 1
    assert run("solve", "--bogus", "1").returncode == 1
    r = run("solve", "--matrix", "a.mtx", "--gen-convdiff")
    assert r.returncode == 1 and "excludes" in r.stderr
    r = run("gen-convdiff", "--nx", "4", "--out", "x.mtx")
    assert r.returncode == 1 and "--ny is required" in r.stderr
    r = run("codec", "compress", "--input", "x")
    assert r.returncode == 1 and "--output is required" in r.stderr
    r = run("codec", "roundtrip", "--input", "x", "--output", "y")  # roundtrip takes no --output
    assert r.returncode == 1
    r = run("solve", "--gen-convdiff", "--nx", "4", "--ny", "4", "--format", "bf16")
    assert r.returncode == 1 and "unknown storage format 'bf16'" in r.stderr
    r = run("solve", "--gen-convdiff", "--nx", "4", "--ny", "4", "--repeat", "0")
    assert r.returncode == 1 and "--repeat must be >= 1" in r.stderr
    r = run("solve", "--matrix", "/nonexistent.mtx")
    assert r.returncode == 1 and r.stderr.startswith("solve: cannot open")
    r = run("bench", "--log2-elements", "4")
    assert r.returncode == 1 and "--log2-elements must be in [5, 32]" in r.stderr


def test_gen_convdiff_and_analyze(tmp_path):
    """gen-convdiff writes the reference generator's matrix (sparse.cpp:249-291,
    restated in the oracle) as MatrixMarket; analyze's histograms (cli.cpp:
    273-357) agree with numpy on it."""
    from oracle import pyoracle as po
    P = po.Port()

    mtx = tmp_path / "cd.mtx"
    r = run("gen-convdiff", "--nx", 9, "--ny", 7, "--peclet", 1.5, "--out", mtx)
    assert r.returncode == 0, r.stderr
    rp, ci, va = P.convdiff(9, 7, 1.5)
    assert r.stdout == f"wrote 63x63 matrix with {len(va)} nonzeros to {mtx}\n"
    lines = mtx.read_text().splitlines()
    assert lines[0].startswith("%%MatrixMarket matrix coordinate real general")
    body = [l for l in lines[1:] if not l.startswith("%")]
    assert body[0].split() == ["63", "63", str(len(va))]
    rows = np.repeat(np.arange(63), np.diff(np.asarray(rp, dtype=np.int64)))
    got = np.array([[float(x) for x in l.split()] for l in body[1:]])
    np.testing.assert_array_equal(got[:, 0] - 1, rows)
    np.testing.assert_array_equal(got[:, 1] - 1, np.asarray(ci, dtype=np.int64))
    np.testing.assert_array_equal(got[:, 2], va)

    pre = tmp_path / "an"
    r = run("analyze", "--matrix", mtx, "--bins", 5, "--out-prefix", pre)
    assert r.returncode == 0, r.stderr
    nz = va[va != 0]
    e = np.frexp(np.abs(nz))[1] - 1  # ilogb
    assert r.stdout == f"values={len(va)} nonzero={len(nz)} exponent_min={e.min()} exponent_max={e.max()}\n"
    ex = np.loadtxt(f"{pre}_exponents.csv", delimiter=",", skiprows=1, dtype=np.int64, ndmin=2)
    np.testing.assert_array_equal(ex[:, 0], np.arange(e.min(), e.max() + 1))
    np.testing.assert_array_equal(ex[:, 1], np.bincount(e - e.min()))
    vh = np.loadtxt(f"{pre}_values.csv", delimiter=",", skiprows=1, ndmin=2)
    assert vh.shape == (5, 3) and vh[:, 2].sum() == len(va)
    assert vh[0, 0] == va.min() and vh[-1, 1] == va.max()


def test_analyze_vector_constant_and_zero(tmp_path):
    v = tmp_path / "v.f64"
    np.full(10, 3.0).tofile(v)
    r = run("analyze", "--vector", v, "--out-prefix", tmp_path / "c")
    assert r.returncode == 0
    assert r.stdout == "values=10 nonzero=10 exponent_min=1 exponent_max=1\n"
    assert (tmp_path / "c_values.csv").read_text() == "bin_lo,bin_hi,count\n3,3,10\n"
    np.zeros(4).tofile(v)
    r = run("analyze", "--vector", v, "--out-prefix", tmp_path / "z")
    assert r.returncode == 0 and r.stdout == "no nonzero values\n"
    assert (tmp_path / "z_exponents.csv").read_text() == "exponent,count\n"
    r = run("analyze", "--out-prefix", tmp_path / "z")
    assert r.returncode == 1 and "one of --matrix / --vector is required" in r.stderr


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("fmt", ["frsz2-32", "f64", "frsz2-21"])
def test_solve_matches_reference_residuals(tmp_path, fmt):
    """`solve --gen-convdiff` with the reference's reduction order writes the
    reference's residuals.csv byte for byte (golden: the reference's own
    gmres_solve, tests/golden/make_golden.py) and its summary line."""
    need_gpu()
    meta = json.load(open(os.path.join(GOLD, "golden.json")))["solves"][f"convdiff100_pe1/{fmt}"]
    res = tmp_path / "res.csv"
    r = run("solve", "--gen-convdiff", "--nx", 100, "--ny", 100, "--peclet", 1, "--format", fmt,
            "--residuals", res, "--reduction", "reference")
    assert r.returncode == 0, r.stderr
    assert res.read_bytes() == open(os.path.join(GOLD, meta["residuals"]), "rb").read()
    kv = dict(t.split("=", 1) for t in r.stdout.split())
    assert kv["matrix"] == "convdiff-100x100-pe1" and kv["format"] == fmt
    assert int(kv["iterations"]) == meta["iterations"] and int(kv["restarts"]) == meta["restarts"]
    assert float(kv["final_rrn"]) == meta["final_rrn"] and kv["converged"] == "1"


@pytest.mark.gpu
def test_solve_matrix_file_rowscale_and_exit_codes(tmp_path):
    need_gpu()
    mtx = tmp_path / "cd8.mtx"
    assert run("gen-convdiff", "--nx", 8, "--ny", 8, "--peclet", 1, "--out", mtx).returncode == 0
    meta = json.load(open(os.path.join(GOLD, "golden.json")))["solves"]["convdiff8_pe1_rs12/frsz2-32"]
    res = tmp_path / "r.csv"
    r = run("solve", "--matrix", mtx, "--row-scale-decades", 12, "--format", "frsz2-32", "--residuals", res,
            "--reduction", "reference", "--repeat", 2)
    assert r.returncode == 0, r.stderr
    assert res.read_bytes() == open(os.path.join(GOLD, meta["residuals"]), "rb").read()
    kv = dict(t.split("=", 1) for t in r.stdout.split())
    assert kv["matrix"] == "cd8.mtx-rs12" and "wall_mean_s" in kv and "wall_min_s" in kv
    # tree order (default): same contract as the solver tests
    r = run("solve", "--matrix", mtx, "--format", "frsz2-32", "--residuals", res)
    assert r.returncode == 0, r.stderr
    # not converged within the cap: exit code 2, history still written
    r = run("solve", "--gen-convdiff", "--nx", 100, "--ny", 100, "--peclet", 1, "--max-iters", 10,
            "--residuals", res)
    assert r.returncode == 2 and "converged=0 iterations=10" in r.stdout
    assert res.read_text().startswith("iteration,rrn,explicit\n0,1,1\n")


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["mixed_4099_s7", "wide_5000_s11"])
@pytest.mark.parametrize("bits", [16, 21, 32])
def test_codec_container_files(tmp_path, case, bits):
    """`codec compress` writes the reference's container bytes (golden files
    from the reference's write_frsz2_file); decompress and roundtrip agree."""
    need_gpu()
    x = np.load(os.path.join(GOLD, f"in_{case}.npy"))
    raw = tmp_path / "in.f64"
    x.astype("<f8").tofile(raw)
    out = tmp_path / "c.frsz2"
    r = run("codec", "compress", "--input", raw, "--output", out, "--bits", bits)
    assert r.returncode == 0, r.stderr
    gold = open(os.path.join(GOLD, f"c_{case}_l{bits}.frsz2"), "rb").read()
    assert out.read_bytes() == gold
    assert r.stdout == f"compressed {len(x)} values to {len(gold) - 24} payload bytes (+24-byte header)\n"
    back = tmp_path / "back.f64"
    r = run("codec", "decompress", "--input", out, "--output", back)
    assert r.returncode == 0 and r.stdout == f"decompressed {len(x)} values\n"
    d = np.fromfile(back, dtype="<f8")
    r = run("codec", "roundtrip", "--input", raw, "--bits", bits)
    assert r.returncode == 0
    kv = dict(t.split("=", 1) for t in r.stdout.split())
    assert int(kv["values"]) == len(x) and int(kv["compressed_bytes"]) == len(gold) - 24
    assert float(kv["max_abs_error"]) == np.max(np.abs(x - d))
    assert float(kv["max_abs_error"]) < float(kv["max_error_bound"])


@pytest.mark.gpu
def test_codec_errors(tmp_path):
    need_gpu()
    bad = tmp_path / "bad.frsz2"
    bad.write_bytes(b"NOTFRSZ2" + bytes(30))
    r = run("codec", "decompress", "--input", bad, "--output", tmp_path / "o")
    assert r.returncode == 1 and r.stderr == "codec: frsz2 container: bad magic\n"
    odd = tmp_path / "odd.f64"
    odd.write_bytes(bytes(12))
    r = run("codec", "roundtrip", "--input", odd)
    assert r.returncode == 1 and "size is not a multiple of 8" in r.stderr


@pytest.mark.gpu
def test_bench_csv(tmp_path):
    need_gpu()
    out = tmp_path / "b.csv"
    r = run("bench", "--log2-elements", 20, "--formats", "f64,frsz2-32", "--intensities", "1,4", "--trials", 2,
            "--out", out)
    assert r.returncode == 0, r.stderr
    rows = out.read_text().splitlines()
    assert rows[0] == "format,intensity,elements,stored_bytes,seconds,stored_gbps,logical_gbps"
    assert [l.split(",")[:3] for l in rows[1:]] == [["f64", "1", "1048576"], ["f64", "4", "1048576"],
                                                      ["frsz2-32", "1", "1048576"], ["frsz2-32", "4", "1048576"]]
    assert len(r.stdout.splitlines()) == 4
