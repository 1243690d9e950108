"""Dictionary-coded SELL-32 SpMV (csrc/dsell.cu): y = A x and r = b - A x
bit-identical to the reference spmv (sparse.cpp:43-56, restated in the
oracle) on stencils, convection-diffusion, ragged rows, empty rows and
row counts off the 32-row slices; matrices outside the dictionary limits
are refused; solves through it equal the CSR-path solves."""
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


def few_valued(rng, n, max_len, offsets, values, empty_frac=0.1):
    """Ragged rows whose entries draw (col - row) from `offsets` (in-row
    order kept sorted) and values from `values`."""
    rows_c, lens = [], []
    for r in range(n):
        L = 0 if rng.random() < empty_frac else int(rng.integers(0, max_len + 1))
        cand = sorted({int(r + o) for o in rng.choice(offsets, size=L)} & set(range(n)))
        rows_c.append(cand)
        lens.append(len(cand))
    rp = np.zeros(n + 1, dtype=np.uint64)
    rp[1:] = np.cumsum(lens)
    ci = np.array([c for cs in rows_c for c in cs], dtype=np.uint64)
    va = rng.choice(values, size=ci.size).astype(np.float64)
    return rp, ci, va


def check_paths(cbg, port, rp, ci, va, seed):
    """Every coding level the matrix admits (2-byte codes, pair codes, row
    patterns, uniform slots -- cbgx_csr_dict_create2) gives the reference's
    y, b - A x and norms bit for bit. Returns the default (highest-level)
    copy."""
    n = rp.size - 1
    A = cbg.DeviceCsr.from_host(cbg.CsrMatrix(n, n, rp, ci, va))
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(n)
    b = rng.standard_normal(n)
    ref = port.spmv(rp, ci, va, x)
    levels = set()
    for max_level in (0, 1, 2, 3):
        D = cbg.DictCsr(A, max_level=max_level)
        level = D.layout()[0]
        assert level <= max_level + 1
        levels.add(level)
        y, nrm = D.spmv(x, want_norm=True)
        assert y.cpu().numpy().tobytes() == ref.tobytes(), level
        assert abs(nrm.item() - float(ref @ ref)) <= 1e-12 * max(1.0, float(ref @ ref))
        _, nrm_ref = D.spmv(x, want_norm=True, reduction=1)
        assert nrm_ref.item() == port.dot(ref, ref)
        r = D.spmv(x, b=b)
        assert r.cpu().numpy().tobytes() == (b - ref).tobytes(), level
    return D


@pytest.mark.parametrize("kind,dims,pe", [(0, (9, 7, 5), 0.0), (1, (6, 6, 6), 1.0), (2, (5, 4, 6), 0.0),
                                          (0, (33, 17, 9), 0.0), (2, (21, 19, 11), 0.0)])
def test_stencils_bit_exact(cbg, port, kind, dims, pe):
    rp, ci, va = port.stencil(kind, *dims, pe=pe)
    D = check_paths(cbg, port, rp, ci, va, kind)
    no, nv, ne = D.info()
    assert no == {0: 7, 1: 7, 2: 27}[kind] and nv <= 7
    assert ne >= ci.size and ne % 32 == 0
    # constant-coefficient stencils on a box: one pattern per (x, y, z)
    # boundary class, 3^3 = 27 row patterns (+1: the all-padding rows that
    # fill the last 32-row slice), every offset with one value -> the
    # uniform-slot kernel (level 4) over the patterns
    if kind != 1:
        n = rp.size - 1
        assert D.layout() == (4, no, 27 + (n % 32 != 0))


def test_row_patterns_beyond_255_fall_back_to_pairs(cbg, port):
    """<= 255 pairs but more than 255 distinct rows: the pair-coded kernel."""
    rng = np.random.default_rng(11)
    n = 6000
    offsets = np.array([-40, -7, -3, -1, 0, 1, 2, 5, 9, 33])
    rp, ci, va = few_valued(rng, n, 8, offsets, np.array([1.5]), empty_frac=0.02)
    D = check_paths(cbg, port, rp, ci, va, 3)
    level, npairs, npat = D.layout()
    assert level == 2 and npairs == 10 and npat == 0


def test_row_patterns_without_uniform_slots(cbg, port):
    """Few row patterns whose offsets carry different values per pattern:
    the row-pattern kernel (level 3), not the uniform-slot one."""
    n = 4096
    rows = []
    for r in range(n):
        k = r % 3  # three row kinds: (-2, -1, 0, +1) with a per-kind value set
        vals = [(0.5, -1.0, 4.0, -1.0), (0.25, -2.0, 5.0, -0.5), (0.5, -1.0, 6.0, -1.0)][k]
        rows.append([(c, v) for c, v in zip((r - 2, r - 1, r, r + 1), vals) if 0 <= c < n])
    rp = np.zeros(n + 1, dtype=np.uint64)
    rp[1:] = np.cumsum([len(x) for x in rows])
    ci = np.array([c for x in rows for c, _ in x], dtype=np.uint64)
    va = np.array([v for x in rows for _, v in x])
    D = check_paths(cbg, port, rp, ci, va, 5)
    assert D.layout()[0] == 3


@pytest.mark.parametrize("nx,ny,pe,dec", [(10, 10, 1.0, 0.0), (37, 29, 3.0, 0.0), (8, 8, 1.0, 12.0)])
def test_convdiff_bit_exact(cbg, port, nx, ny, pe, dec):
    rp, ci, va = port.convdiff(nx, ny, pe, decades=dec)
    if dec:  # geometric row scaling: one value set per row, beyond the dictionary
        n = rp.size - 1
        A = cbg.DeviceCsr.from_host(cbg.CsrMatrix(n, n, rp, ci, va))
        if len(np.unique(va)) > 255:
            with pytest.raises(Exception):
                cbg.DictCsr(A)
            return
    check_paths(cbg, port, rp, ci, va, nx)


@pytest.mark.parametrize("n,max_len,nvals", [(1, 3, 2), (31, 5, 3), (33, 9, 200), (1000, 27, 255), (4099, 40, 17)])
def test_ragged_rows_bit_exact(cbg, port, n, max_len, nvals):
    rng = np.random.default_rng(n)
    offsets = np.unique(rng.integers(-3 * n, 3 * n + 1, size=60))
    values = rng.standard_normal(nvals)
    rp, ci, va = few_valued(rng, n, max_len, offsets, values)
    if ci.size == 0:
        pytest.skip("empty matrix")
    check_paths(cbg, port, rp, ci, va, n)


def test_refuses_outside_dictionary_limits(cbg):
    rng = np.random.default_rng(5)
    n = 2000
    # 256 distinct values
    rp = np.arange(n + 1, dtype=np.uint64)
    ci = np.arange(n, dtype=np.uint64)
    va = np.arange(n, dtype=np.float64) % 256 + 1.0
    A = cbg.DeviceCsr.from_host(cbg.CsrMatrix(n, n, rp, ci, va))
    with pytest.raises(Exception, match="255 distinct"):
        cbg.DictCsr(A)
    # 255 distinct values: accepted
    va2 = np.arange(n, dtype=np.float64) % 255 + 1.0
    D = cbg.DictCsr(cbg.DeviceCsr.from_host(cbg.CsrMatrix(n, n, rp, ci, va2)))
    assert D.info()[:2] == (1, 255)
    # 300 distinct column offsets
    ci3 = ((np.arange(n) + np.arange(n) % 300) % n).astype(np.uint64)
    A3 = cbg.DeviceCsr.from_host(cbg.CsrMatrix(n, n, rp, ci3, np.ones(n)))
    with pytest.raises(Exception, match="255 distinct"):
        cbg.DictCsr(A3)
    # random sparse matrix (many offsets): refused, solver keeps CSR
    rng = np.random.default_rng(1)
    lens = rng.integers(1, 8, size=n)
    rp4 = np.zeros(n + 1, dtype=np.uint64)
    rp4[1:] = np.cumsum(lens)
    ci4 = np.concatenate([np.sort(rng.choice(n, size=int(L), replace=False)) for L in lens]).astype(np.uint64)
    A4 = cbg.DeviceCsr.from_host(cbg.CsrMatrix(n, n, rp4, ci4, np.ones(ci4.size)))
    with pytest.raises(Exception):
        cbg.DictCsr(A4)


@pytest.mark.parametrize("fmt", ["frsz2-32", "frsz2-16", "f64"])
def test_solves_through_dictionary_match_csr(cbg, port, fmt):
    """Reference order: the dictionary path reproduces the oracle's history
    byte for byte; tree order: the same solve as the CSR paths (the SpMV is
    bit-identical; only the fused norm's reduction tree differs)."""
    rp, ci, va = port.stencil(1, 14, 13, 12, pe=1.0)
    b, _ = port.generate_problem(rp, ci, va)
    n = rp.size - 1

    def run(red, dict_spmv):
        cfg = cbg.GmresConfig(restart=30, storage_format=cbg.StorageFormat.parse(fmt), reduction=red,
                              dict_spmv=dict_spmv)
        return cbg.gmres_solve(cbg.CsrMatrix(n, n, rp, ci, va), b, np.zeros(n), cfg)

    o = port.gmres(rp, ci, va, b, fmt=fmt, restart=30)
    r = run(1, True)
    assert [(h.iteration, h.rrn, h.is_explicit) for h in r.residual_history] == o["history"]
    assert np.asarray(r.solution).tobytes() == o["x"].tobytes()
    t1, t0 = run(0, True), run(0, False)
    assert abs(t1.total_iterations - t0.total_iterations) <= 2
    assert t1.converged and t1.final_rrn <= 1e-10
    # both solves stop at RRN <= 1e-10: near-zero components may differ at that level
    x1, x0 = np.asarray(t1.solution), np.asarray(t0.solution)
    assert np.allclose(x1, x0, rtol=1e-7, atol=1e-9 * np.abs(x0).max())


@pytest.mark.parametrize("special", [np.inf, -np.inf, np.nan])
def test_nonfinite_x_matches_reference(cbg, port, special):
    """Padding codes gather x[r] * 0.0: a non-finite x[r] must not leak into
    rows whose real entries do not produce it (exact recompute path); rows
    that do reference it give the reference's result."""
    rp, ci, va = port.stencil(0, 9, 7, 5)
    n = rp.size - 1
    A = cbg.DeviceCsr.from_host(cbg.CsrMatrix(n, n, rp, ci, va))
    D = cbg.DictCsr(A)
    x = np.random.default_rng(3).standard_normal(n)
    x[[0, 17, n - 1]] = special  # boundary rows (padded) and an interior row
    ref = port.spmv(rp, ci, va, x)
    y = D.spmv(x).cpu().numpy()
    np.testing.assert_array_equal(np.isnan(y), np.isnan(ref))
    fin = ~np.isnan(ref)
    assert y[fin].tobytes() == ref[fin].tobytes()


def test_understated_row_length_hint_refused_or_exact(cbg, port):
    """cbgx.h documents max_row_nnz as a hint (0 = unknown): a hint below
    the longest row must not cut rows short (dsell.cu:427)."""
    rp, ci, va = port.stencil(0, 12, 11, 10)
    n = rp.size - 1
    A = cbg.DeviceCsr.from_host(cbg.CsrMatrix(n, n, rp, ci, va))
    A.desc.max_row_nnz = 2  # the real longest row has 7 entries
    try:
        D = cbg.DictCsr(A)
    except Exception as e:  # refused: the caller keeps CSR
        assert "max_row_nnz" in str(e)
        return
    x = np.random.default_rng(3).standard_normal(n)
    assert D.spmv(x).cpu().numpy().tobytes() == port.spmv(rp, ci, va, x).tobytes()


def test_tall_matrix_refused(cbg):
    """Padding codes gather x[r]: x must hold n_rows values (ADVICE r01:
    dsell.cu:293), so a matrix with n_cols < n_rows is refused."""
    n_rows, n_cols = 64, 40
    rp = np.arange(n_rows + 1, dtype=np.uint64)
    ci = (np.arange(n_rows) % n_cols).astype(np.uint64)
    va = np.ones(n_rows)
    A = cbg.DeviceCsr.from_host(cbg.CsrMatrix(n_rows, n_cols, rp, ci, va))
    with pytest.raises(Exception, match="n_cols >= n_rows"):
        cbg.DictCsr(A)


@pytest.mark.parametrize("offsets", [(-100, -10, -2, 0, 2, 10, 100), (-37, -1, 0, 1), (-5, -4, -3, 0, 3, 4, 5)])
def test_uniform_slots_without_triples(cbg, port, offsets):
    """Constant-coefficient band matrices whose offsets do not form the
    (o - 1, o, o + 1) triples of the shuffle path: the uniform-slot kernel
    gathers every slot, bit-exact (7 slots: the S = 7 kernel without
    shuffles; 4 slots: the generic S <= 8 one)."""
    n = 5000
    vals = {o: (4.0 if o == 0 else -1.0 / (1 + abs(o))) for o in offsets}
    rows = [[(r + o, vals[o]) for o in offsets if 0 <= r + o < n] for r in range(n)]
    rp = np.zeros(n + 1, dtype=np.uint64)
    rp[1:] = np.cumsum([len(x) for x in rows])
    ci = np.array([c for x in rows for c, _ in x], dtype=np.uint64)
    va = np.array([v for x in rows for _, v in x])
    D = check_paths(cbg, port, rp, ci, va, 9)
    assert D.layout()[0] == 4


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_uniform_slots_random_subsets(cbg, port, seed):
    """Every row takes a random subset of 8 offsets (one value per offset;
    dense enough for the ELL4 layout the pair codes need): ~100 row patterns
    over one slot list -> the uniform-slot kernel with arbitrary slot masks,
    row counts off the 32-row slices; non-finite x entries propagate exactly
    as in the reference."""
    rng = np.random.default_rng(seed)
    n = 3000 + 17 * seed
    offsets = np.array([-40, -31, -1, 0, 1, 2, 64, 90])
    vals = rng.standard_normal(offsets.size)
    rows = []
    for r in range(n):
        pick = rng.random(offsets.size) < 0.9
        rows.append([(r + o, v) for o, v, p in zip(offsets, vals, pick) if p and 0 <= r + o < n])
    rp = np.zeros(n + 1, dtype=np.uint64)
    rp[1:] = np.cumsum([len(x) for x in rows])
    ci = np.array([c for x in rows for c, _ in x], dtype=np.uint64)
    va = np.array([v for x in rows for _, v in x])
    D = check_paths(cbg, port, rp, ci, va, seed)
    level, _, npat = D.layout()
    assert level == 4 and npat > 32
    x = rng.standard_normal(n)
    x[rng.integers(0, n, 5)] = [np.inf, -np.inf, np.nan, np.inf, np.nan]
    ref = port.spmv(rp, ci, va, x)
    y = D.spmv(x).cpu().numpy()
    np.testing.assert_array_equal(np.isnan(y), np.isnan(ref))
    fin = ~np.isnan(ref)
    assert y[fin].tobytes() == ref[fin].tobytes()


def test_create2_rejects_unknown_level(cbg, port):
    rp, ci, va = port.stencil(0, 5, 5, 5)
    n = rp.size - 1
    A = cbg.DeviceCsr.from_host(cbg.CsrMatrix(n, n, rp, ci, va))
    with pytest.raises(Exception, match="max_level"):
        cbg.DictCsr(A, max_level=4)
