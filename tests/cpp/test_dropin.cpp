// test_dropin.cpp -- the reference's own test cases (test_frsz2.cpp,
// test_basis.cpp, test_gmres.cpp, acceptance.cpp) restated against the
// drop-in C++ API (include/cbg/*.hpp -> libcbg_b200.so -> libcbgx.so on the
// GPU). Built and run by tests/test_dropin_gpu.py. Prints one line per
// check group and exits non-zero on any failure.
#include <algorithm>
#include <bit>
#include <cmath>
#include <cstdio>
#include <limits>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "cbg/bench.hpp"
#include "cbg/frsz2.hpp"
#include "cbg/gmres.hpp"

using namespace cbg;

static int g_fail = 0;
#define CHECK(c)                                                          \
    do {                                                                  \
        if (!(c)) {                                                       \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);      \
            ++g_fail;                                                     \
        }                                                                 \
    } while (0)

template <class E, class F>
static bool throws(F&& f, const char* msg = nullptr) {
    try {
        f();
    } catch (const E& e) {
        return msg == nullptr || std::string(e.what()) == msg;
    } catch (...) {
        return false;
    }
    return false;
}

static std::vector<double> uniform(size_t n, uint64_t seed, double lo = -1.0, double hi = 1.0) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> d(lo, hi);
    std::vector<double> v(n);
    for (double& x : v) x = d(rng);
    return v;
}

static bool same(double a, double b) { return std::bit_cast<uint64_t>(a) == std::bit_cast<uint64_t>(b); }

static void codec() {
    // test_frsz2.cpp:37-75
    const std::vector<double> v4 = {1.0, 0.5, 0.0, -0.25};
    const BlockEncoding enc = compress_block(v4, 32);
    CHECK(enc.e_max == 1023);
    CHECK(enc.codes.size() == 4 && enc.codes[0] == 0x40000000u && enc.codes[1] == 0x20000000u &&
          enc.codes[2] == 0 && enc.codes[3] == 0x90000000u);
    CHECK(compress_block(std::vector<double>{0.0, 0.0}, 32).e_max == 0);
    std::vector<double> bad = {1.0, 2.0, std::numeric_limits<double>::infinity(), 0.5};
    CHECK(throws<std::invalid_argument>([&] { compress_block(bad, 16); }, "frsz2: non-finite value at index 2"));
    CHECK(throws<std::invalid_argument>([&] { compress(bad, Frsz2Params{32, 32}); },
                                        "frsz2: non-finite value at index 2"));
    // sizes (:77-96), storage (:299-305), bound (:307-313)
    CHECK(compress({}, Frsz2Params{32, 32}).exponents().empty());
    CHECK(compress(uniform(33, 1), Frsz2Params{32, 32}).payload().size() == 64);
    CHECK(compress(uniform(32, 2), Frsz2Params{32, 21}).payload().size() == 21);
    CHECK(storage_bytes(64, Frsz2Params{32, 32}) == 264);
    CHECK(storage_bytes(32, Frsz2Params{32, 21}) == 88);
    CHECK(max_abs_error_bound(1023, 32) == 0x1p-30);
    CHECK(throws<std::invalid_argument>([] { compress({}, Frsz2Params{0, 32}); }));
    CHECK(throws<std::invalid_argument>([] { compress({}, Frsz2Params{32, 65}); }));
    // element / block agreement and round trips (:98-173)
    for (uint32_t l : {16u, 21u, 32u, 7u, 50u}) {
        const auto v = uniform(100, 100 + l);
        const CompressedVector cv = compress(v, Frsz2Params{32, l});
        std::vector<double> buf(32);
        for (size_t b = 0; b < cv.num_blocks(); ++b) {
            decompress_block(cv, b, buf);
            for (size_t r = 0; r < 32 && b * 32 + r < cv.size(); ++r) CHECK(same(buf[r], decompress_value(cv, b * 32 + r)));
        }
        CHECK(throws<std::out_of_range>([&] { decompress_block(cv, cv.num_blocks(), buf); }));
    }
    for (uint32_t l : {2u, 16u, 21u, 32u, 47u, 64u}) {
        const auto v = uniform(257, 7000 + l, -100.0, 100.0);
        const CompressedVector cv = compress(v, Frsz2Params{32, l});
        const CompressedVector cv2 = compress(decompress(cv), Frsz2Params{32, l});
        CHECK(std::equal(cv.exponents().begin(), cv.exponents().end(), cv2.exponents().begin()));
        CHECK(std::equal(cv.payload().begin(), cv.payload().end(), cv2.payload().begin()));
    }
    {
        const auto back = decompress(compress(std::vector<double>{-0.0, 0.0, 1.0, -1.0}, Frsz2Params{4, 16}));
        CHECK(std::signbit(back[0]) && back[0] == 0.0 && !std::signbit(back[1]));
        const auto sub = decompress(compress(std::vector<double>{5e-320, -5e-320, 1.0, 2.0}, Frsz2Params{4, 32}));
        CHECK(sub[0] == 0.0 && std::signbit(sub[1]) && sub[2] == 1.0);
    }
    // container golden bytes (acceptance.cpp:152-186)
    static const unsigned char golden[] = {'F', 'R', 'S', 'Z', '2', 0, 1, 0, 4, 0, 0, 0, 0x20, 0, 0, 0,
                                           4, 0, 0, 0, 0, 0, 0, 0, 0xFF, 3, 0, 0, 0, 0, 0, 0x40,
                                           0, 0, 0, 0x20, 0, 0, 0, 0, 0, 0, 0, 0x90};
    std::ostringstream os;
    write_frsz2_file(os, compress(v4, Frsz2Params{4, 32}));
    const std::string bytes = os.str();
    CHECK(bytes.size() == sizeof(golden) && std::equal(bytes.begin(), bytes.end(), reinterpret_cast<const char*>(golden)));
    std::istringstream is(bytes);
    const auto back = decompress(read_frsz2_file(is));
    CHECK(back == v4);
    std::istringstream badmagic("NOTFRSZ2 whatever");
    CHECK(throws<std::runtime_error>([&] { read_frsz2_file(badmagic); }, "frsz2 container: bad magic"));
    std::printf("codec: done\n");
}

static void basis() {
    // test_basis.cpp:42-214
    CHECK(StorageFormat::parse("frsz2-21")->frsz2.bit_length == 21);
    CHECK(!StorageFormat::parse("fp64").has_value());
    CHECK(throws<std::invalid_argument>([] { StorageFormat::frsz2_format(24); }));
    for (const char* name : {"f64", "f32", "f16", "frsz2-16", "frsz2-21", "frsz2-32"}) {
        const StorageFormat fmt = *StorageFormat::parse(name);
        const size_t n = 77;
        const auto v = uniform(n, 6);
        KrylovBasis b(n, 2, fmt);
        b.write_vector(0, v);
        std::vector<double> buf(32);
        for (size_t blk = 0; blk < b.num_blocks(); ++blk) {
            b.read_block(0, blk, buf);
            for (size_t r = 0; r < 32; ++r) {
                const size_t i = blk * 32 + r;
                if (i < n) CHECK(same(buf[r], b.read_element(0, i)));
                else CHECK(buf[r] == 0.0);
            }
        }
        CHECK(throws<std::out_of_range>([&] { b.read_block(0, b.num_blocks(), buf); }));
        CHECK(throws<std::out_of_range>([&] { b.read_block(1, 0, buf); }));
    }
    {
        KrylovBasis b(4, 1, StorageFormat::f16());
        b.write_vector(0, std::vector<double>{1e9, -1e9, 65504.0, 0.25});
        CHECK(b.read_element(0, 0) == 65504.0 && b.read_element(0, 1) == -65504.0 && b.read_element(0, 3) == 0.25);
    }
    {
        KrylovBasis b(32, 2, StorageFormat::f64());
        const auto v = uniform(32, 4);
        CHECK(throws<std::out_of_range>([&] { b.write_vector(1, v); }));
        b.write_vector(0, v);
        b.write_vector(1, v);
        CHECK(throws<std::out_of_range>([&] { b.write_vector(2, v); }));
        CHECK(throws<std::invalid_argument>([&] { b.write_vector(0, uniform(31, 5)); }));
        KrylovBasis fb(4, 1, StorageFormat::frsz2_format(16));
        CHECK(throws<std::invalid_argument>([&] { fb.write_vector(0, std::vector<double>{1.0, std::nan(""), 0.0, 0.0}); }));
    }
    for (const char* name : {"f64", "f32", "frsz2-32"}) {
        const size_t n = 1000;
        KrylovBasis b(n, 2, *StorageFormat::parse(name));
        const auto col = uniform(n, 7);
        b.write_vector(0, col);
        std::vector<double> dec(n);
        for (size_t i = 0; i < n; ++i) dec[i] = b.read_element(0, i);
        const auto w = uniform(n, 8);
        double s = 0.0, c = 0.0;  // Kahan (oracle_utils.hpp:20-28)
        for (size_t i = 0; i < n; ++i) {
            const double t = dec[i] * w[i] - c, u = s + t;
            c = (u - s) - t;
            s = u;
        }
        CHECK(std::abs(b.dot(0, w) - s) <= std::abs(s) * 0x1p-40 + 0x1p-48);
        auto y = col;
        KrylovBasis f(n, 1, StorageFormat::f64());
        f.write_vector(0, col);
        f.subtract_scaled(0, 1.0, y);
        CHECK(std::all_of(y.begin(), y.end(), [](double x) { return x == 0.0; }));
    }
    std::printf("basis: done\n");
}

static CsrMatrix diag(const std::vector<double>& d) {
    CsrMatrix a;
    a.n_rows = a.n_cols = d.size();
    a.row_ptrs.resize(d.size() + 1);
    for (size_t i = 0; i < d.size(); ++i) {
        a.row_ptrs[i + 1] = i + 1;
        a.col_idx.push_back(i);
        a.values.push_back(d[i]);
    }
    return a;
}

static void solver() {
    // test_gmres.cpp:84-142 hand cases of the host Givens
    {
        HessenbergLsq lsq(4);
        lsq.reset(4.0);
        std::vector<double> col = {2.0, 0.0};
        CHECK(lsq.add_column(col) == 0.0);
        std::vector<double> y(1);
        lsq.solve_y(y);
        CHECK(y[0] == 2.0);
        HessenbergLsq z(4);
        z.reset(1.0);
        std::vector<double> zc = {0.0, 0.0};
        CHECK(z.add_column(zc) == 0.0);
        std::vector<double> zy(1);
        CHECK(throws<SolverBreakdown>([&] { z.solve_y(zy); }));
    }
    // arnoldi hand case (test_gmres.cpp:144-167)
    {
        KrylovBasis b(3, 2, StorageFormat::f64());
        b.write_vector(0, std::vector<double>{1.0, 0.0, 0.0});
        std::vector<double> w = {1.0, 1.0, 0.0}, h(1);
        const auto r = arnoldi_orthogonalize(b, 1, w, h, 0.5);
        CHECK(h[0] == 1.0 && w[0] == 0.0 && w[1] == 1.0 && r.h_next == 1.0 && !r.reorthogonalized && !r.breakdown);
    }
    // identity / diag / zero rhs / cap / overflow (test_gmres.cpp:236-299)
    {
        const auto b = uniform(5, 30);
        GmresConfig cfg;
        cfg.target_rrn = 1e-12;
        const auto r = gmres_solve(diag(std::vector<double>(5, 1.0)), b, std::vector<double>(5, 0.0), cfg);
        CHECK(r.converged && r.total_iterations == 1 && r.final_rrn <= 1e-14);
        const auto r4 = gmres_solve(diag({1, 2, 3, 4}), std::vector<double>(4, 1.0), std::vector<double>(4, 0.0), cfg);
        CHECK(r4.converged && r4.total_iterations <= 4);
        const auto r0 = gmres_solve(diag({1, 2}), std::vector<double>(2, 0.0), std::vector<double>(2, 0.0), {});
        CHECK(r0.converged && r0.total_iterations == 0 && r0.final_rrn == 0.0);
        const CsrMatrix a = gen_convdiff(10, 10, 1.0);
        const auto [bb, xs] = generate_problem(a);
        GmresConfig capc;
        capc.target_rrn = 1e-12;
        capc.max_total_iterations = 5;
        const auto rc = gmres_solve(a, bb, std::vector<double>(a.n_cols, 0.0), capc);
        CHECK(!rc.converged && rc.total_iterations == 5 && rc.residual_history.back().is_explicit);
        CsrMatrix o;
        o.n_rows = o.n_cols = 2;
        o.row_ptrs = {0, 2, 4};
        o.col_idx = {0, 1, 0, 1};
        o.values = {1.5e308, -1.5e308, -1.5e308, 1.5e308};
        CHECK(throws<SolverBreakdown>([&] { gmres_solve(o, std::vector<double>{1.0, -1.0}, std::vector<double>(2, 0.0), {}); }));
    }
    // acceptance.cpp:278-312 criterion 7 in reference reduction order: the
    // pinned counts, exactly
    {
        const CsrMatrix a = gen_convdiff(100, 100, 1.0);
        const auto [b, xs] = generate_problem(a);
        GmresConfig cfg;
        cfg.reduction = GmresConfig::Reduction::reference;
        size_t its[3];
        int k = 0;
        for (const auto& fmt : {StorageFormat::f64(), StorageFormat::frsz2_format(32), StorageFormat::f32()}) {
            cfg.storage_format = fmt;
            const auto r = gmres_solve(a, b, std::vector<double>(a.n_cols, 0.0), cfg);
            CHECK(r.converged);
            its[k++] = r.total_iterations;
        }
        std::printf("criterion 7 (reference order): f64=%zu frsz2-32=%zu f32=%zu\n", its[0], its[1], its[2]);
        CHECK(its[0] == 626 && its[1] == 627 && its[2] == 658);
    }
    // criterion 8: f16 fails, frsz2-32 succeeds on the rescaled instance
    {
        CsrMatrix a = gen_convdiff(8, 8, 1.0);
        rescale_rows_geometric(a, 12.0);
        const auto [b, xs] = generate_problem(a);
        GmresConfig cfg;
        cfg.storage_format = StorageFormat::frsz2_format(32);
        const auto rz = gmres_solve(a, b, std::vector<double>(a.n_cols, 0.0), cfg);
        cfg.storage_format = StorageFormat::f16();
        cfg.max_total_iterations = 3000;
        const auto rh = gmres_solve(a, b, std::vector<double>(a.n_cols, 0.0), cfg);
        CHECK(rz.converged && !rh.converged);
    }
    // determinism (test_gmres.cpp:348-369) on the fast path
    {
        const CsrMatrix a = gen_convdiff(15, 15, 1.0);
        const auto [b, xs] = generate_problem(a);
        GmresConfig cfg;
        cfg.storage_format = StorageFormat::frsz2_format(32);
        const auto r1 = gmres_solve(a, b, std::vector<double>(a.n_cols, 0.0), cfg);
        const auto r2 = gmres_solve(a, b, std::vector<double>(a.n_cols, 0.0), cfg);
        CHECK(r1.residual_history.size() == r2.residual_history.size());
        for (size_t i = 0; i < r1.residual_history.size(); ++i) CHECK(same(r1.residual_history[i].rrn, r2.residual_history[i].rrn));
        for (size_t i = 0; i < r1.solution.size(); ++i) CHECK(same(r1.solution[i], r2.solution[i]));
    }
    std::printf("solver: done\n");
}

// MatrixMarket I/O (test_sparsela.cpp:136-208 restated).
static void matrix_market() {
    {
        std::istringstream mm("%%MatrixMarket matrix coordinate real general\n% a comment\n2 2 3\n1 1 2.0\n2 1 1.0\n2 2 3.0\n");
        const CsrMatrix a = parse_matrix_market(mm);
        a.validate();
        CHECK(a.n_rows == 2 && a.nnz() == 3);
        const auto y = spmv(a, std::vector<double>{1.0, 1.0});
        CHECK(y[0] == 2.0 && y[1] == 4.0);
    }
    {
        std::istringstream mm("%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n2 1 5.0\n2 2 1.0\n");
        const CsrMatrix a = parse_matrix_market(mm);
        a.validate();
        CHECK(a.nnz() == 3);
        CHECK(a.col_idx[0] == 1 && a.values[0] == 5.0 && a.col_idx[1] == 0 && a.values[1] == 5.0);
        std::istringstream dup("%%MatrixMarket matrix coordinate real general\n1 1 2\n1 1 2.0\n1 1 0.5\n");
        const CsrMatrix b = parse_matrix_market(dup);
        CHECK(b.nnz() == 1 && b.values[0] == 2.5);
    }
    {
        std::istringstream h("%%MatrixMarket matrix array real general\n");
        CHECK(throws<std::runtime_error>([&] { parse_matrix_market(h); },
                                         "matrix market: line 1: only 'matrix coordinate' files are supported"));
        std::istringstream pat("%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 1\n");
        CHECK(throws<std::runtime_error>([&] { parse_matrix_market(pat); }));
        std::istringstream cx("%%MatrixMarket matrix coordinate complex general\n2 2 1\n1 1 1 0\n");
        CHECK(throws<std::runtime_error>([&] { parse_matrix_market(cx); }));
        std::istringstream oob("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n");
        CHECK(throws<std::runtime_error>([&] { parse_matrix_market(oob); }, "matrix market: line 3: index out of bounds"));
        std::istringstream bad("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 abc\n");
        CHECK(throws<std::runtime_error>([&] { parse_matrix_market(bad); }));
    }
    {
        const CsrMatrix a = gen_convdiff(7, 6, 1.0);
        std::stringstream ss;
        write_matrix_market(ss, a);
        const CsrMatrix b = parse_matrix_market(ss);
        CHECK(a.n_rows == b.n_rows && a.n_cols == b.n_cols && a.nnz() == b.nnz());
        CHECK(a.row_ptrs == b.row_ptrs && a.col_idx == b.col_idx);
        for (size_t k = 0; k < a.nnz() && k < b.nnz(); ++k) CHECK(same(a.values[k], b.values[k]));
    }
    std::printf("matrix market: done\n");
}

// run_read_benchmark (bench.hpp; bench.cpp:100-152 argument checks and
// result shape) on the device read sweep.
static void bench() {
    const std::vector<StorageFormat> fmts = {StorageFormat::f64(), StorageFormat::frsz2_format(32),
                                             StorageFormat::frsz2_format(16)};
    const std::vector<int> ints = {1, 3};
    const auto res = run_read_benchmark(1000, fmts, ints, 2, 7);
    CHECK(res.size() == 6);
    for (size_t i = 0; i < res.size(); ++i) {
        CHECK(res[i].format == fmts[i / 2].name());
        CHECK(res[i].intensity == ints[i % 2]);
        CHECK(res[i].elements == 992);
        CHECK(res[i].stored_bytes == fmts[i / 2].column_bytes(992));
        CHECK(res[i].seconds > 0.0 && res[i].stored_gbps > 0.0 && res[i].logical_gbps > 0.0);
    }
    CHECK(throws<std::invalid_argument>([&] { run_read_benchmark(31, fmts, ints, 2, 7); }));
    CHECK(throws<std::invalid_argument>([&] { run_read_benchmark(64, fmts, ints, 0, 7); }));
    const std::vector<int> bad = {0};
    CHECK(throws<std::invalid_argument>([&] { run_read_benchmark(64, fmts, bad, 1, 7); }));
    std::printf("bench: done\n");
}

int main() {
    codec();
    basis();
    solver();
    matrix_market();
    bench();
    std::printf(g_fail ? "%d check(s) failed\n" : "all drop-in checks passed\n", g_fail);
    return g_fail ? 1 : 0;
}
