// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" bridge onto the UNMODIFIED reference library (the .cpp files
// under /root/reference/proj/src compiled in place by oracle/Makefile into
// oracle/_ref/libcbgref.so). It only calls the reference's public API
// (proj/include/cbg/*.hpp); nothing here re-implements reference logic.
// Used by tests (to pin oracle/cbg_oracle.c against the real reference) and
// by bench.py --impl reference (the reference CPU arm).
#include <cstdint>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "cbg/frsz2.hpp"
#include "cbg/gmres.hpp"
#include "cbg/half.hpp"
#include "cbg/sparse.hpp"

namespace {
thread_local std::string g_err;

cbg::CsrMatrix make_csr(size_t n, const uint64_t* rp, const uint64_t* ci,
                        const double* va) {
    cbg::CsrMatrix a;
    a.n_rows = a.n_cols = n;
    a.row_ptrs.assign(rp, rp + n + 1);
    a.col_idx.assign(ci, ci + rp[n]);
    a.values.assign(va, va + rp[n]);
    return a;
}

cbg::StorageFormat make_fmt(int fmt, uint32_t l) {
    switch (fmt) {
    case 0: return cbg::StorageFormat::f64();
    case 1: return cbg::StorageFormat::f32();
    case 2: return cbg::StorageFormat::f16();
    default: return cbg::StorageFormat::frsz2_format(l);
    }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// frsz2.hpp:70-71 compress; returns 2 + message on non-finite input
int ref_compress(const double* v, uint64_t n, uint32_t bs, uint32_t l,
                 uint32_t* exps, uint32_t* payload) {
    try {
        const auto cv = cbg::compress(std::span<const double>(v, n),
                                      cbg::Frsz2Params{bs, l});
        std::memcpy(exps, cv.exponents().data(), cv.exponents().size() * 4);
        std::memcpy(payload, cv.payload().data(), cv.payload().size() * 4);
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// container bytes of compress(v) (frsz2.hpp:84-85)
int ref_compress_container(const double* v, uint64_t n, uint32_t bs,
                           uint32_t l, uint8_t* out, uint64_t cap,
                           uint64_t* len) {
    try {
        const auto cv = cbg::compress(std::span<const double>(v, n),
                                      cbg::Frsz2Params{bs, l});
        std::ostringstream os;
        cbg::write_frsz2_file(os, cv);
        const std::string s = os.str();
        *len = s.size();
        if (s.size() > cap) return 1;
        std::memcpy(out, s.data(), s.size());
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// decompress from container bytes (frsz2.hpp:84-86)
int ref_decompress_container(const uint8_t* buf, uint64_t len, double* out) {
    try {
        std::istringstream is(std::string(reinterpret_cast<const char*>(buf), len));
        const auto cv = cbg::read_frsz2_file(is);
        cbg::decompress(cv, std::span<double>(out, cv.size()));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

uint16_t ref_half_from_double(double x) { return cbg::half_from_double(x); }
double ref_half_to_double(uint16_t h) { return cbg::half_to_double(h); }

void ref_spmv(uint64_t n, const uint64_t* rp, const uint64_t* ci,
              const double* va, const double* x, double* y) {
    const auto a = make_csr(n, rp, ci, va);
    const auto r = cbg::spmv(a, std::span<const double>(x, n));
    std::memcpy(y, r.data(), n * 8);
}

int ref_generate_problem(uint64_t n, const uint64_t* rp, const uint64_t* ci,
                         const double* va, double* b, double* x_sol) {
    try {
        const auto a = make_csr(n, rp, ci, va);
        auto [bb, xx] = cbg::generate_problem(a);
        std::memcpy(b, bb.data(), n * 8);
        std::memcpy(x_sol, xx.data(), n * 8);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

int ref_gen_convdiff(uint64_t nx, uint64_t ny, double pe, double decades,
                     uint64_t* rp, uint64_t* ci, double* va) {
    try {
        auto a = cbg::gen_convdiff(nx, ny, pe);
        if (decades != 0.0) cbg::rescale_rows_geometric(a, decades);
        std::memcpy(rp, a.row_ptrs.data(), a.row_ptrs.size() * 8);
        std::memcpy(ci, a.col_idx.data(), a.col_idx.size() * 8);
        std::memcpy(va, a.values.data(), a.values.size() * 8);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// gmres.hpp:69-75
int ref_arnoldi(int fmt, uint32_t l, uint64_t n, uint64_t cols,
                const double* colvals, double* w, double* h, double eta,
                double* out4) {
    try {
        cbg::KrylovBasis basis(n, cols ? cols : 1, make_fmt(fmt, l));
        for (uint64_t j = 0; j < cols; ++j)
            basis.write_vector(j, std::span<const double>(colvals + j * n, n));
        const auto r = cbg::arnoldi_orthogonalize(
            basis, cols, std::span<double>(w, n), std::span<double>(h, cols), eta);
        out4[0] = r.omega;
        out4[1] = r.h_next;
        out4[2] = r.reorthogonalized;
        out4[3] = r.breakdown;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// gmres.hpp:113-115. history arrays sized >= hist_cap.
int ref_gmres_solve(uint64_t n, const uint64_t* rp, const uint64_t* ci,
                    const double* va, const double* b, const double* x0,
                    uint64_t restart, double target, uint64_t max_it,
                    double eta, int fmt, uint32_t l, int* converged,
                    uint64_t* iters, uint64_t* restarts, double* final_rrn,
                    double* x_out, uint64_t* hist_iter, double* hist_rrn,
                    uint8_t* hist_explicit, uint64_t hist_cap,
                    uint64_t* hist_len, double* wall_seconds) {
    try {
        const auto a = make_csr(n, rp, ci, va);
        cbg::GmresConfig cfg;
        cfg.restart = restart;
        cfg.target_rrn = target;
        cfg.max_total_iterations = max_it;
        cfg.eta = eta;
        cfg.storage_format = make_fmt(fmt, l);
        const auto r = cbg::gmres_solve(a, std::span<const double>(b, n),
                                        std::span<const double>(x0, n), cfg);
        *converged = r.converged;
        *iters = r.total_iterations;
        *restarts = r.restarts;
        *final_rrn = r.final_rrn;
        *wall_seconds = r.wall_seconds;
        std::memcpy(x_out, r.solution.data(), n * 8);
        *hist_len = r.residual_history.size();
        for (size_t i = 0; i < r.residual_history.size() && i < hist_cap; ++i) {
            hist_iter[i] = r.residual_history[i].iteration;
            hist_rrn[i] = r.residual_history[i].rrn;
            hist_explicit[i] = r.residual_history[i].is_explicit;
        }
        return 0;
    } catch (const cbg::SolverBreakdown& e) {
        g_err = e.what();
        *iters = e.iteration;
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

}  // extern "C"
