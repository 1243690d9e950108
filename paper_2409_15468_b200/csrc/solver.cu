// solver.cu -- restarted CB-GMRES with the Krylov basis in FRSZ2 (or
// f64/f32/f16) on the device and the Hessenberg least squares on the host.
//
// Reference control flow: gmres_solve, gmres.cpp:141-252, and
// arnoldi_orthogonalize, gmres.cpp:36-71. Per Arnoldi step the device runs
//   spmv (+ fused ||w||^2 = omega^2)            gmres.cpp:210, :43
//   cgs_dot over all used+1 columns             gmres.cpp:44-46
//   cgs_update over all used+1 columns (+ fused ||w||^2 = h_next^2)  :47-50
// and one small device->host copy [h_next^2, omega^2, h_0..h_used] feeds the
// host-side re-orthogonalisation test, finite checks and Givens update.
// The next basis column (scale by 1/h_next fused into the compressor, which
// also emits the fp64 v for the next SpMV) is written from device scalars,
// so 1/sqrt is evaluated with IEEE sqrt/div exactly like the host's
// scale(1.0 / h_next, w) (gmres.cpp:231).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>

#include "basis.cuh"
#include "common.cuh"
#include "lsq.h"
#include "reduce.cuh"
#include "solver.h"

namespace cbgx {

void launch_spmv(const cbgx_csr& A, const double* x, const double* b, double* y, double* norm,
                 int reduction, Workspace* ws, cudaStream_t st);

namespace {

constexpr size_t kHn = 0;     // ||w||^2 after the update (h_next^2)
constexpr size_t kOmega = 1;  // ||w||^2 before orthogonalisation
constexpr size_t kH = 2;      // h[0..m]

struct BreakdownError : Error {
    BreakdownError(const std::string& m, uint64_t it) : Error(CBGX_EBREAKDOWN, m, it) {}
};

int fmt_from_cfg(const cbgx_gmres_config& c) {
    cbgx_basis tmp{};
    tmp.kind = c.format_kind;
    tmp.bit_length = c.bit_length;
    return fmt_of(tmp);
}

}  // namespace

// CUDA-event phase timing (device time per phase, summed over launches).
struct Solver::PhaseTimer {
    bool on = false;
    std::vector<cudaEvent_t> pool;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> marks;
    size_t next = 0;
    cudaStream_t st = nullptr;
    int open_phase = -1;
    cudaEvent_t open_ev = nullptr;
    cudaEvent_t ev() {
        if (next == pool.size()) {
            cudaEvent_t e;
            CBGX_CUDA(cudaEventCreate(&e));
            pool.push_back(e);
        }
        return pool[next++];
    }
    void begin(int phase) {
        if (!on) return;
        open_phase = phase;
        open_ev = ev();
        CBGX_CUDA(cudaEventRecord(open_ev, st));
    }
    void end() {
        if (!on || open_phase < 0) return;
        cudaEvent_t e = ev();
        CBGX_CUDA(cudaEventRecord(e, st));
        marks.push_back({open_phase, {open_ev, e}});
        open_phase = -1;
    }
    void collect(cbgx_solve_stats* s) {
        if (!on) return;
        CBGX_CUDA(cudaStreamSynchronize(st));
        for (auto& m : marks) {
            float ms = 0.f;
            CBGX_CUDA(cudaEventElapsedTime(&ms, m.second.first, m.second.second));
            s->phase_ms[m.first] += ms;
        }
        marks.clear();
        next = 0;
    }
    ~PhaseTimer() {
        for (auto e : pool) cudaEventDestroy(e);
    }
};

Solver::Solver(const cbgx_csr& A, const cbgx_gmres_config& cfg, Comm* comm, Halo* halo)
    : A_(A), cfg_(cfg), comm_(comm), halo_(halo), n_(A.n_rows) {
    if (cfg.restart < 1) throw Error(CBGX_EINVAL, "gmres: restart must be >= 1");
    if (!(cfg.target_rrn > 0.0)) throw Error(CBGX_EINVAL, "gmres: target_rrn must be > 0");
    if (!(cfg.eta > 0.0 && cfg.eta < 1.0)) throw Error(CBGX_EINVAL, "gmres: eta must be in (0, 1)");
    if (cfg.reduction != CBGX_REDUCE_TREE && cfg.reduction != CBGX_REDUCE_REFERENCE)
        throw Error(CBGX_EINVAL, "gmres: unknown reduction mode");
    if (cfg.reduction == CBGX_REDUCE_REFERENCE && comm && comm->size() > 1)
        throw Error(CBGX_EINVAL, "gmres: reference-order reductions need a single rank");
    if (!halo && A.n_rows != A.n_cols) throw Error(CBGX_EINVAL, "gmres: matrix must be square");
    (void)fmt_from_cfg(cfg);
    ws_.device = current_device();
    const uint64_t m = cfg.restart;
    uint64_t data_bytes = 0, exp_bytes = 0;
    const int st = cbgx_basis_layout(cfg.format_kind, cfg.bit_length, n_, m + 1, &V_, &data_bytes, &exp_bytes);
    if (st != CBGX_OK) throw Error(st, cbgx_last_error());
    CBGX_CUDA(cudaMalloc(&d_basis_, data_bytes));
    CBGX_CUDA(cudaMemset(d_basis_, 0, data_bytes));
    V_.d_data = d_basis_;
    if (exp_bytes) {
        CBGX_CUDA(cudaMalloc(&d_exp_, exp_bytes));
        CBGX_CUDA(cudaMemset(d_exp_, 0, exp_bytes));
    }
    V_.d_exp = d_exp_;
    const uint64_t ghosts = halo ? halo->n_ghost : 0;
    CBGX_CUDA(cudaMalloc(&d_r_, std::max<uint64_t>(n_, 1) * sizeof(double)));
    CBGX_CUDA(cudaMalloc(&d_v_, std::max<uint64_t>(n_ + ghosts, 1) * sizeof(double)));
    CBGX_CUDA(cudaMalloc(&d_w_, std::max<uint64_t>(n_, 1) * sizeof(double)));
    CBGX_CUDA(cudaMalloc(&d_scal_, (3 * m + 16) * sizeof(double)));
    CBGX_CUDA(cudaMallocHost(&h_pinned_, (3 * m + 16) * sizeof(double)));
}

Solver::~Solver() {
    cudaFree(d_basis_);
    cudaFree(d_exp_);
    cudaFree(d_r_);
    cudaFree(d_v_);
    cudaFree(d_w_);
    cudaFree(d_scal_);
    cudaFreeHost(h_pinned_);
}

void Solver::reduce(double* d_vals, size_t count, cudaStream_t st) {
    if (comm_ && comm_->size() > 1) comm_->sum_partials(d_vals, count, st);
}

double Solver::fetch_scalar(const double* d, cudaStream_t st) {
    CBGX_CUDA(cudaMemcpyAsync(h_pinned_, d, sizeof(double), cudaMemcpyDeviceToHost, st));
    CBGX_CUDA(cudaStreamSynchronize(st));
    return h_pinned_[0];
}

void Solver::solve(const double* d_b, const double* d_x0, double* d_x, cbgx_history* hist,
                   cbgx_solve_stats* stats, cudaStream_t st) {
    const auto t_start = std::chrono::steady_clock::now();
    cbgx_solve_stats S{};
    PhaseTimer timer;
    timer.on = (cfg_.flags & CBGX_SOLVER_PHASE_TIMING) != 0;
    timer.st = st;
    const int red = static_cast<int>(cfg_.reduction);
    const uint64_t m = cfg_.restart;
    const uint64_t n = n_;
    const int fmt = fmt_from_cfg(cfg_);
    const double bpv = stored_bytes_per_value(fmt);
    const double rp_bytes = A_.row_ptr_bits / 8.0;
    const double spmv_bytes = A_.nnz * 12.0 + (n + 1) * rp_bytes + 16.0 * n;
    uint64_t hist_len = 0;
    auto push = [&](uint64_t it, double rrn, bool ex) {
        if (hist && hist_len < hist->capacity) {
            if (hist->iteration) hist->iteration[hist_len] = it;
            if (hist->rrn) hist->rrn[hist_len] = rrn;
            if (hist->is_explicit) hist->is_explicit[hist_len] = ex ? 1 : 0;
        }
        ++hist_len;
    };
    auto count = [&](int phase, double bytes, uint64_t launches = 1) {
        S.phase_bytes[phase] += bytes;
        S.phase_launches[phase] += launches;
        S.kernel_launches += launches;
    };
    double* scal = d_scal_;
    double* h_u = scal + kH + m + 2;  // re-orthogonalisation coefficients u
    double* h_y = h_u + m + 2;        // least-squares solution y
    double* rn = h_y + m + 2;         // ||b||^2, then ||r||^2 at each restart
    double* hs = h_pinned_;

    // ||b|| (gmres.cpp:161)
    timer.begin(CBGX_PHASE_RESIDUAL);
    launch_dot(d_b, d_b, n, red, rn, &ws_, st);
    reduce(rn, 1, st);
    timer.end();
    count(CBGX_PHASE_RESIDUAL, 16.0 * n);
    const double norm_b = std::sqrt(fetch_scalar(rn, st));
    if (norm_b == 0.0) {
        CBGX_CUDA(cudaMemsetAsync(d_x, 0, n * sizeof(double), st));
        push(0, 0.0, true);
        S.converged = 1;
        S.final_rrn = 0.0;
    } else {
        if (d_x != d_x0) CBGX_CUDA(cudaMemcpyAsync(d_x, d_x0, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
        GivensLsq lsq(m);
        std::vector<double> hcol(m + 2), y(m);
        uint64_t iter = 0, cycles = 0;
        double last = 0.0;
        for (;;) {
            // Explicit residual r = b - A x (gmres.cpp:181-190).
            timer.begin(CBGX_PHASE_RESIDUAL);
            const double* xin = d_x;
            if (halo_) {
                CBGX_CUDA(cudaMemcpyAsync(d_v_, d_x, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
                halo_->exchange(d_v_, st);
                xin = d_v_;
            }
            launch_spmv(A_, xin, d_b, d_r_, rn, red, &ws_, st);
            reduce(rn, 1, st);
            timer.end();
            count(CBGX_PHASE_RESIDUAL, spmv_bytes + 8.0 * n);
            const double beta = std::sqrt(fetch_scalar(rn, st));
            const double explicit_rrn = beta / norm_b;
            if (!std::isfinite(explicit_rrn)) throw BreakdownError("gmres: non-finite residual", iter);
            push(iter, explicit_rrn, true);
            last = explicit_rrn;
            if (explicit_rrn <= cfg_.target_rrn) {
                S.converged = 1;
                break;
            }
            if (iter >= cfg_.max_total_iterations) {
                S.converged = 0;
                break;
            }
            ++cycles;
            lsq.reset(beta);
            // v = r * (1/beta); column 0 (gmres.cpp:201-204)
            timer.begin(CBGX_PHASE_WRITE);
            launch_basis_write(V_, 0, d_r_, rn, 1, d_v_, nullptr, st);
            timer.end();
            count(CBGX_PHASE_WRITE, 16.0 * n + bpv * n);

            uint64_t used = 0;
            bool cycle_done = false;
            while (!cycle_done && used < m && iter < cfg_.max_total_iterations) {
                ++iter;
                const uint32_t cols = static_cast<uint32_t>(used + 1);
                // w = A v, omega^2 fused (gmres.cpp:210, :43)
                if (halo_) {
                    timer.begin(CBGX_PHASE_COMM);
                    halo_->exchange(d_v_, st);
                    timer.end();
                }
                timer.begin(CBGX_PHASE_SPMV);
                launch_spmv(A_, d_v_, nullptr, d_w_, scal + kOmega, red, &ws_, st);
                timer.end();
                count(CBGX_PHASE_SPMV, spmv_bytes);
                // h = V^T w (gmres.cpp:44-46)
                timer.begin(CBGX_PHASE_DOT);
                launch_cgs_dot(V_, 0, cols, d_w_, 0, red, scal + kH, &ws_, st);
                timer.end();
                count(CBGX_PHASE_DOT, cols * bpv * n + 8.0 * n);
                if (comm_ && comm_->size() > 1) {
                    timer.begin(CBGX_PHASE_COMM);
                    reduce(scal + kOmega, cols + 1, st);
                    timer.end();
                }
                // w -= V h, h_next^2 fused (gmres.cpp:47-50)
                timer.begin(CBGX_PHASE_UPDATE);
                launch_cgs_update(V_, 0, cols, scal + kH, 1.0, d_w_, scal + kHn, red, &ws_, st);
                timer.end();
                count(CBGX_PHASE_UPDATE, cols * bpv * n + 16.0 * n);
                if (comm_ && comm_->size() > 1) {
                    timer.begin(CBGX_PHASE_COMM);
                    reduce(scal + kHn, 1, st);
                    timer.end();
                }
                CBGX_CUDA(cudaMemcpyAsync(hs, scal, (kH + cols) * sizeof(double), cudaMemcpyDeviceToHost, st));
                CBGX_CUDA(cudaStreamSynchronize(st));
                const double omega = std::sqrt(hs[kOmega]);
                double h_next = std::sqrt(hs[kHn]);
                for (uint64_t i = 0; i < cols; ++i) hcol[i] = hs[kH + i];
                bool breakdown = false;
                if (h_next < cfg_.eta * omega) {
                    // one re-orthogonalisation pass (gmres.cpp:53-68)
                    ++S.reorth_passes;
                    const double before = h_next;
                    timer.begin(CBGX_PHASE_DOT);
                    launch_cgs_dot(V_, 0, cols, d_w_, 0, red, h_u, &ws_, st);
                    reduce(h_u, cols, st);
                    timer.end();
                    count(CBGX_PHASE_DOT, cols * bpv * n + 8.0 * n);
                    timer.begin(CBGX_PHASE_UPDATE);
                    launch_cgs_update(V_, 0, cols, h_u, 1.0, d_w_, scal + kHn, red, &ws_, st);
                    reduce(scal + kHn, 1, st);
                    timer.end();
                    count(CBGX_PHASE_UPDATE, cols * bpv * n + 16.0 * n);
                    CBGX_CUDA(cudaMemcpyAsync(hs + kH + m + 2, h_u, cols * sizeof(double), cudaMemcpyDeviceToHost, st));
                    CBGX_CUDA(cudaMemcpyAsync(hs + kHn, scal + kHn, sizeof(double), cudaMemcpyDeviceToHost, st));
                    CBGX_CUDA(cudaStreamSynchronize(st));
                    for (uint64_t i = 0; i < cols; ++i) hcol[i] += hs[kH + m + 2 + i];
                    h_next = std::sqrt(hs[kHn]);
                    breakdown = h_next < cfg_.eta * before;
                }
                breakdown = breakdown || h_next == 0.0;
                if (!std::isfinite(omega) || !std::isfinite(h_next))
                    throw BreakdownError("gmres: non-finite Arnoldi step", iter);
                hcol[used + 1] = h_next;
                for (uint64_t i = 0; i <= used + 1; ++i)
                    if (!std::isfinite(hcol[i])) throw BreakdownError("gmres: non-finite Hessenberg entry", iter);
                double estimate = 0.0;
                lsq.add_column(hcol.data(), used + 2, &estimate);
                ++used;
                const double implicit_rrn = estimate / norm_b;
                if (!breakdown) {
                    // v = w / h_next; column `used` (gmres.cpp:230-234)
                    timer.begin(CBGX_PHASE_WRITE);
                    launch_basis_write(V_, used, d_w_, scal + kHn, 1, d_v_, nullptr, st);
                    timer.end();
                    count(CBGX_PHASE_WRITE, 16.0 * n + bpv * n);
                }
                cycle_done = breakdown || implicit_rrn <= cfg_.target_rrn || used == m ||
                             iter >= cfg_.max_total_iterations;
                if (!cycle_done) push(iter, implicit_rrn, false);
            }
            // x += V y (gmres.cpp:242-243, :134-139)
            const long bad = lsq.solve_y(y.data());
            if (bad >= 0) throw BreakdownError("gmres: singular triangular factor", static_cast<uint64_t>(bad));
            timer.begin(CBGX_PHASE_SOLUTION);
            std::memcpy(hs, y.data(), used * sizeof(double));
            CBGX_CUDA(cudaMemcpyAsync(h_y, hs, used * sizeof(double), cudaMemcpyHostToDevice, st));
            launch_cgs_update(V_, 0, static_cast<uint32_t>(used), h_y, -1.0, d_x, nullptr, red, &ws_, st);
            timer.end();
            count(CBGX_PHASE_SOLUTION, used * bpv * n + 16.0 * n);
            // The H2D above reads the pinned buffer asynchronously; the next
            // fetch synchronises before it is reused.
        }
        S.total_iterations = iter;
        S.restarts = cycles > 0 ? cycles - 1 : 0;
        S.final_rrn = last;
    }
    CBGX_CUDA(cudaStreamSynchronize(st));
    timer.collect(&S);
    S.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    if (hist) hist->length = hist_len;
    if (stats) *stats = S;
}

}  // namespace cbgx

using namespace cbgx;

namespace {

cbgx_gmres_config checked(const cbgx_gmres_config* cfg) {
    if (!cfg) throw Error(CBGX_EINVAL, "gmres: null config");
    return *cfg;
}

}  // namespace

extern "C" {

int cbgx_solver_create(const cbgx_csr* A, const cbgx_gmres_config* cfg, cbgx_comm* comm,
                       cbgx_solver** out) {
    return guard([&] {
        if (!A || !out) throw Error(CBGX_EINVAL, "solver: null argument");
        if (comm) throw Error(CBGX_EINVAL, "solver: use cbgx_solver_create_dist for a communicator");
        auto* h = new SolverHandle();
        try {
            h->solver = std::make_unique<Solver>(*A, checked(cfg), nullptr, nullptr);
        } catch (...) {
            delete h;
            throw;
        }
        *out = reinterpret_cast<cbgx_solver*>(h);
    });
}

int cbgx_solver_destroy(cbgx_solver* s) {
    return guard([&] { delete reinterpret_cast<SolverHandle*>(s); });
}

int cbgx_solver_solve(cbgx_solver* s, const double* d_b, const double* d_x0, double* d_x,
                      cbgx_history* hist, cbgx_solve_stats* stats, void* stream) {
    return guard([&] {
        if (!s) throw Error(CBGX_EINVAL, "solver: null handle");
        reinterpret_cast<SolverHandle*>(s)->solver->solve(d_b, d_x0, d_x, hist, stats, as_stream(stream));
    });
}

int cbgx_gmres_solve_host(uint64_t n, const uint64_t* row_ptrs, const uint64_t* col_idx,
                          const double* values, const double* b, const double* x0,
                          const cbgx_gmres_config* cfg, double* x_out, cbgx_history* hist,
                          cbgx_solve_stats* stats) {
    return guard([&] {
        const cbgx_gmres_config c = checked(cfg);
        if (n > 0x7FFFFFFFull) throw Error(CBGX_EINVAL, "gmres: n must fit int32 column indices");
        const uint64_t nnz = row_ptrs[n];
        const bool wide = nnz > 0x7FFFFFFFull;
        std::vector<int32_t> ci(nnz);
        for (uint64_t k = 0; k < nnz; ++k) {
            if (col_idx[k] >= n) throw Error(CBGX_EINVAL, "csr: column index out of range");
            ci[k] = static_cast<int32_t>(col_idx[k]);
        }
        std::vector<int32_t> rp32;
        if (!wide) {
            rp32.resize(n + 1);
            for (uint64_t r = 0; r <= n; ++r) rp32[r] = static_cast<int32_t>(row_ptrs[r]);
        }
        cudaStream_t st = nullptr;
        void* d_rp = nullptr;
        int32_t* d_ci = nullptr;
        double *d_va = nullptr, *d_b = nullptr, *d_x0 = nullptr, *d_x = nullptr;
        auto cleanup = [&] {
            cudaFree(d_rp); cudaFree(d_ci); cudaFree(d_va); cudaFree(d_b); cudaFree(d_x0); cudaFree(d_x);
        };
        try {
            const size_t rpb = wide ? 8 : 4;
            CBGX_CUDA(cudaMalloc(&d_rp, (n + 1) * rpb));
            CBGX_CUDA(cudaMalloc(&d_ci, std::max<uint64_t>(nnz, 1) * 4));
            CBGX_CUDA(cudaMalloc(&d_va, std::max<uint64_t>(nnz, 1) * 8));
            CBGX_CUDA(cudaMalloc(&d_b, std::max<uint64_t>(n, 1) * 8));
            CBGX_CUDA(cudaMalloc(&d_x0, std::max<uint64_t>(n, 1) * 8));
            CBGX_CUDA(cudaMalloc(&d_x, std::max<uint64_t>(n, 1) * 8));
            CBGX_CUDA(cudaMemcpy(d_rp, wide ? static_cast<const void*>(row_ptrs) : static_cast<const void*>(rp32.data()),
                                 (n + 1) * rpb, cudaMemcpyHostToDevice));
            CBGX_CUDA(cudaMemcpy(d_ci, ci.data(), nnz * 4, cudaMemcpyHostToDevice));
            CBGX_CUDA(cudaMemcpy(d_va, values, nnz * 8, cudaMemcpyHostToDevice));
            CBGX_CUDA(cudaMemcpy(d_b, b, n * 8, cudaMemcpyHostToDevice));
            CBGX_CUDA(cudaMemcpy(d_x0, x0, n * 8, cudaMemcpyHostToDevice));
            cbgx_csr A{n, n, nnz, d_rp, wide ? 64u : 32u, d_ci, d_va};
            Solver solver(A, c, nullptr, nullptr);
            solver.solve(d_b, d_x0, d_x, hist, stats, st);
            CBGX_CUDA(cudaMemcpy(x_out, d_x, n * 8, cudaMemcpyDeviceToHost));
        } catch (...) {
            cleanup();
            throw;
        }
        cleanup();
    });
}

}  // extern "C"
