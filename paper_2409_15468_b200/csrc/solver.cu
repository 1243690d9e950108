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
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>

#include "basis.cuh"
#include "common.cuh"
#include "lsq.h"
#include "reduce.cuh"
#include "solver.h"

namespace cbgx {

void launch_spmv(const cbgx_csr& A, const double* x, const double* b, double* y, double* norm,
                 int reduction, Workspace* ws, cudaStream_t st);
uint32_t csr_max_row_nnz(const cbgx_csr& A, cudaStream_t st);

namespace {

// Step slot layout: [hn1, hn2, omega^2, h[0..m], u[0..m]] where hn1/hn2 are
// ||w||^2 after the first/second CGS pass and u the second pass's
// coefficients (host adds them to h, gmres.cpp:65-67).
constexpr size_t kHn1 = 0;
constexpr size_t kHn2 = 1;
constexpr size_t kOmega = 2;
constexpr size_t kH = 3;
inline size_t kU(uint64_t m) { return kH + m + 1; }
inline size_t kSlot(uint64_t m) { return (kU(m) + m + 1 + 3) / 4 * 4; }

// A/B switch: CBGX_OMEGA_PARTS=0 keeps the SpMV's own last-block omega^2
// reduction in the fused path.
bool omega_parts_enabled() {
    static const bool v = [] {
        const char* e = getenv("CBGX_OMEGA_PARTS");
        return !e || atoi(e) != 0;
    }();
    return v;
}

struct BreakdownError : Error {
    BreakdownError(const std::string& m, uint64_t it) : Error(CBGX_EBREAKDOWN, m, it) {}
};

__global__ void narrow_csr_kernel(const uint64_t* __restrict__ rp64, uint64_t n, int32_t* __restrict__ rp32,
                                  const uint64_t* __restrict__ ci64, uint64_t nnz, int32_t* __restrict__ ci32,
                                  uint64_t* __restrict__ bad) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < nnz; k += stride) {
        const uint64_t c = ci64[k];
        if (c >= n) *bad = 1;
        ci32[k] = static_cast<int32_t>(c);
    }
    if (rp32)
        for (uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; r <= n; r += stride)
            rp32[r] = static_cast<int32_t>(rp64[r]);
}

void narrow_csr(const uint64_t* rp64, uint64_t n, int32_t* rp32, const uint64_t* ci64, uint64_t nnz,
                int32_t* ci32, uint64_t* bad, cudaStream_t st) {
    const int grid = static_cast<int>(std::min<uint64_t>((std::max(nnz, n + 1) + 255) / 256, sm_count() * 8ull));
    CBGX_K(narrow_csr_kernel<<<std::max(grid, 1), 256, 0, st>>>(rp64, n, rp32, ci64, nnz, ci32, bad));
    CBGX_CUDA(cudaGetLastError());
}

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
    setup_matrix(true, nullptr);
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
    if (exp_bytes) {
        // per-column exponent ranges (vote-free fast decode, cbgx.h)
        CBGX_CUDA(cudaMalloc(&d_erange_, 2 * (m + 1) * sizeof(uint32_t)));
        CBGX_CUDA(cudaMemset(d_erange_, 0, 2 * (m + 1) * sizeof(uint32_t)));
        V_.d_erange = d_erange_;
    }
    const uint64_t ghosts = halo ? halo->n_ghost : 0;
    CBGX_CUDA(cudaMalloc(&d_r_, std::max<uint64_t>(n_, 1) * sizeof(double)));
    CBGX_CUDA(cudaMalloc(&d_v_, std::max<uint64_t>(n_ + ghosts, 1) * sizeof(double)));
    CBGX_CUDA(cudaMalloc(&d_w_, std::max<uint64_t>(n_, 1) * sizeof(double)));
    const size_t scal = 2 * kSlot(m) + 2 * m + 16;
    CBGX_CUDA(cudaMalloc(&d_scal_, scal * sizeof(double)));
    if (comm_ && comm_->size() > 1) CBGX_CUDA(cudaMalloc(&d_pack_, 2 * (m + 2) * sizeof(double)));
    CBGX_CUDA(cudaMemset(d_scal_, 0, scal * sizeof(double)));
    // mapped: the fused orthogonalisation writes the step slot straight into
    // it (no device-to-host copy between the step's kernels)
    CBGX_CUDA(cudaHostAlloc(&h_pinned_, scal * sizeof(double), cudaHostAllocMapped));
    CBGX_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d_hpinned_), h_pinned_, 0));
    for (auto& e : step_ev_) CBGX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    // The zero-fills above run on the legacy stream; solves may run on a
    // non-blocking stream that does not order after it.
    CBGX_CUDA(cudaStreamSynchronize(nullptr));
}

// Matrix-dependent SpMV state: longest row, staged-tile plan, SELL-32 copy.
// Staged (TMA bulk-copy) CSR SpMV when every 256-row tile fits a stage
// (measured on B200, scripts/spmv_micro.py: 7-pt 128^3 57 vs 65 us, 256^3
// 93% vs 81% of HBM peak); for long rows a SELL-32 copy when memory allows
// (27-pt 128^3: 4.8 vs 5.4 ms/solve of SpMV), else staged with smaller
// tiles, else the plain CSR kernel.
void Solver::setup_matrix(bool before_basis, cudaStream_t st, const unsigned long long* stats) {
    sell_.reset();
    if (dict_) dict_->ready = false;
    tile_rows_ = 0;
    if (stats) A_.max_row_nnz = static_cast<uint32_t>(stats[0]);
    if (A_.max_row_nnz == 0) A_.max_row_nnz = csr_max_row_nnz(A_, st);
    // Dictionary-coded SELL-32 (dsell.cu) when the matrix has <= 255 distinct
    // values and column offsets: 2 B per entry instead of 12 (single rank,
    // or a halo in the window layout, which keeps the column offsets).
    if ((!halo_ || halo_->window) && !(cfg_.flags & CBGX_SOLVER_NO_DICT_SPMV) && A_.max_row_nnz <= 64) {
        uint64_t db = 0, eb = 0;
        if (before_basis) {
            cbgx_basis tmp{};
            cbgx_basis_layout(cfg_.format_kind, cfg_.bit_length, n_, cfg_.restart + 1, &tmp, &db, &eb);
        }
        if (!dict_) dict_ = std::make_unique<DictSell>();
        // reserve: the basis (when not allocated yet) + the solver vectors
        if (build_dict_sell(A_, static_cast<double>(db + eb) + 8.0 * n_ * 8, st, *dict_)) {
            int_s0_ = int_s1_ = 0;
            if (halo_ && comm_ && comm_->size() > 1 && dict_->ell8_w) {
                // interior slices: every row of them has only own columns
                uint64_t gb[2];
                ghost_row_bounds(A_, halo_->own_offset(), gb, st);
                int_s0_ = (gb[0] + 31) / 32;
                int_s1_ = gb[1] / 32;
                if (int_s0_ >= int_s1_) int_s0_ = int_s1_ = 0;
            }
            return;
        }
    }
    uint32_t plan = 0;
    if (!(cfg_.flags & CBGX_SOLVER_NO_TMA_SPMV)) plan = stats ? plan_from_stats(stats) : plan_spmv_tiles(A_, st);
    if (plan >= 128 && A_.max_row_nnz < 16) tile_rows_ = plan;
    if (!tile_rows_ && !(cfg_.flags & CBGX_SOLVER_NO_SELL) && A_.max_row_nnz >= 16) {
        uint64_t db = 0, eb = 0;
        if (before_basis) {
            cbgx_basis tmp{};
            cbgx_basis_layout(cfg_.format_kind, cfg_.bit_length, n_, cfg_.restart + 1, &tmp, &db, &eb);
        }
        size_t free_b = 0, total_b = 0;
        CBGX_CUDA(cudaMemGetInfo(&free_b, &total_b));
        const double after_basis = static_cast<double>(free_b) - static_cast<double>(db + eb) - 64.0 * n_ * 8;
        if (after_basis > 0) sell_ = build_sell(A_, 0.8 * after_basis / static_cast<double>(free_b), st);
    }
    if (!tile_rows_ && !sell_) tile_rows_ = plan;  // no SELL copy (memory): staged if any tile fits
}

void Solver::rebind(const cbgx_csr& A, cudaStream_t st, const unsigned long long* stats) {
    if (A.n_rows != n_ || A.n_cols != A_.n_cols) throw Error(CBGX_EINVAL, "solver: rebind needs the same shape");
    A_ = A;
    setup_matrix(false, st, stats);
}

void Solver::collect_phases(double* ms, size_t count) {
    cbgx_solve_stats S{};
    if (timer_) timer_->collect(&S);
    for (size_t i = 0; i < count && i < CBGX_NUM_PHASES; ++i) ms[i] = S.phase_ms[i];
}

Solver::~Solver() {
    delete timer_;
    for (auto e : step_ev_)
        if (e) cudaEventDestroy(e);
    cudaFree(d_basis_);
    cudaFree(d_exp_);
    cudaFree(d_erange_);
    cudaFree(d_r_);
    cudaFree(d_v_);
    cudaFree(d_w_);
    cudaFree(d_scal_);
    cudaFree(d_pack_);
    cudaFreeHost(h_pinned_);
    if (side_) cudaStreamDestroy(side_);
    if (ev_v_) cudaEventDestroy(ev_v_);
    if (ev_h_) cudaEventDestroy(ev_h_);
}

void Solver::spmv(const double* x, const double* b, double* y, double* norm, cudaStream_t st, bool pdl) {
    if (dict_ && dict_->ready) launch_spmv_dict(A_, *dict_, x, b, y, norm, static_cast<int>(cfg_.reduction), &ws_, st, pdl);
    else if (tile_rows_) launch_spmv_tma(A_, tile_rows_, x, b, y, norm, static_cast<int>(cfg_.reduction), &ws_, st, pdl);
    else if (sell_) launch_spmv_sell(A_, *sell_, x, b, y, norm, static_cast<int>(cfg_.reduction), &ws_, st);
    else launch_spmv(A_, x, b, y, norm, static_cast<int>(cfg_.reduction), &ws_, st);
}

void Solver::halo_spmv(double* v, double* y, double* norm, cudaStream_t st) {
    if (int_s1_ > int_s0_ && dict_ && dict_->ready && dict_->ell8_w) {
        if (!side_) {
            CBGX_CUDA(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
            CBGX_CUDA(cudaEventCreateWithFlags(&ev_v_, cudaEventDisableTiming));
            CBGX_CUDA(cudaEventCreateWithFlags(&ev_h_, cudaEventDisableTiming));
        }
        // exchange on the side stream once v is written; the interior rows
        // meanwhile; then the boundary rows (norm partials added in a fixed
        // order: interior, lower boundary, upper boundary)
        CBGX_CUDA(cudaEventRecord(ev_v_, st));
        CBGX_CUDA(cudaStreamWaitEvent(side_, ev_v_, 0));
        halo_->exchange(v, side_);
        CBGX_CUDA(cudaEventRecord(ev_h_, side_));
        launch_spmv_pell_range(A_, *dict_, v, y, norm, int_s0_, int_s1_, false, &ws_, st);
        CBGX_CUDA(cudaStreamWaitEvent(st, ev_h_, 0));
        launch_spmv_pell_range(A_, *dict_, v, y, norm, 0, int_s0_, true, &ws_, st);
        launch_spmv_pell_range(A_, *dict_, v, y, norm, int_s1_, dict_->nslices, true, &ws_, st);
        return;
    }
    halo_->exchange(v, st);
    spmv(v, nullptr, y, norm, st);
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
    if (!timer_) timer_ = new PhaseTimer();
    PhaseTimer& timer = *timer_;
    timer.on = (cfg_.flags & (CBGX_SOLVER_PHASE_TIMING | CBGX_SOLVER_PHASE_TIMING_DEFERRED)) != 0;
    timer.st = st;
    const int red = static_cast<int>(cfg_.reduction);
    const uint64_t m = cfg_.restart;
    const uint64_t n = n_;
    const int fmt = fmt_from_cfg(cfg_);
    const double bpv = stored_bytes_per_value(fmt);
    const double rp_bytes = A_.row_ptr_bits / 8.0;
    const double spmv_bytes = dict_ && dict_->ready ? dict_->code_bytes() + (dict_->ell_w ? 0.0 : (dict_->nslices + 1) * 8.0) + 16.0 * n
                                    : A_.nnz * 12.0 + (n + 1) * rp_bytes + 16.0 * n;
    const bool multi = comm_ && comm_->size() > 1;
    // own rows of the SpMV input vector (after the lower ghosts in the
    // halo's window layout)
    const uint64_t vo = halo_ ? halo_->own_offset() : 0;
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
    // Device scalars: two step slots (double-buffered so step i+1 can run
    // while the host still reads step i), then y and the restart norm.
    const size_t slot = kSlot(m);
    double* y_dev = d_scal_ + 2 * slot;
    double* rn = y_dev + m + 2;

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

        // Fused orthogonalisation: single GPU, tree reductions, and a grid
        // that can hold every row's w in registers (probed once per solver).
        if (fused_state_ == 0) {
            fused_state_ = (!multi && !halo_ && red == CBGX_REDUCE_TREE && fused_eligible(V_, m)) ? 1 : 2;
        }
        const bool use_fused = fused_state_ == 1 && !(cfg_.flags & CBGX_SOLVER_NO_FUSION);
        // One Arnoldi step on the device (gmres.cpp:210-234 minus the host
        // Givens): spmv, CGS pass, gated second pass, scaled write of the
        // next column, and one D2H of the step's slot. `used` columns are in
        // the basis when the step starts; it writes column used+1.
        auto enqueue_step = [&](uint64_t used, int p) {
            const auto te = std::chrono::steady_clock::now();
            double* sl = d_scal_ + p * slot;
            const uint32_t cols = static_cast<uint32_t>(used + 1);
            GateArg gate;
            gate.hn1 = sl + kHn1;
            gate.omega2 = sl + kOmega;
            gate.eta = cfg_.eta;
            // In the fused path the SpMV and the orthogonalisation are
            // programmatic dependent launches (each starts while the previous
            // kernel drains) unless phase timing puts events between them.
            const bool pdl = use_fused && !timer.on;
            timer.begin(CBGX_PHASE_SPMV);
            // fused path over the pair-coded SpMV: omega^2 stays as per-CTA
            // partials that every fused CTA sums (no last-block tail here)
            uint32_t om_count = 0;
            if (use_fused && !halo_ && dict_ && dict_->ready && dict_->ell8_w && omega_parts_enabled())
                om_count = launch_spmv_pell_parts(A_, *dict_, d_v_, d_w_, &ws_, st, pdl);
            if (om_count) {
            } else if (halo_) {
                halo_spmv(d_v_, d_w_, sl + kOmega, st);  // halo exchange + w = A v, omega^2
            } else {
                spmv(d_v_, nullptr, d_w_, sl + kOmega, st, pdl);  // w = A v, omega^2
            }
            timer.end();
            count(CBGX_PHASE_SPMV, spmv_bytes);
            if (use_fused) {
                // one cooperative launch: dot, update, gated second pass and
                // the scaled write of column used+1, w register-resident
                timer.begin(CBGX_PHASE_ORTHO);
                const bool ok = launch_arnoldi_fused(V_, cols, d_w_, d_v_ + vo, sl, static_cast<uint32_t>(kU(m)), cfg_.eta,
                                                     static_cast<uint32_t>(m), d_hpinned_ + p * slot, pdl, &ws_, st,
                                                     om_count);
                timer.end();
                if (!ok) throw Error(CBGX_EINTERNAL, "fused orthogonalisation became ineligible");
                count(CBGX_PHASE_ORTHO, 2.0 * cols * bpv * n + 8.0 * n + 8.0 * n + bpv * n);
            } else {
                timer.begin(CBGX_PHASE_DOT);
                launch_cgs_dot(V_, 0, cols, d_w_, 0, red, sl + kH, &ws_, st, GateArg{}, !multi);  // h = V^T w
                timer.end();
                count(CBGX_PHASE_DOT, cols * bpv * n + 8.0 * n);
                if (multi) {
                    timer.begin(CBGX_PHASE_COMM);
                    reduce(sl + kOmega, cols + 1, st);
                    timer.end();
                }
                timer.begin(CBGX_PHASE_UPDATE);
                // w -= V h; ||w||^2 (multi-rank: into the packed slot the
                // second pass's partials follow)
                double* pk = multi ? d_pack_ + p * (m + 2) : nullptr;
                launch_cgs_update(V_, 0, cols, sl + kH, 1.0, d_w_, multi ? pk : sl + kHn1, red, &ws_, st);
                timer.end();
                count(CBGX_PHASE_UPDATE, cols * bpv * n + 16.0 * n);
                if (multi) {
                    // Second CGS pass run speculatively (re-orthogonalisation is
                    // the rule on these problems), so hn1 and u cross the ranks
                    // in ONE collective; the gate then decides on the device
                    // whether update2 runs and the host whether u is used.
                    timer.begin(CBGX_PHASE_DOT);
                    launch_cgs_dot(V_, 0, cols, d_w_, 0, red, pk + 1, &ws_, st, GateArg{}, false);
                    timer.end();
                    timer.begin(CBGX_PHASE_COMM);
                    comm_->sum_partials_split(pk, cols + 1, sl + kHn1, sl + kU(m), st);
                    timer.end();
                } else {
                    // Second CGS pass, gated on the device by the reference's test
                    // h_next < eta * omega (gmres.cpp:51-68); empty launches otherwise.
                    timer.begin(CBGX_PHASE_DOT);
                    launch_cgs_dot(V_, 0, cols, d_w_, 0, red, sl + kU(m), &ws_, st, gate, true);
                    timer.end();
                }
                timer.begin(CBGX_PHASE_UPDATE);
                launch_cgs_update(V_, 0, cols, sl + kU(m), 1.0, d_w_, sl + kHn2, red, &ws_, st, gate);
                timer.end();
                if (multi) reduce(sl + kHn2, 1, st);
                S.kernel_launches += 2;
                // v = w / h_next of the last pass that ran; column used+1
                // (gmres.cpp:230-234). Written even when the host will later
                // detect a breakdown: that column is then never read.
                ScaleArg sc;
                sc.src = sl + kHn1;
                sc.mode = 2;
                sc.gate = gate;
                timer.begin(CBGX_PHASE_WRITE);
                launch_basis_write(V_, used + 1, d_w_, sc, d_v_ + vo, nullptr, st);
                timer.end();
                count(CBGX_PHASE_WRITE, 16.0 * n + bpv * n);
            }
            if (!use_fused)  // the fused kernel wrote the mapped slot itself
                CBGX_CUDA(cudaMemcpyAsync(h_pinned_ + p * slot, sl, kU(m) * sizeof(double) + cols * sizeof(double),
                                          cudaMemcpyDeviceToHost, st));
            CBGX_CUDA(cudaEventRecord(step_ev_[p], st));
            S.host_enqueue_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - te).count();
        };

        for (;;) {
            // Explicit residual r = b - A x (gmres.cpp:181-190).
            timer.begin(CBGX_PHASE_RESIDUAL);
            const double* xin = d_x;
            if (halo_) {
                CBGX_CUDA(cudaMemcpyAsync(d_v_ + vo, d_x, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
                halo_->exchange(d_v_, st);
                xin = d_v_;
            }
            spmv(xin, d_b, d_r_, rn, st);
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
            ScaleArg sc0;
            sc0.src = rn;
            sc0.mode = 1;
            launch_basis_write(V_, 0, d_r_, sc0, d_v_ + vo, nullptr, st);
            timer.end();
            count(CBGX_PHASE_WRITE, 16.0 * n + bpv * n);

            uint64_t used = 0;
            bool cycle_done = false;
            // Steps that can run in this cycle (restart and iteration cap).
            const uint64_t max_steps = std::min<uint64_t>(m, cfg_.max_total_iterations - iter);
            uint64_t enqueued = 0;
            double rrn_prev = 0.0, rrn_last = 0.0;  // implicit RRN after steps used-2, used-1
            while (!cycle_done) {
                // Look one step ahead: the device works on step used+1 while
                // the host runs Givens on step `used` -- unless step `used`
                // is predicted to end the cycle by convergence (the last
                // residual ratio carried one step: rrn_last^2 / rrn_prev <=
                // 4 target), where the lookahead step would be wasted work
                // (the cycle's largest Arnoldi step). A wrong prediction only
                // exposes the host's Givens latency for that step.
                const bool near = used >= 2 && rrn_last * (rrn_last / rrn_prev) <= 4.0 * cfg_.target_rrn;
                const uint64_t want = used + (near ? 1 : 2);
                while (enqueued < max_steps && enqueued < want) {
                    enqueue_step(enqueued, static_cast<int>(enqueued & 1));
                    ++enqueued;
                }
                const int p = static_cast<int>(used & 1);
                const auto tw = std::chrono::steady_clock::now();
                CBGX_CUDA(cudaEventSynchronize(step_ev_[p]));
                S.host_wait_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tw).count();
                const double* hs = h_pinned_ + p * slot;
                ++iter;
                const uint32_t cols = static_cast<uint32_t>(used + 1);
                const double omega = std::sqrt(hs[kOmega]);
                double h_next = std::sqrt(hs[kHn1]);
                for (uint64_t i = 0; i < cols; ++i) hcol[i] = hs[kH + i];
                bool breakdown = false;
                if (h_next < cfg_.eta * omega) {
                    // the device ran the second pass (gmres.cpp:53-68)
                    ++S.reorth_passes;
                    if (use_fused) {
                        S.phase_bytes[CBGX_PHASE_ORTHO] += 2.0 * cols * bpv * n;
                    } else {
                        count(CBGX_PHASE_DOT, cols * bpv * n + 8.0 * n);
                        count(CBGX_PHASE_UPDATE, cols * bpv * n + 16.0 * n);
                    }
                    const double before = h_next;
                    for (uint64_t i = 0; i < cols; ++i) hcol[i] += hs[kU(m) + i];
                    h_next = std::sqrt(hs[kHn2]);
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
                rrn_prev = rrn_last;
                rrn_last = implicit_rrn;
                cycle_done = breakdown || implicit_rrn <= cfg_.target_rrn || used == m ||
                             iter >= cfg_.max_total_iterations;
                if (!cycle_done) push(iter, implicit_rrn, false);
            }
            // A speculative step beyond the cycle end may still be in flight;
            // it only touched w, v, its scalar slot and basis column used+1..,
            // none of which the solution update below reads.
            // x += V y (gmres.cpp:242-243, :134-139)
            const long bad = lsq.solve_y(y.data());
            if (bad >= 0) throw BreakdownError("gmres: singular triangular factor", static_cast<uint64_t>(bad));
            timer.begin(CBGX_PHASE_SOLUTION);
            double* hy = h_pinned_ + 2 * slot;
            std::memcpy(hy, y.data(), used * sizeof(double));
            CBGX_CUDA(cudaMemcpyAsync(y_dev, hy, used * sizeof(double), cudaMemcpyHostToDevice, st));
            launch_cgs_update(V_, 0, static_cast<uint32_t>(used), y_dev, -1.0, d_x, nullptr, red, &ws_, st);
            timer.end();
            count(CBGX_PHASE_SOLUTION, used * bpv * n + 16.0 * n);
        }
        S.total_iterations = iter;
        S.restarts = cycles > 0 ? cycles - 1 : 0;
        S.final_rrn = last;
    }
    CBGX_CUDA(cudaStreamSynchronize(st));
    if (cfg_.flags & CBGX_SOLVER_PHASE_TIMING) timer.collect(&S);
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


// Per-device state kept between cbgx_gmres_solve_host calls: the staging
// buffers (grown to the largest problem seen), a stream, and the last
// solver. Every call still copies its host inputs and result; only the
// allocations are reused (cudaMalloc/cudaFree, pinned allocations and the
// basis set-up are what a fresh call would otherwise pay). Released by
// cbgx_host_cache_release.
struct HostSolveCache {
    std::mutex mu;
    cudaStream_t st = nullptr, st2 = nullptr;
    cudaEvent_t ev_idx = nullptr, ev_narrow = nullptr, ev_va = nullptr, ev_setup = nullptr;
    uint64_t cap_n = 0, cap_nnz = 0;
    uint64_t* d_rp64 = nullptr;
    uint64_t* d_ci64 = nullptr;
    double* d_va = nullptr;
    double* d_b = nullptr;
    double* d_x0 = nullptr;
    double* d_x = nullptr;
    int32_t* d_ci = nullptr;
    int32_t* d_rp32 = nullptr;
    uint64_t* d_bad = nullptr;
    uint64_t* h_bad = nullptr;
    std::unique_ptr<Solver> solver;
    void free_buffers() {
        for (void* p : {static_cast<void*>(d_rp64), static_cast<void*>(d_ci64), static_cast<void*>(d_va),
                        static_cast<void*>(d_b), static_cast<void*>(d_x0), static_cast<void*>(d_x),
                        static_cast<void*>(d_ci), static_cast<void*>(d_rp32), static_cast<void*>(d_bad)})
            if (p) cudaFree(p);
        d_rp64 = d_ci64 = d_bad = nullptr;
        d_va = d_b = d_x0 = d_x = nullptr;
        d_ci = d_rp32 = nullptr;
        cap_n = cap_nnz = 0;
    }
    void release() {
        solver.reset();
        free_buffers();
        if (h_bad) cudaFreeHost(h_bad);
        h_bad = nullptr;
        if (st) cudaStreamDestroy(st);
        if (st2) cudaStreamDestroy(st2);
        if (ev_idx) cudaEventDestroy(ev_idx);
        if (ev_narrow) cudaEventDestroy(ev_narrow);
        if (ev_va) cudaEventDestroy(ev_va);
        if (ev_setup) cudaEventDestroy(ev_setup);
        st = st2 = nullptr;
        ev_idx = ev_narrow = ev_va = ev_setup = nullptr;
    }
    void ensure(uint64_t n, uint64_t nnz, bool wide) {
        (void)wide;
        if (!st) CBGX_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        if (!st2) CBGX_CUDA(cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking));
        if (!ev_idx) CBGX_CUDA(cudaEventCreateWithFlags(&ev_idx, cudaEventDisableTiming));
        if (!ev_narrow) CBGX_CUDA(cudaEventCreateWithFlags(&ev_narrow, cudaEventDisableTiming));
        if (!ev_va) CBGX_CUDA(cudaEventCreateWithFlags(&ev_va, cudaEventDisableTiming));
        if (!ev_setup) CBGX_CUDA(cudaEventCreateWithFlags(&ev_setup, cudaEventDisableTiming));
        if (!h_bad) CBGX_CUDA(cudaMallocHost(&h_bad, 6 * sizeof(uint64_t)));
        if (n <= cap_n && nnz <= cap_nnz && d_bad) return;
        solver.reset();  // it points into the buffers
        free_buffers();
        const uint64_t N = std::max<uint64_t>(n, 1), Z = std::max<uint64_t>(nnz, 1);
        CBGX_CUDA(cudaMalloc(&d_rp64, (N + 1) * 8));
        CBGX_CUDA(cudaMalloc(&d_ci64, Z * 8));
        CBGX_CUDA(cudaMalloc(&d_va, Z * 8));
        CBGX_CUDA(cudaMalloc(&d_b, N * 8));
        CBGX_CUDA(cudaMalloc(&d_x0, N * 8));
        CBGX_CUDA(cudaMalloc(&d_x, N * 8));
        CBGX_CUDA(cudaMalloc(&d_ci, Z * 4));
        CBGX_CUDA(cudaMalloc(&d_rp32, (N + 1) * 4));
        CBGX_CUDA(cudaMalloc(&d_bad, 6 * 8));  // [bad index flag, csr stats x5]
        cap_n = n;
        cap_nnz = nnz;
    }
};

bool same_config(const cbgx_gmres_config& a, const cbgx_gmres_config& b) {
    return a.restart == b.restart && a.target_rrn == b.target_rrn && a.max_total_iterations == b.max_total_iterations &&
           a.eta == b.eta && a.format_kind == b.format_kind && a.bit_length == b.bit_length &&
           a.reduction == b.reduction && a.flags == b.flags;
}

HostSolveCache& host_cache() {
    static HostSolveCache* caches = new HostSolveCache[64];  // never destroyed: no CUDA calls at exit
    const int d = current_device();
    if (d < 0 || d >= 64) throw Error(CBGX_EINVAL, "device index out of range");
    return caches[d];
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

int cbgx_solver_phase_times(cbgx_solver* s, double* ms, uint64_t count) {
    return guard([&] {
        if (!s) throw Error(CBGX_EINVAL, "solver: null handle");
        reinterpret_cast<SolverHandle*>(s)->solver->collect_phases(ms, count);
    });
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
        HostSolveCache& H = host_cache();
        std::lock_guard<std::mutex> lock(H.mu);
        static const bool prof = [] {
            const char* e = getenv("CBGX_PROFILE_HOST_SOLVE");
            return e && e[0] == '1';
        }();
        auto tnow = [] { return std::chrono::steady_clock::now(); };
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        const auto t0 = tnow();
        H.ensure(n, nnz, wide);
        cudaStream_t st = H.st;
        // Stream-ordered staging: the size_t CSR of the reference
        // (CsrMatrix, sparse.hpp:17-26) goes over as-is and is narrowed on the
        // device (int32 columns, int32/int64 row offsets).
        CBGX_CUDA(cudaMemsetAsync(H.d_bad, 0, 8, st));
        CBGX_CUDA(cudaMemcpyAsync(H.d_rp64, row_ptrs, (n + 1) * 8, cudaMemcpyHostToDevice, st));
        CBGX_CUDA(cudaMemcpyAsync(H.d_ci64, col_idx, nnz * 8, cudaMemcpyHostToDevice, st));
        // narrowing + CSR statistics on a second stream, overlapped with the
        // remaining uploads (values, b, x0)
        CBGX_CUDA(cudaEventRecord(H.ev_idx, st));
        CBGX_CUDA(cudaStreamWaitEvent(H.st2, H.ev_idx, 0));
        void* d_rp = wide ? static_cast<void*>(H.d_rp64) : static_cast<void*>(H.d_rp32);
        narrow_csr(H.d_rp64, n, wide ? nullptr : H.d_rp32, H.d_ci64, nnz, H.d_ci, H.d_bad, H.st2);
        cbgx_csr A{n, n, nnz, d_rp, wide ? 64u : 32u, H.d_ci, H.d_va};
        // the SpMV set-up statistics ride along with the range check: one sync
        launch_csr_stats(A, reinterpret_cast<unsigned long long*>(H.d_bad + 1), H.st2);
        CBGX_CUDA(cudaMemcpyAsync(H.d_va, values, nnz * 8, cudaMemcpyHostToDevice, st));
        CBGX_CUDA(cudaEventRecord(H.ev_va, st));
        CBGX_CUDA(cudaMemcpyAsync(H.d_b, b, n * 8, cudaMemcpyHostToDevice, st));
        CBGX_CUDA(cudaMemcpyAsync(H.d_x0, x0, n * 8, cudaMemcpyHostToDevice, st));
        if (prof) CBGX_CUDA(cudaStreamSynchronize(st));
        const auto t1 = tnow();
        // the range check and statistics (second stream) while b and x0 still
        // upload on the first
        CBGX_CUDA(cudaMemcpyAsync(H.h_bad, H.d_bad, 6 * 8, cudaMemcpyDeviceToHost, H.st2));
        CBGX_CUDA(cudaStreamSynchronize(H.st2));
        if (*H.h_bad) throw Error(CBGX_EINVAL, "csr: column index out of range");
        const unsigned long long* csr_stats = reinterpret_cast<const unsigned long long*>(H.h_bad + 1);
        const auto t2 = tnow();
        // One solver per configuration and shape, kept between calls (its
        // basis, vectors and workspaces); only the matrix-dependent SpMV
        // state is recomputed for the new contents -- on the second stream,
        // once the values are in, overlapped with the b / x0 upload.
        if (H.solver && H.solver->rows() == n && same_config(H.solver->config(), c)) {
            CBGX_CUDA(cudaStreamWaitEvent(H.st2, H.ev_va, 0));
            H.solver->rebind(A, H.st2, csr_stats);
            CBGX_CUDA(cudaEventRecord(H.ev_setup, H.st2));
            CBGX_CUDA(cudaStreamWaitEvent(st, H.ev_setup, 0));
        } else {
            // a new solver sets itself up on the legacy stream: everything first
            CBGX_CUDA(cudaStreamSynchronize(st));
            H.solver.reset();
            H.solver = std::make_unique<Solver>(A, c, nullptr, nullptr);
        }
        const auto t3 = tnow();
        H.solver->solve(H.d_b, H.d_x0, H.d_x, hist, stats, st);
        const auto t4 = tnow();
        CBGX_CUDA(cudaMemcpyAsync(x_out, H.d_x, n * 8, cudaMemcpyDeviceToHost, st));
        CBGX_CUDA(cudaStreamSynchronize(st));
        if (prof)
            fprintf(stderr, "cbgx host solve: h2d %.3f ms (%.1f GB/s) narrow %.3f setup %.3f solve %.3f d2h %.3f\n",
                    ms(t0, t1), ((n + 1) * 8.0 + nnz * 16.0 + n * 16.0) / ms(t0, t1) / 1e6, ms(t1, t2), ms(t2, t3),
                    ms(t3, t4), ms(t4, tnow()));
    });
}

int cbgx_host_cache_release(void) {
    return guard([&] {
        HostSolveCache& H = host_cache();
        std::lock_guard<std::mutex> lock(H.mu);
        H.release();
    });
}

}  // extern "C"
