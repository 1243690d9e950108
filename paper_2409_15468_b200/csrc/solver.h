// solver.h -- device-resident restarted CB-GMRES driver (host control loop).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

#include "cbgx.h"
#include "reduce.cuh"
#include "runtime.h"

namespace cbgx {

// Cross-rank plumbing for the row-partitioned solve. A null Comm means one
// rank (single GPU).
struct Comm {
    virtual ~Comm() = default;
    virtual int rank() const = 0;
    virtual int size() const = 0;
    // d_vals[0..count) hold this rank's partial sums. Replace them by the
    // sum over ranks taken in rank order 0..P-1 (identical on every rank,
    // independent of the collective's algorithm).
    virtual void sum_partials(double* d_vals, size_t count, cudaStream_t st) = 0;
    // The same combine for a packed vector d_src[0..count): the sum of
    // element 0 goes to *d_first, of elements 1.. to d_rest[0..count-1)
    // (two slots of the step that are not adjacent -- one collective).
    virtual void sum_partials_split(const double* d_src, size_t count, double* d_first, double* d_rest,
                                    cudaStream_t st) = 0;
    // Gather `bytes` from every rank into d_recv[rank * bytes].
    virtual void allgather(const void* d_send, void* d_recv, size_t bytes, cudaStream_t st) = 0;
    struct Msg {
        int peer;
        void* d_buf;
        size_t bytes;
    };
    // Grouped point-to-point exchange (all sends and receives in flight together).
    virtual void exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs,
                          cudaStream_t st) = 0;
    virtual void barrier(cudaStream_t st) = 0;
};

// Halo plan: which own rows each peer needs (packed by a gather kernel),
// and where each peer's ghosts land in the local vector (after the own rows).
struct Halo {
    Comm* comm = nullptr;
    uint64_t n_local = 0;
    uint64_t n_ghost = 0;
    std::vector<int> send_peers, recv_peers;
    std::vector<uint64_t> send_offsets;   // into d_send_idx / d_send_buf (size peers+1)
    std::vector<uint64_t> recv_offsets;   // into ghost region (size peers+1)
    int32_t* d_send_idx = nullptr;        // local row indices to pack
    double* d_send_buf = nullptr;
    // window layout: the local vector is [win_lo ghosts | own rows | ghosts]
    // (global rows [rb - win_lo, re + ...)); compact: [own rows | ghosts]
    bool window = false;
    uint64_t win_lo = 0;
    uint64_t own_offset() const { return window ? win_lo : 0; }
    ~Halo();
    void exchange(double* d_vec, cudaStream_t st) const;  // fills the ghost slots of d_vec
};

class Solver {
public:
    Solver(const cbgx_csr& A, const cbgx_gmres_config& cfg, Comm* comm, Halo* halo);
    ~Solver();
    void solve(const double* d_b, const double* d_x0, double* d_x, cbgx_history* hist,
               cbgx_solve_stats* stats, cudaStream_t st);

    // Device time per phase accumulated over deferred-timing solves (resets).
    void collect_phases(double* ms, size_t count);
    // Same shape, new matrix contents/pointers: recompute the SpMV state,
    // keep every allocation (basis, vectors, workspaces).
    void rebind(const cbgx_csr& A, cudaStream_t st, const unsigned long long* stats = nullptr);
    uint64_t rows() const { return n_; }
    const cbgx_gmres_config& config() const { return cfg_; }

private:
    struct PhaseTimer;
    PhaseTimer* timer_ = nullptr;
    void reduce(double* d_vals, size_t count, cudaStream_t st);
    void spmv(const double* x, const double* b, double* y, double* norm, cudaStream_t st, bool pdl = false);
    // Halo exchange of v + w = A v (+ ||w||^2): with a pair-coded window-
    // layout matrix, the interior rows (no ghost columns) overlap the
    // exchange, which runs on a side stream; otherwise exchange, then SpMV.
    void halo_spmv(double* v, double* y, double* norm, cudaStream_t st);
    double fetch_scalar(const double* d, cudaStream_t st);
    void setup_matrix(bool before_basis, cudaStream_t st, const unsigned long long* stats = nullptr);

    cbgx_csr A_;
    cbgx_gmres_config cfg_;
    Comm* comm_;
    Halo* halo_;
    uint64_t n_;
    cbgx_basis V_{};
    void* d_basis_ = nullptr;
    uint32_t* d_exp_ = nullptr;
    uint32_t* d_erange_ = nullptr;  // per-column exponent ranges (FRSZ2)
    double* d_r_ = nullptr;
    double* d_v_ = nullptr;   // n + ghosts
    double* d_w_ = nullptr;
    double* d_scal_ = nullptr;
    double* d_pack_ = nullptr;   // multi-rank: per slot parity [hn1, u[0..m]] partials (one collective)   // [0] omega^2 [1] hn^2 [2] ||b||^2 [3] ||r||^2 [4..] h / u / y
    double* h_pinned_ = nullptr;
    double* d_hpinned_ = nullptr;  // device alias of the mapped h_pinned_
    cudaEvent_t step_ev_[2] = {nullptr, nullptr};
    // interior slices [int_s0_, int_s1_) of the local matrix (no ghost
    // columns) for the overlapped halo SpMV; side stream and its events
    uint64_t int_s0_ = 0, int_s1_ = 0;
    cudaStream_t side_ = nullptr;
    cudaEvent_t ev_v_ = nullptr, ev_h_ = nullptr;
    int fused_state_ = 0;
    std::unique_ptr<Sell> sell_;
    std::unique_ptr<DictSell> dict_;  // dictionary-coded SELL-32 (preferred when it applies)
    uint32_t tile_rows_ = 0;      // staged SpMV tile height (0: not used)
    Workspace ws_;
};

struct SolverHandle {
    std::unique_ptr<Solver> solver;
};

}  // namespace cbgx
