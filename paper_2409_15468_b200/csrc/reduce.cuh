// reduce.cuh -- deterministic two-stage reduction epilogue shared by every
// reducing kernel (CGS dot/update norms, SpMV norms, BLAS-1 dot).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>

#include "common.cuh"
#include "runtime.h"

namespace cbgx {

// Lane L's share of column k over `rows` CTA partial rows: rows L, L+32, ...
// summed in that order. All loads are issued before the first add (the
// partials sit in L2; a dependent load-add loop would pay one L2 round trip
// per row).
__device__ __forceinline__ double lane_sum_rows(const double* __restrict__ partials, uint32_t stride, uint32_t k,
                                                unsigned rows, int lane) {
    constexpr int kMax = 24;  // up to 768 CTAs
    double v[kMax];
#pragma unroll
    for (int i = 0; i < kMax; ++i) {
        const unsigned c = lane + 32u * i;
        v[i] = c < rows ? __ldcg(partials + static_cast<uint64_t>(c) * stride + k) : 0.0;
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < kMax; ++i)
        if (lane + 32u * i < rows) s = __dadd_rn(s, v[i]);
    for (unsigned c = lane + 32u * kMax; c < rows; c += 32)
        s = __dadd_rn(s, __ldcg(partials + static_cast<uint64_t>(c) * stride + k));
    return s;
}

// red: shared [nwarps][ncol] per-warp partials. Writes this CTA's row of
// partials[gridDim.x][ncol]; the last CTA to arrive (ticket) sums the rows
// in CTA order into out[ncol] and re-arms the ticket. The summation order
// depends only on gridDim.x, so results are bit-reproducible run to run.
__device__ __forceinline__ void block_finalize(const double* red, int nwarps, uint32_t ncol,
                                               double* __restrict__ partials,
                                               unsigned* __restrict__ ticket,
                                               double* __restrict__ out, bool accumulate = false) {
    __shared__ bool s_last;
    for (uint32_t k = threadIdx.x; k < ncol; k += blockDim.x) {
        double s = red[k];
        for (int w = 1; w < nwarps; ++w) s = __dadd_rn(s, red[w * ncol + k]);
        partials[static_cast<uint64_t>(blockIdx.x) * ncol + k] = s;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // Column k: lane L sums CTA rows L, L+32, ... in order, then a fixed
    // butterfly across the warp -- the same shape every launch.
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (uint32_t k = warp; k < ncol; k += nw) {
        const double s = warp_sum(lane_sum_rows(partials, ncol, k, gridDim.x, lane));
        // accumulate: add to the value an earlier launch left (a split SpMV)
        if (lane == 0) out[k] = accumulate ? __dadd_rn(out[k], s) : s;
    }
    if (threadIdx.x == 0) *ticket = 0u;
}

// SELL-32 copy of a CSR matrix (see sparse.cu).
struct Sell {
    double* val = nullptr;
    int32_t* col = nullptr;
    uint64_t* soff = nullptr;
    uint64_t nslices = 0;
    uint64_t entries = 0;
    ~Sell();
};
// nullptr when the copy would take more than max_fraction_of_free of free memory.
std::unique_ptr<Sell> build_sell(const cbgx_csr& A, double max_fraction_of_free, cudaStream_t st);
void launch_spmv_sell(const cbgx_csr& A, const Sell& S, const double* x, const double* b, double* y, double* norm,
                      int reduction, Workspace* ws, cudaStream_t st);

// Dictionary-coded SELL-32 copy (see dsell.cu): 2-byte codes into <= 255
// distinct values and <= 255 distinct column offsets.
struct DictSell {
    uint16_t* codes = nullptr;
    uint64_t* soff = nullptr;  // SELL layout only
    int32_t* off = nullptr;    // [256]
    double* val = nullptr;     // [256]
    uint64_t nslices = 0;
    uint64_t entries = 0;
    uint32_t n_off = 0, n_val = 0;
    // build options (cbgx_csr_dict_create2): 0 = 2-byte codes only,
    // 1 = up to pair codes, 2 = up to row patterns, 3 = up to uniform slots
    // (default)
    uint32_t max_level = 3;
    uint32_t ell_w = 0;  // > 0: ELL4 layout, every row padded to this width
    bool ready = false;
    // Pair-coded ELL8 copy (when the matrix holds <= 255 distinct (value,
    // column offset) pairs): 1-byte codes into one pair table, rows padded
    // to a multiple of 8 entries (0xFF = padding). Used by the SpMV when set.
    uint8_t* codes8 = nullptr;
    uint64_t entries8 = 0, codes8_cap = 0;
    uint32_t ell8_w = 0;   // > 0: the pair-coded copy is valid
    uint32_t n_pair = 0;
    double* pair_val = nullptr;   // [256]
    int32_t* pair_off = nullptr;  // [256]
    uint8_t* map8 = nullptr;      // [65536] 2-byte code -> pair index
    unsigned* bitmap = nullptr;   // [2048] codes present
    // Row-pattern copy (when the pair-coded rows take <= 255 distinct
    // patterns): one byte per row into a table of {offsets, values} per
    // pattern. Used by the SpMV when n_pat > 0.
    uint8_t* pid = nullptr;
    uint64_t pid_cap = 0;
    uint4* ptab = nullptr;        // n_pat * 96 * G bytes
    uint8_t* pcnt = nullptr;      // [256] leading real entries per pattern
    // Uniform-slot copy (n_slots > 0): the patterns' offsets embed into one
    // list of <= 32 slots with one value each; pmask[p] = the slots of p
    uint32_t n_slots = 0;
    uint32_t* pmask = nullptr;    // [256]
    alignas(8) unsigned char uslots[384];  // USlots (dsell.cu): int32 off[32], fp64 val[32]
    uint32_t n_pat = 0, ptab_u4 = 0;
    unsigned long long* pkeys = nullptr;  // build scratch [1024]
    uint2* pwords = nullptr;              // build scratch [1024 * 4]
    uint8_t* pslot = nullptr;             // build scratch [1024]
    // matrix bytes one SpMV streams (the codes actually read)
    double code_bytes() const {
        return n_pat ? static_cast<double>(nslices) * 32.0
                     : ell8_w ? static_cast<double>(entries8) : 2.0 * static_cast<double>(entries);
    }
    // build scratch and capacities (kept across rebuilds)
    unsigned long long* tabs = nullptr;
    unsigned* flags = nullptr;
    uint8_t* idx = nullptr;
    uint64_t codes_cap = 0, soff_cap = 0;
    ~DictSell();
};
// (Re)builds D for A, reusing its buffers; false when A does not fit the
// dictionaries or a (re)allocated copy would take more than 80% of the free
// memory less reserve_bytes (kept for later allocations, e.g. the basis).
// Stream-ordered on return (no trailing synchronisation).
bool build_dict_sell(const cbgx_csr& A, double reserve_bytes, cudaStream_t st, DictSell& D);
void launch_spmv_dict(const cbgx_csr& A, const DictSell& D, const double* x, const double* b, double* y, double* norm,
                      int reduction, Workspace* ws, cudaStream_t st, bool pdl = false);
// Pair-coded SpMV of the 32-row slices [s_begin, s_end) (D.ell8_w != 0); the
// norm (tree order) is written, or added to *norm when `accumulate`.
// Pair-coded SpMV y = A x whose CTAs leave their omega^2 = ||y||^2 partials
// in ws->omega_parts (the fused orthogonalisation sums them); returns the
// partial count, 0 when D has no pair-coded copy (nothing launched).
uint32_t launch_spmv_pell_parts(const cbgx_csr& A, const DictSell& D, const double* x, double* y, Workspace* ws,
                                cudaStream_t st, bool pdl);
void launch_spmv_pell_range(const cbgx_csr& A, const DictSell& D, const double* x, double* y, double* norm,
                            uint64_t s_begin, uint64_t s_end, bool accumulate, Workspace* ws, cudaStream_t st);
// Rows touching the halo of a local matrix whose own columns are
// [lo, lo + n_rows): out[0] = 1 + last row with a column below lo (0: none),
// out[1] = first row with a column >= lo + n_rows (n_rows: none). Synchronous.
void ghost_row_bounds(const cbgx_csr& A, uint64_t lo, uint64_t out[2], cudaStream_t st);

// Staged (TMA) CSR SpMV: plan_spmv_tiles returns the tile height (32..256
// rows, 0 when some tile would exceed the stage capacity).
uint32_t plan_spmv_tiles(const cbgx_csr& A, cudaStream_t st);
// Stream-ordered CSR statistics [max_row, max 32/64/128/256-row tile nnz]
// into d_out[5] (no sync), and the tile plan they imply.
void launch_csr_stats(const cbgx_csr& A, unsigned long long* d_out, cudaStream_t st);
uint32_t plan_from_stats(const unsigned long long* h);
void launch_spmv_tma(const cbgx_csr& A, uint32_t tile_rows, const double* x, const double* b, double* y,
                     double* norm, int reduction, Workspace* ws, cudaStream_t st, bool pdl = false);

// Deterministic <x, y>. REDUCE_TREE: fixed-shape tree; REDUCE_REFERENCE:
// one thread, sequential from +0.0 (sparse.cpp:58-67).
void launch_dot(const double* x, const double* y, uint64_t n, int reduction, double* out,
                Workspace* ws, cudaStream_t st, const GateArg& gate = GateArg{});

// gate: run only when the device-side re-orthogonalisation test holds.
// coop: the dynamic-tile dot (a cooperative launch with a grid barrier);
// false for callers that may run several grids concurrently on one device
// (the threaded partitioned solve).
void launch_cgs_dot(const cbgx_basis& V, uint64_t first, uint32_t cols, const double* w, int wn,
                    int reduction, double* h, Workspace* ws, cudaStream_t st,
                    const GateArg& gate = GateArg{}, bool coop = true);
void launch_cgs_update(const cbgx_basis& V, uint64_t first, uint32_t cols, const double* h,
                       double sign, double* w, double* norm, int reduction, Workspace* ws,
                       cudaStream_t st, const GateArg& gate = GateArg{});
// Fused single-GPU orthogonalisation + next-column write (one cooperative
// launch; see cgs.cu). Returns false (nothing launched) when the problem is
// too large for the register-resident w of a co-resident grid.
bool fused_eligible(const cbgx_basis& V, uint64_t max_cols);
// host_slot: mapped pinned copy of the step slot written by the kernel (no
// D2H copy in the stream); pdl: programmatic dependent launch.
// om_count > 0: omega^2 is the fixed-order sum of the SpMV's om_count CTA
// partials in ws->omega_parts (launch_spmv_pell_parts), computed by every
// CTA; otherwise it is read from slot[2].
bool launch_arnoldi_fused(const cbgx_basis& V, uint32_t cols, const double* w, double* v_out, double* slot,
                          uint32_t u_off, double eta, uint32_t max_cols, double* host_slot, bool pdl,
                          Workspace* ws, cudaStream_t st, uint32_t om_count = 0);
void launch_basis_write(const cbgx_basis& V, uint64_t j, const double* x, const ScaleArg& scale,
                        double* v_out, uint64_t* bad, cudaStream_t st);
// Read benchmark sweep of one basis column (readbench.cu's C-ABI).
void launch_read_sweep(const cbgx_basis& V, uint64_t col, uint64_t n, int intensity, double mul, double add,
                       double* out, Workspace* ws, cudaStream_t st);
void launch_basis_read(const cbgx_basis& V, uint64_t j, uint64_t first, uint64_t count, double* out,
                       cudaStream_t st);

}  // namespace cbgx
