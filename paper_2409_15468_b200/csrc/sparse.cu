// sparse.cu -- CSR SpMV (fused norm / residual epilogues), BLAS-1 and the
// device-side 3-D stencil generators.
//
// Reference: sparse.cpp:43-84 (spmv, dot, norm2, scale, axpy), gmres.cpp:
// 181-190 (explicit residual). SpMV accumulates each row left to right from
// +0.0 with separate multiply/add roundings, so y is bit-identical to the
// reference; only the fused norms depend on the (fixed) reduction tree.
#include <cub/device/device_scan.cuh>

#include <algorithm>

#include "common.cuh"
#include "pipeline.cuh"
#include "reduce.cuh"
#include "runtime.h"

namespace cbgx {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

int rows_grid(uint64_t rows) {
    const uint64_t want = (rows + kThreads - 1) / kThreads;
    const uint64_t cap = static_cast<uint64_t>(sm_count()) * 8;
    return static_cast<int>(std::max<uint64_t>(1, std::min(want, cap)));
}

// MODE 0: y = A x.  MODE 1: y = b - A x.
template <typename RP, int MODE>
__global__ void __launch_bounds__(kThreads)
spmv_kernel(uint64_t n_rows, const RP* __restrict__ rp, const int32_t* __restrict__ ci,
            const double* __restrict__ va, const double* __restrict__ x,
            const double* __restrict__ b, double* __restrict__ y, int with_norm,
            double* __restrict__ partials, unsigned* __restrict__ ticket,
            double* __restrict__ norm_out) {
    __shared__ double red[kWarps];
    double acc = 0.0;
    for (uint64_t r = blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x; r < n_rows;
         r += static_cast<uint64_t>(gridDim.x) * kThreads) {
        const uint64_t k0 = static_cast<uint64_t>(__ldg(rp + r));
        const uint64_t k1 = static_cast<uint64_t>(__ldg(rp + r + 1));
        double s = 0.0;
        // batches of 8 entries: all index/value loads, then all gathers, then
        // the in-order multiply-adds (sparse.cpp:50-52 order, two roundings)
        for (uint64_t k = k0; k < k1; k += 8) {
            int32_t c[8];
            double v[8], xv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const bool in = k + i < k1;
                c[i] = in ? __ldg(ci + k + i) : 0;
                v[i] = in ? __ldg(va + k + i) : 0.0;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) xv[i] = k + i < k1 ? __ldg(x + c[i]) : 0.0;
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (k + i < k1) s = __dadd_rn(s, __dmul_rn(v[i], xv[i]));
        }
        if (MODE == 1) s = __dsub_rn(__ldg(b + r), s);
        y[r] = s;
        if (with_norm) acc = __dadd_rn(acc, __dmul_rn(s, s));
    }
    if (!with_norm) return;
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    block_finalize(red, kWarps, 1, partials, ticket, norm_out);
}

// ---------------------------------------------------------------- SELL-32
// Sliced ELLPACK copy of a CSR matrix built once at solver setup: slice s
// holds rows 32s..32s+31; entry k of every row of the slice is stored at
// off[s] + 32k + lane, so a warp streams the slice with fully coalesced
// loads. Entries keep their in-row order and padding is never added, so
// y is bit-identical to the CSR SpMV (and to the reference).
template <typename RP>
__global__ void sell_len_kernel(const RP* __restrict__ rp, uint64_t n, uint64_t nslices, uint64_t* __restrict__ slen) {
    for (uint64_t sl = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) / 32; sl < nslices + 1;
         sl += static_cast<uint64_t>(gridDim.x) * blockDim.x / 32) {
        const int lane = threadIdx.x & 31;
        const uint64_t r = sl * 32 + lane;
        const unsigned len = (sl < nslices && r < n) ? static_cast<unsigned>(rp[r + 1] - rp[r]) : 0u;
        const unsigned m = __reduce_max_sync(0xFFFFFFFFu, len);
        if (lane == 0) slen[sl] = static_cast<uint64_t>(m) * 32;
    }
}

template <typename RP>
__global__ void sell_fill_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ ci,
                                 const double* __restrict__ va, uint64_t n, const uint64_t* __restrict__ soff,
                                 double* __restrict__ sv, int32_t* __restrict__ sc) {
    for (uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; r < (n + 31) / 32 * 32;
         r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t sl = r / 32, lane = r % 32;
        const uint64_t off = soff[sl], ml = (soff[sl + 1] - off) / 32;
        const uint64_t k0 = r < n ? static_cast<uint64_t>(rp[r]) : 0, len = r < n ? static_cast<uint64_t>(rp[r + 1]) - k0 : 0;
        for (uint64_t k = 0; k < ml; ++k) {
            sv[off + k * 32 + lane] = k < len ? va[k0 + k] : 0.0;
            sc[off + k * 32 + lane] = k < len ? ci[k0 + k] : 0;
        }
    }
}

template <typename RP, int MODE>
__global__ void __launch_bounds__(kThreads)
sell_spmv_kernel(uint64_t n_rows, const RP* __restrict__ rp, const uint64_t* __restrict__ soff,
                 const int32_t* __restrict__ sc, const double* __restrict__ sv, const double* __restrict__ x,
                 const double* __restrict__ b, double* __restrict__ y, int with_norm,
                 double* __restrict__ partials, unsigned* __restrict__ ticket, double* __restrict__ norm_out) {
    __shared__ double red[kWarps];
    const int lane = threadIdx.x & 31;
    double acc = 0.0;
    const uint64_t nsl = (n_rows + 31) / 32;
    for (uint64_t sl = (blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x) / 32; sl < nsl;
         sl += static_cast<uint64_t>(gridDim.x) * kWarps) {
        const uint64_t r = sl * 32 + lane;
        const bool live = r < n_rows;
        const uint32_t len = live ? static_cast<uint32_t>(__ldg(rp + r + 1) - __ldg(rp + r)) : 0u;
        const uint64_t off = __ldg(soff + sl);
        const uint32_t ml = static_cast<uint32_t>((__ldg(soff + sl + 1) - off) / 32);
        const double* v = sv + off + lane;
        const int32_t* c = sc + off + lane;
        double s = 0.0;
        for (uint32_t k = 0; k < ml; k += 8) {
            double vv[8], xv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const bool in = k + i < ml;
                const int32_t col = in ? __ldcs(c + (k + i) * 32) : 0;
                vv[i] = in ? __ldcs(v + (k + i) * 32) : 0.0;
                xv[i] = k + i < len ? __ldg(x + col) : 0.0;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (k + i < len) s = __dadd_rn(s, __dmul_rn(vv[i], xv[i]));
        }
        if (live) {
            if (MODE == 1) s = __dsub_rn(__ldg(b + r), s);
            y[r] = s;
            if (with_norm) acc = __dadd_rn(acc, __dmul_rn(s, s));
        }
    }
    if (!with_norm) return;
    acc = warp_sum(acc);
    if (lane == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    block_finalize(red, kWarps, 1, partials, ticket, norm_out);
}


// ------------------------------------------------------- staged CSR (TMA)
// Row tiles of TR rows (a power of two <= 256 chosen at setup so that no
// tile holds more than kTileEntries entries). One producer thread per CTA
// bulk-copies (cp.async.bulk, SASS UBLKCP) each tile's column indices,
// values and row offsets -- contiguous CSR segments -- into a kStages-deep
// shared-memory ring, keeping ~100 KB per CTA in flight independent of how
// many loads the consumer threads have outstanding. The consumers then
//   1. entry-parallel: p_k = RN(values[k] * x[col[k]]) for every entry of
//      the tile (conflict-free shared reads, x gathered through L2), written
//      back in place;
//   2. row-parallel: y[r] = ((0 + p_k0) + p_k0+1) + ... in row order.
// That is exactly the reference's mul-then-add sequence (sparse.cpp:50-52),
// so y is bit-identical to spmv(). The last <16 B of an array that a bulk
// copy cannot cover (end of allocation) is read directly from global.
#ifndef SPMV_TILE_ENTRIES
#define SPMV_TILE_ENTRIES 2048
#endif
#ifndef SPMV_STAGES
#define SPMV_STAGES 4
#endif
constexpr int kTileEntries = SPMV_TILE_ENTRIES;
constexpr int kSpmvStages = SPMV_STAGES;
constexpr int kSpmvConsumers = 256;
// Consumer groups take alternate tiles (measured on B200: one group of 8
// warps with 256-row tiles beats two groups with 128-row tiles -- the
// producer's per-tile cost dominates at smaller tiles).
#ifndef SPMV_GROUPS
#define SPMV_GROUPS 2
#endif
constexpr int kSpmvGroups = SPMV_GROUPS;
constexpr int kGroupThreads = kSpmvConsumers / kSpmvGroups;
constexpr int kTileRowsMax = 256;  // a group thread owns up to 256 / kGroupThreads rows of a tile
constexpr int kSpmvThreads = kSpmvConsumers + 32;

template <typename RP>
struct TileGeo {
    static constexpr uint32_t val_bytes = (kTileEntries + 2) * 8;
    static constexpr uint32_t col_bytes = (kTileEntries + 4) * 4;
    static constexpr uint32_t rp_bytes = (kTileRowsMax + 1 + 16 / sizeof(RP)) * sizeof(RP) + 16;
    static constexpr uint32_t stage = (val_bytes + col_bytes + rp_bytes + 127) / 128 * 128;
};

__device__ __forceinline__ void spmv_group_sync(int g) {
    if (g == 0) asm volatile("bar.sync 1, %0;" ::"n"(kGroupThreads) : "memory");
    else asm volatile("bar.sync 2, %0;" ::"n"(kGroupThreads) : "memory");
}

// Aligned window of a contiguous array segment [b, e) of element size ES:
// start aligned down to 16 B; bytes rounded down so the copy never reads
// past the array end `total` (elements beyond `got` are read from global).
template <int ES>
__device__ __forceinline__ void seg_window(uint64_t b, uint64_t e, uint64_t total, uint64_t& a0, uint32_t& bytes) {
    constexpr uint64_t per = 16 / ES;
    a0 = b / per * per;
    uint64_t a1 = (e + per - 1) / per * per;
    if (a1 > total) a1 = total / per * per;
    bytes = a1 > a0 ? static_cast<uint32_t>((a1 - a0) * ES) : 0u;
}

template <typename RP, int MODE>
__global__ void __launch_bounds__(kSpmvThreads)
spmv_tma_kernel(uint64_t n_rows, uint64_t nnz, uint32_t tile_rows, const RP* __restrict__ rp,
                const int32_t* __restrict__ ci, const double* __restrict__ va, const double* __restrict__ x,
                const double* __restrict__ b, double* __restrict__ y, int with_norm,
                double* __restrict__ partials, unsigned* __restrict__ ticket, double* __restrict__ norm_out) {
    using G = TileGeo<RP>;
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kSpmvStages * G::stage);
    uint64_t* empty = full + kSpmvStages;
    double* red = reinterpret_cast<double*>(empty + kSpmvStages);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kSpmvStages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kGroupThreads / 32);
        }
        fence_barrier_init();
    }
    __syncthreads();
    pdl_trigger();  // the orthogonalisation after us may launch (it waits for this grid)
    const uint64_t ntiles = (n_rows + tile_rows - 1) / tile_rows;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == kSpmvConsumers / 32) {
        // Producer warp: the entry ranges of the next 32 tiles are fetched
        // together (lane j: tile i0 + j), so issuing a tile never waits on a
        // dependent global load; lane 0 issues the bulk copies.
        const uint64_t policy = policy_evict_first();
        uint32_t i = 0;
        for (uint64_t tb = blockIdx.x; tb < ntiles; tb += 32ull * gridDim.x) {
            const uint64_t mt = tb + static_cast<uint64_t>(lane) * gridDim.x;
            uint64_t mk0 = 0, mk1 = 0;
            if (mt < ntiles) {
                const uint64_t r0 = mt * tile_rows, r1 = min(n_rows, r0 + tile_rows);
                mk0 = static_cast<uint64_t>(__ldg(rp + r0));
                mk1 = static_cast<uint64_t>(__ldg(rp + r1));
            }
            for (int j = 0; j < 32; ++j, ++i) {
                const uint64_t tile = tb + static_cast<uint64_t>(j) * gridDim.x;
                if (tile >= ntiles) break;
                const uint64_t k0 = __shfl_sync(0xFFFFFFFFu, mk0, j), k1 = __shfl_sync(0xFFFFFFFFu, mk1, j);
                if (lane == 0) {
                    const uint64_t r0 = tile * tile_rows, r1 = min(n_rows, r0 + tile_rows);
                    const int stage = i % kSpmvStages;
                    mbar_wait(empty + stage, ((i / kSpmvStages) & 1) ^ 1);
                    unsigned char* dst = smem + stage * G::stage;
                    uint64_t av, ac, ar;
                    uint32_t bv, bc, br;
                    seg_window<8>(k0, k1, nnz, av, bv);
                    seg_window<4>(k0, k1, nnz, ac, bc);
                    seg_window<sizeof(RP)>(r0, r1 + 1, n_rows + 1, ar, br);
                    mbar_arrive_expect_tx(full + stage, bv + bc + br);
                    if (bv) bulk_g2s(dst, va + av, bv, full + stage, policy);
                    if (bc) bulk_g2s(dst + G::val_bytes, ci + ac, bc, full + stage, policy);
                    if (br) bulk_g2s(dst + G::val_bytes + G::col_bytes, rp + ar, br, full + stage, policy);
                }
                __syncwarp();
            }
        }
        return;
    }
    // programmatic dependent of the orthogonalisation that wrote x: the
    // producer streams the (constant) matrix right away, the consumers wait
    // for the predecessor before gathering x or writing y
    pdl_wait();
    double acc = 0.0;
    const int g = warp / (kGroupThreads / 32);
    const uint32_t t = threadIdx.x % kGroupThreads;
    uint32_t i = g;
    for (uint64_t tile = blockIdx.x + static_cast<uint64_t>(g) * gridDim.x; tile < ntiles;
         tile += static_cast<uint64_t>(kSpmvGroups) * gridDim.x, i += kSpmvGroups) {
        const uint64_t r0 = tile * tile_rows, r1 = min(n_rows, r0 + tile_rows);
        const uint32_t nrows = static_cast<uint32_t>(r1 - r0);
        const int stage = i % kSpmvStages;
        unsigned char* st = smem + stage * G::stage;
        double* sv = reinterpret_cast<double*>(st);
        const int32_t* sc = reinterpret_cast<const int32_t*>(st + G::val_bytes);
        const RP* sr = reinterpret_cast<const RP*>(st + G::val_bytes + G::col_bytes);
        constexpr uint64_t pr = 16 / sizeof(RP);
        const uint32_t orr = static_cast<uint32_t>(r0 % pr);   // rp[r0] at sr[orr]
        mbar_wait(full + stage, (i / kSpmvStages) & 1);
        // Tail tile of the arrays (the bulk copies stop at the last whole
        // 16 B): uniform slow path straight from global memory.
        const bool tail = r1 + 1 > (n_rows + 1) / pr * pr;
        uint64_t k0, k1;
        if (!tail) {
            k0 = static_cast<uint64_t>(sr[orr]);
            k1 = static_cast<uint64_t>(sr[orr + nrows]);
        } else {
            k0 = static_cast<uint64_t>(__ldg(rp + r0));
            k1 = static_cast<uint64_t>(__ldg(rp + r1));
        }
        const bool gtail = tail || (k1 + 1) / 2 * 2 > nnz / 2 * 2 || (k1 + 3) / 4 * 4 > nnz / 4 * 4;
        if (gtail) {
            for (uint64_t r = r0 + t; r < r1; r += kGroupThreads) {
                const uint64_t a = static_cast<uint64_t>(__ldg(rp + r)), e = static_cast<uint64_t>(__ldg(rp + r + 1));
                double s = 0.0;
                for (uint64_t k = a; k < e; ++k) s = __dadd_rn(s, __dmul_rn(__ldg(va + k), __ldg(x + __ldg(ci + k))));
                if (MODE == 1) s = __dsub_rn(__ldg(b + r), s);
                y[r] = s;
                if (with_norm) acc = __dadd_rn(acc, __dmul_rn(s, s));
            }
        } else {
            const uint32_t ov = static_cast<uint32_t>(k0 & 1), oc = static_cast<uint32_t>(k0 & 3);
            const uint32_t base = static_cast<uint32_t>(k0);  // low bits: in-tile offsets only
            if constexpr (true) {
                if (tile_rows >= static_cast<uint32_t>(kGroupThreads)) {
                    // short rows: one thread per row (two interleaved rows,
                    // lr and lr + kGroupThreads, when the tile has 2x the
                    // group's threads), loads for up to 8 entries of each row
                    // issued together, products added in row order
                    for (uint32_t lr = t; lr < nrows; lr += 2 * kGroupThreads) {
                        const uint32_t lr2 = lr + kGroupThreads;
                        const bool two = lr2 < nrows;
                        const uint32_t a = static_cast<uint32_t>(sr[orr + lr]) - base;
                        const uint32_t e = static_cast<uint32_t>(sr[orr + lr + 1]) - base;
                        const uint32_t a2 = two ? static_cast<uint32_t>(sr[orr + lr2]) - base : 0u;
                        const uint32_t e2 = two ? static_cast<uint32_t>(sr[orr + lr2 + 1]) - base : 0u;
                        double s = 0.0, s2 = 0.0;
                        const uint32_t len = max(e - a, e2 - a2);
                        for (uint32_t k = 0; k < len; k += 8) {
                            int32_t c[8], c2[8];
                            double v[8], xv[8], v2[8], xv2[8];
#pragma unroll
                            for (int u = 0; u < 8; ++u) {
                                const bool in = a + k + u < e, in2 = a2 + k + u < e2;
                                c[u] = in ? sc[a + k + u + oc] : 0;
                                v[u] = in ? sv[a + k + u + ov] : 0.0;
                                c2[u] = in2 ? sc[a2 + k + u + oc] : 0;
                                v2[u] = in2 ? sv[a2 + k + u + ov] : 0.0;
                            }
#pragma unroll
                            for (int u = 0; u < 8; ++u) {
                                xv[u] = a + k + u < e ? __ldg(x + c[u]) : 0.0;
                                xv2[u] = a2 + k + u < e2 ? __ldg(x + c2[u]) : 0.0;
                            }
#pragma unroll
                            for (int u = 0; u < 8; ++u) {
                                if (a + k + u < e) s = __dadd_rn(s, __dmul_rn(v[u], xv[u]));
                                if (a2 + k + u < e2) s2 = __dadd_rn(s2, __dmul_rn(v2[u], xv2[u]));
                            }
                        }
                        const uint64_t r = r0 + lr;
                        if (MODE == 1) s = __dsub_rn(__ldg(b + r), s);
                        y[r] = s;
                        if (with_norm) acc = __dadd_rn(acc, __dmul_rn(s, s));
                        if (two) {
                            const uint64_t rr = r0 + lr2;
                            if (MODE == 1) s2 = __dsub_rn(__ldg(b + rr), s2);
                            y[rr] = s2;
                            if (with_norm) acc = __dadd_rn(acc, __dmul_rn(s2, s2));
                        }
                    }
                } else {
                    // long rows: products entry-parallel (in place), then
                    // the row sums in order
                    const uint32_t cnt = static_cast<uint32_t>(k1 - k0);
                    for (uint32_t e0 = t; e0 < cnt; e0 += 8 * kGroupThreads) {
                        int32_t c[8];
                        double v[8], xv[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const uint32_t e = e0 + u * kGroupThreads;
                            c[u] = e < cnt ? sc[e + oc] : 0;
                            v[u] = e < cnt ? sv[e + ov] : 0.0;
                        }
#pragma unroll
                        for (int u = 0; u < 8; ++u) xv[u] = e0 + u * kGroupThreads < cnt ? __ldg(x + c[u]) : 0.0;
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const uint32_t e = e0 + u * kGroupThreads;
                            if (e < cnt) sv[e + ov] = __dmul_rn(v[u], xv[u]);
                        }
                    }
                    spmv_group_sync(g);
                    for (uint32_t lr = t; lr < nrows; lr += kGroupThreads) {
                        const uint32_t a = static_cast<uint32_t>(sr[orr + lr]) - base + ov;
                        const uint32_t e = static_cast<uint32_t>(sr[orr + lr + 1]) - base + ov;
                        double s = 0.0;
                        for (uint32_t k = a; k < e; ++k) s = __dadd_rn(s, sv[k]);
                        const uint64_t r = r0 + lr;
                        if (MODE == 1) s = __dsub_rn(__ldg(b + r), s);
                        y[r] = s;
                        if (with_norm) acc = __dadd_rn(acc, __dmul_rn(s, s));
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + stage);
    }
    if (!with_norm) return;
    acc = warp_sum(acc);
    if (lane == 0) red[warp] = acc;
    // the producer warp has exited (or exits without waiting on anything):
    // __syncthreads counts only the remaining threads
    __syncthreads();
    block_finalize(red, kSpmvConsumers / 32, 1, partials, ticket, norm_out);
}



__global__ void __launch_bounds__(kThreads)
dot_kernel(const double* __restrict__ x, const double* __restrict__ y, uint64_t n,
           double* __restrict__ partials, unsigned* __restrict__ ticket, double* __restrict__ out,
           GateArg gate) {
    if (!gate.open()) return;
    __shared__ double red[kWarps];
    double acc = 0.0;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * kThreads)
        acc = __dadd_rn(acc, __dmul_rn(x[i], y[i]));
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    block_finalize(red, kWarps, 1, partials, ticket, out);
}

__global__ void serial_dot_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                  uint64_t n, double* __restrict__ out, GateArg gate) {
    if (!gate.open()) return;
    double s = 0.0;
    for (uint64_t i = 0; i < n; ++i) s = __dadd_rn(s, __dmul_rn(x[i], y[i]));
    *out = s;
}

__global__ void scale_kernel(double a, double* __restrict__ x, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        x[i] = __dmul_rn(x[i], a);
}

__global__ void axpy_kernel(double a, const double* __restrict__ x, double* __restrict__ y, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        y[i] = __dadd_rn(y[i], __dmul_rn(a, x[i]));
}

// ------------------------------------------------------ stencils
struct Grid3 {
    uint64_t nx, ny, nz;
};

__host__ __device__ __forceinline__ int stencil_count(int kind, Grid3 g, uint64_t row) {
    const uint64_t x = row % g.nx, y = (row / g.nx) % g.ny, z = row / (g.nx * g.ny);
    const int cx = 1 + (x > 0) + (x + 1 < g.nx);
    const int cy = 1 + (y > 0) + (y + 1 < g.ny);
    const int cz = 1 + (z > 0) + (z + 1 < g.nz);
    return kind == 2 ? cx * cy * cz : (cx + cy + cz - 2);
}

template <typename RP>
__global__ void stencil_count_kernel(int kind, Grid3 g, uint64_t row_begin, uint64_t rows,
                                     RP* __restrict__ counts) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i <= rows;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        counts[i] = i < rows ? static_cast<RP>(stencil_count(kind, g, row_begin + i)) : RP(0);
}

// Emits row entries in ascending column order (dz, dy, dx lexicographic),
// the 3-D analogue of gen_convdiff's S, W, C, E, N order (sparse.cpp:265-286).
template <typename RP>
__global__ void stencil_fill_kernel(int kind, Grid3 g, double pe, uint64_t row_begin, uint64_t rows,
                                    int64_t col_offset, const RP* __restrict__ rp,
                                    int32_t* __restrict__ ci, double* __restrict__ va) {
    const double centre = kind == 0 ? 6.0 : (kind == 1 ? 6.0 + 3.0 * pe : 26.0);
    const double upwind = kind == 1 ? -(1.0 + pe) : -1.0;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < rows;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t row = row_begin + i;
        const int64_t x = row % g.nx, y = (row / g.nx) % g.ny, z = row / (g.nx * g.ny);
        uint64_t k = static_cast<uint64_t>(rp[i]);
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int nzc = (dx != 0) + (dy != 0) + (dz != 0);
                    if (kind != 2 && nzc > 1) continue;
                    if (x + dx < 0 || x + dx >= static_cast<int64_t>(g.nx)) continue;
                    if (y + dy < 0 || y + dy >= static_cast<int64_t>(g.ny)) continue;
                    if (z + dz < 0 || z + dz >= static_cast<int64_t>(g.nz)) continue;
                    const int64_t col = static_cast<int64_t>(row) +
                                        (dz * static_cast<int64_t>(g.ny) + dy) * static_cast<int64_t>(g.nx) + dx;
                    double v = -1.0;
                    if (nzc == 0) v = centre;
                    else if (dx < 0 || dy < 0 || dz < 0) v = upwind;
                    ci[k] = static_cast<int32_t>(col - col_offset);
                    va[k] = v;
                    ++k;
                }
    }
}

template <typename RP>
void stencil_generate(int kind, Grid3 g, double pe, uint64_t rb, uint64_t re, int64_t col_offset,
                      RP* rp, int32_t* ci, double* va, cudaStream_t st) {
    const uint64_t rows = re - rb;
    const int grid = static_cast<int>(std::min<uint64_t>((rows + 256) / 256 + 1, sm_count() * 16ull));
    CBGX_K(stencil_count_kernel<RP><<<grid, 256, 0, st>>>(kind, g, rb, rows, rp));
    CBGX_CUDA(cudaGetLastError());
    size_t tmp_bytes = 0;
    CBGX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, rp, rp, rows + 1, st));
    void* tmp = nullptr;
    CBGX_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
    CBGX_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, rp, rp, rows + 1, st));
    CBGX_CUDA(cudaFreeAsync(tmp, st));
    CBGX_K(stencil_fill_kernel<RP><<<grid, 256, 0, st>>>(kind, g, pe, rb, rows, col_offset, rp, ci, va));
    CBGX_CUDA(cudaGetLastError());
}

void check_csr(const cbgx_csr* A) {
    if (!A) throw Error(CBGX_EINVAL, "csr: null matrix");
    if (A->row_ptr_bits != 32 && A->row_ptr_bits != 64) throw Error(CBGX_EINVAL, "csr: row_ptr_bits must be 32 or 64");
    if (A->row_ptr_bits == 32 && A->nnz > 0x7FFFFFFFull) throw Error(CBGX_EINVAL, "csr: nnz needs 64-bit row_ptr");
}

}  // namespace

void launch_spmv(const cbgx_csr& A, const double* x, const double* b, double* y, double* norm,
                 int reduction, Workspace* ws, cudaStream_t st) {
    const int grid = rows_grid(A.n_rows);
    const bool fused = norm && reduction == CBGX_REDUCE_TREE;
    double* partials = fused ? ws->get_partials(grid) : nullptr;
    unsigned* ticket = fused ? ws->get_counter() : nullptr;
#define CBGX_SPMV(RP, MODE)                                                                     \
    CBGX_K(spmv_kernel<RP, MODE><<<grid, kThreads, 0, st>>>(A.n_rows, static_cast<const RP*>(A.d_row_ptr), \
                                                     A.d_col_idx, A.d_values, x, b, y, fused,     \
                                                     partials, ticket, norm))
    if (A.row_ptr_bits == 32) {
        if (b) CBGX_SPMV(int32_t, 1); else CBGX_SPMV(int32_t, 0);
    } else {
        if (b) CBGX_SPMV(int64_t, 1); else CBGX_SPMV(int64_t, 0);
    }
#undef CBGX_SPMV
    CBGX_CUDA(cudaGetLastError());
    if (norm && !fused) launch_dot(y, y, A.n_rows, CBGX_REDUCE_REFERENCE, norm, ws, st);
}

Sell::~Sell() {
    if (val) cudaFree(val);
    if (col) cudaFree(col);
    if (soff) cudaFree(soff);
}

template <typename RP>
static void sell_build(const cbgx_csr& A, Sell& S, cudaStream_t st) {
    const RP* rp = static_cast<const RP*>(A.d_row_ptr);
    S.nslices = (A.n_rows + 31) / 32;
    CBGX_CUDA(cudaMalloc(&S.soff, (S.nslices + 1) * sizeof(uint64_t)));
    const int g1 = static_cast<int>(std::min<uint64_t>((S.nslices + 1 + 7) / 8 + 1, sm_count() * 16ull));
    CBGX_K(sell_len_kernel<RP><<<g1, 256, 0, st>>>(rp, A.n_rows, S.nslices, S.soff));
    size_t tmp_bytes = 0;
    CBGX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, S.soff, S.soff, S.nslices + 1, st));
    void* tmp = nullptr;
    CBGX_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
    CBGX_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, S.soff, S.soff, S.nslices + 1, st));
    CBGX_CUDA(cudaFreeAsync(tmp, st));
    uint64_t total = 0;
    CBGX_CUDA(cudaMemcpyAsync(&total, S.soff + S.nslices, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    CBGX_CUDA(cudaStreamSynchronize(st));
    S.entries = total;
    CBGX_CUDA(cudaMalloc(&S.val, std::max<uint64_t>(total, 1) * 8));
    CBGX_CUDA(cudaMalloc(&S.col, std::max<uint64_t>(total, 1) * 4));
    const int g2 = rows_grid(S.nslices * 32);
    CBGX_K(sell_fill_kernel<RP><<<g2, kThreads, 0, st>>>(rp, A.d_col_idx, A.d_values, A.n_rows, S.soff, S.val, S.col));
    CBGX_CUDA(cudaStreamSynchronize(st));
}

std::unique_ptr<Sell> build_sell(const cbgx_csr& A, double max_fraction_of_free, cudaStream_t st) {
    size_t free_b = 0, total_b = 0;
    CBGX_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const double need = (A.nnz * 1.05 + 32.0 * ((A.n_rows + 31) / 32)) * 12.0;
    if (need > max_fraction_of_free * static_cast<double>(free_b)) return nullptr;
    auto S = std::make_unique<Sell>();
    if (A.row_ptr_bits == 32) sell_build<int32_t>(A, *S, st);
    else sell_build<int64_t>(A, *S, st);
    return S;
}

void launch_spmv_sell(const cbgx_csr& A, const Sell& S, const double* x, const double* b, double* y, double* norm,
                      int reduction, Workspace* ws, cudaStream_t st) {
    const int grid = rows_grid(A.n_rows);
    const bool fused = norm && reduction == CBGX_REDUCE_TREE;
    double* partials = fused ? ws->get_partials(grid) : nullptr;
    unsigned* ticket = fused ? ws->get_counter() : nullptr;
#define CBGX_SELL(RP, MODE)                                                                                   \
    CBGX_K(sell_spmv_kernel<RP, MODE><<<grid, kThreads, 0, st>>>(A.n_rows, static_cast<const RP*>(A.d_row_ptr), \
                                                                S.soff, S.col, S.val, x, b, y, fused, partials, \
                                                                ticket, norm))
    if (A.row_ptr_bits == 32) {
        if (b) CBGX_SELL(int32_t, 1); else CBGX_SELL(int32_t, 0);
    } else {
        if (b) CBGX_SELL(int64_t, 1); else CBGX_SELL(int64_t, 0);
    }
#undef CBGX_SELL
    CBGX_CUDA(cudaGetLastError());
    if (norm && !fused) launch_dot(y, y, A.n_rows, CBGX_REDUCE_REFERENCE, norm, ws, st);
}


// One pass over the row offsets: longest row and the largest entry count of
// any 32/64/128/256-row tile (blocks of 256 threads own aligned 256-row
// tiles). out: [max_row, t32, t64, t128, t256], zeroed by the caller.
template <typename RP>
__global__ void __launch_bounds__(256) csr_stats_kernel(const RP* __restrict__ rp, uint64_t n,
                                                        unsigned long long* __restrict__ out) {
    __shared__ unsigned long long t32[8];
    unsigned long long mrow = 0, m[4] = {0, 0, 0, 0};
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint64_t base = blockIdx.x * 256ull; base < n; base += 256ull * gridDim.x) {
        const uint64_t r = base + threadIdx.x;
        const uint64_t a = r < n ? static_cast<uint64_t>(rp[r]) : 0, e = r < n ? static_cast<uint64_t>(rp[r + 1]) : 0;
        mrow = max(mrow, static_cast<unsigned long long>(e - a));
        if (lane == 0) {
            const uint64_t r0 = min(n, base + static_cast<uint64_t>(32 * warp)), r1 = min(n, base + static_cast<uint64_t>(32 * warp + 32));
            t32[warp] = static_cast<unsigned long long>(rp[r1] - rp[r0]);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long c[8];
            for (int g = 0; g < 8; ++g) c[g] = t32[g];
            for (int g = 0; g < 8; ++g) m[0] = max(m[0], c[g]);
            for (int g = 0; g < 8; g += 2) m[1] = max(m[1], c[g] + c[g + 1]);
            for (int g = 0; g < 8; g += 4) m[2] = max(m[2], c[g] + c[g + 1] + c[g + 2] + c[g + 3]);
            m[3] = max(m[3], c[0] + c[1] + c[2] + c[3] + c[4] + c[5] + c[6] + c[7]);
        }
        __syncthreads();
    }
    for (int o = 16; o > 0; o >>= 1) mrow = max(mrow, __shfl_xor_sync(0xFFFFFFFFu, mrow, o));
    if (lane == 0) atomicMax(out, mrow);
    if (threadIdx.x == 0)
        for (int i = 0; i < 4; ++i) atomicMax(out + 1 + i, m[i]);
}

void launch_csr_stats(const cbgx_csr& A, unsigned long long* d_out, cudaStream_t st) {
    CBGX_CUDA(cudaMemsetAsync(d_out, 0, 5 * sizeof(unsigned long long), st));
    if (A.n_rows == 0) return;
    const int grid = rows_grid((A.n_rows + 255) / 256);
    if (A.row_ptr_bits == 32)
        CBGX_K(csr_stats_kernel<int32_t><<<grid, 256, 0, st>>>(static_cast<const int32_t*>(A.d_row_ptr), A.n_rows, d_out));
    else
        CBGX_K(csr_stats_kernel<int64_t><<<grid, 256, 0, st>>>(static_cast<const int64_t*>(A.d_row_ptr), A.n_rows, d_out));
    CBGX_CUDA(cudaGetLastError());
}

uint32_t plan_from_stats(const unsigned long long* h) {
    for (int i = 3; i >= 0; --i)
        if ((32 << i) <= kTileRowsMax && h[1 + i] <= static_cast<unsigned long long>(kTileEntries)) return 32u << i;
    return 0;
}

static void csr_stats_sync(const cbgx_csr& A, unsigned long long h[5], cudaStream_t st) {
    unsigned long long* d = nullptr;
    CBGX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), 5 * sizeof(unsigned long long), st));
    launch_csr_stats(A, d, st);
    CBGX_CUDA(cudaMemcpyAsync(h, d, 5 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CBGX_CUDA(cudaFreeAsync(d, st));
    CBGX_CUDA(cudaStreamSynchronize(st));
}

uint32_t plan_spmv_tiles(const cbgx_csr& A, cudaStream_t st) {
    if (A.n_rows == 0) return 0;
    unsigned long long h[5];
    csr_stats_sync(A, h, st);
    return plan_from_stats(h);
}

template <typename RP, int MODE>
static void spmv_tma_launch(const cbgx_csr& A, uint32_t tile_rows, const double* x, const double* b, double* y,
                            int fused, double* norm, Workspace* ws, cudaStream_t st, bool pdl) {
    static int per_sm = -1;  // per (RP, MODE) instantiation; one device geometry
    const size_t smem = kSpmvStages * (TileGeo<RP>::stage + 16) + 64;
    if (per_sm < 0) {
        CBGX_CUDA(cudaFuncSetAttribute(spmv_tma_kernel<RP, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)));
        CBGX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, spmv_tma_kernel<RP, MODE>, kSpmvThreads, smem));
        per_sm = std::max(per_sm, 1);
    }
    const uint64_t ntiles = (A.n_rows + tile_rows - 1) / tile_rows;
    const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(ntiles, static_cast<uint64_t>(sm_count()) * per_sm)));
    double* partials = fused ? ws->get_partials(grid) : nullptr;
    unsigned* ticket = fused ? ws->get_counter() : nullptr;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(kSpmvThreads);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = pdl ? 1 : 0;
    note_launch();
    CBGX_CUDA(cudaLaunchKernelEx(&lc, spmv_tma_kernel<RP, MODE>, A.n_rows, A.nnz, tile_rows,
                                 static_cast<const RP*>(A.d_row_ptr), A.d_col_idx, A.d_values, x, b, y, fused,
                                 partials, ticket, norm));
}

void launch_spmv_tma(const cbgx_csr& A, uint32_t tile_rows, const double* x, const double* b, double* y,
                     double* norm, int reduction, Workspace* ws, cudaStream_t st, bool pdl) {
    const int fused = norm && reduction == CBGX_REDUCE_TREE;
    if (A.row_ptr_bits == 32) {
        if (b) spmv_tma_launch<int32_t, 1>(A, tile_rows, x, b, y, fused, norm, ws, st, pdl);
        else spmv_tma_launch<int32_t, 0>(A, tile_rows, x, b, y, fused, norm, ws, st, pdl);
    } else {
        if (b) spmv_tma_launch<int64_t, 1>(A, tile_rows, x, b, y, fused, norm, ws, st, pdl);
        else spmv_tma_launch<int64_t, 0>(A, tile_rows, x, b, y, fused, norm, ws, st, pdl);
    }
    CBGX_CUDA(cudaGetLastError());
    if (norm && !fused) launch_dot(y, y, A.n_rows, CBGX_REDUCE_REFERENCE, norm, ws, st);
}

uint32_t csr_max_row_nnz(const cbgx_csr& A, cudaStream_t st) {
    if (A.n_rows == 0) return 0;
    unsigned long long h[5];
    csr_stats_sync(A, h, st);
    return static_cast<uint32_t>(h[0]);
}

void launch_dot(const double* x, const double* y, uint64_t n, int reduction, double* out,
                Workspace* ws, cudaStream_t st, const GateArg& gate) {
    if (reduction == CBGX_REDUCE_REFERENCE) {
        CBGX_K(serial_dot_kernel<<<1, 1, 0, st>>>(x, y, n, out, gate));
    } else {
        const int grid = rows_grid(n);
        CBGX_K(dot_kernel<<<grid, kThreads, 0, st>>>(x, y, n, ws->get_partials(grid), ws->get_counter(), out, gate));
    }
    CBGX_CUDA(cudaGetLastError());
}

}  // namespace cbgx

using namespace cbgx;

extern "C" {

int cbgx_csr_spmv(const cbgx_csr* A, const double* d_x, double* d_y, double* d_ynorm2, int reduction,
                  cbgx_workspace* ws, void* stream) {
    return guard([&] {
        check_csr(A);
        if (d_ynorm2 && !ws) throw Error(CBGX_EINVAL, "spmv: fused norm needs a workspace");
        launch_spmv(*A, d_x, nullptr, d_y, d_ynorm2, reduction, ws_of(ws), as_stream(stream));
    });
}

int cbgx_csr_spmv_plan(const cbgx_csr* A, uint32_t* tile_rows, void* stream) {
    return guard([&] {
        check_csr(A);
        if (!tile_rows) throw Error(CBGX_EINVAL, "spmv: null output");
        *tile_rows = plan_spmv_tiles(*A, as_stream(stream));
    });
}

int cbgx_csr_spmv_staged(const cbgx_csr* A, uint32_t tile_rows, const double* d_x, const double* d_b,
                         double* d_y, double* d_ynorm2, int reduction, cbgx_workspace* ws, void* stream) {
    return guard([&] {
        check_csr(A);
        if (tile_rows < 32 || tile_rows > static_cast<uint32_t>(kTileRowsMax) || (tile_rows & (tile_rows - 1)))
            throw Error(CBGX_EINVAL, "spmv: tile_rows must be a power of two in [32, 256]");
        if (d_ynorm2 && !ws) throw Error(CBGX_EINVAL, "spmv: fused norm needs a workspace");
        if (A->n_rows == 0) return;
        launch_spmv_tma(*A, tile_rows, d_x, d_b, d_y, d_ynorm2, reduction, ws_of(ws), as_stream(stream));
    });
}

int cbgx_csr_residual(const cbgx_csr* A, const double* d_x, const double* d_b, double* d_r,
                      double* d_rnorm2, int reduction, cbgx_workspace* ws, void* stream) {
    return guard([&] {
        check_csr(A);
        if (!d_b) throw Error(CBGX_EINVAL, "residual: null b");
        if (d_rnorm2 && !ws) throw Error(CBGX_EINVAL, "residual: fused norm needs a workspace");
        launch_spmv(*A, d_x, d_b, d_r, d_rnorm2, reduction, ws_of(ws), as_stream(stream));
    });
}

int cbgx_dot(const double* d_x, const double* d_y, uint64_t n, int reduction, double* d_out,
             cbgx_workspace* ws, void* stream) {
    return guard([&] {
        if (reduction == CBGX_REDUCE_TREE && !ws) throw Error(CBGX_EINVAL, "dot: null workspace");
        launch_dot(d_x, d_y, n, reduction, d_out, ws_of(ws), as_stream(stream));
    });
}

int cbgx_scale(double alpha, double* d_x, uint64_t n, void* stream) {
    return guard([&] {
        if (!n) return;
        CBGX_K(scale_kernel<<<rows_grid(n), kThreads, 0, as_stream(stream)>>>(alpha, d_x, n));
        CBGX_CUDA(cudaGetLastError());
    });
}

int cbgx_axpy(double alpha, const double* d_x, double* d_y, uint64_t n, void* stream) {
    return guard([&] {
        if (!n) return;
        CBGX_K(axpy_kernel<<<rows_grid(n), kThreads, 0, as_stream(stream)>>>(alpha, d_x, d_y, n));
        CBGX_CUDA(cudaGetLastError());
    });
}

uint64_t cbgx_stencil_nnz(int kind, uint64_t nx, uint64_t ny, uint64_t nz, uint64_t rb, uint64_t re) {
    // Partial x-lines row by row, whole x-lines in closed form:
    // sum_x cx = 3nx - 2 (nx >= 1).
    const Grid3 g{nx, ny, nz};
    if (nx == 0 || ny == 0 || nz == 0 || rb >= re) return 0;
    uint64_t total = 0;
    uint64_t row = rb;
    while (row < re) {
        const uint64_t x = row % nx;
        if (x == 0 && row + nx <= re) {
            const uint64_t y = (row / nx) % ny, z = row / (nx * ny);
            const uint64_t cy = 1 + (y > 0) + (y + 1 < ny), cz = 1 + (z > 0) + (z + 1 < nz);
            const uint64_t sx = 3 * nx - 2;
            total += kind == 2 ? sx * cy * cz : sx + nx * (cy + cz - 2);
            row += nx;
        } else {
            total += static_cast<uint64_t>(stencil_count(kind, g, row));
            ++row;
        }
    }
    return total;
}

int cbgx_stencil_generate(int kind, uint64_t nx, uint64_t ny, uint64_t nz, double pe, uint64_t rb,
                          uint64_t re, int64_t col_offset, void* d_row_ptr, uint32_t bits,
                          int32_t* d_col_idx, double* d_values, void* stream) {
    return guard([&] {
        if (kind < 0 || kind > 2) throw Error(CBGX_EINVAL, "stencil: kind must be 0, 1 or 2");
        if (rb > re || re > nx * ny * nz) throw Error(CBGX_ERANGE, "stencil: bad row range");
        const Grid3 g{nx, ny, nz};
        if (bits == 32) stencil_generate(kind, g, pe, rb, re, col_offset, static_cast<int32_t*>(d_row_ptr), d_col_idx, d_values, as_stream(stream));
        else if (bits == 64) stencil_generate(kind, g, pe, rb, re, col_offset, static_cast<int64_t*>(d_row_ptr), d_col_idx, d_values, as_stream(stream));
        else throw Error(CBGX_EINVAL, "stencil: row_ptr_bits must be 32 or 64");
    });
}

}  // extern "C"
