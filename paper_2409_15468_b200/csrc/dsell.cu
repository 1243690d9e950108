// dsell.cu -- dictionary-coded SELL-32 SpMV ("DSELL").
//
// The SpMV of the reference (sparse.cpp:43-56) streams 12 B per entry (8 B
// value + 4 B column) on the device -- for the structured-grid systems of
// the paper's configurations (7/27-point stencils, 5-point convection-
// diffusion) that is all the solver reads besides the basis. Those matrices
// hold a handful of distinct values and a handful of distinct column offsets
// (col - row). At setup the solver detects that (at most 255 of each) and
// builds a SELL-32 copy whose entries are 2-byte codes
//     code = value_index << 8 | offset_index      (0xFFFF = slice padding)
// into two tiny dictionaries kept in shared memory, so an entry costs 2 B of
// HBM instead of 12 (6x fewer matrix bytes). Entry k of row 32s + lane sits
// at soff[s] + 32 k + lane (coalesced 64-B warp loads), entries keep their
// in-row order, and the decoded (value, column) pairs are exactly the CSR's,
// so y is bit-identical to spmv() (products and sums in row order, separate
// roundings). Matrices outside the pattern (more distinct values/offsets,
// halo-remapped columns) keep the CSR paths.
//
// Three further levels, each built from the previous one when it applies
// (cbgx_csr_dict_create2 caps the level):
//   pair codes    <= 255 distinct (value, offset) pairs: 1 byte per entry
//                 (pell_spmv_kernel);
//   row patterns  <= 255 distinct rows of pair codes: 1 byte per ROW into
//                 per-pattern {offsets, values} tables (ppat_spmv_kernel);
//   uniform slots the patterns' offsets embed into one sorted list of <= 32
//                 slots with one value each (constant coefficients): a slot
//                 mask per pattern, offsets/values as kernel parameters
//                 (uslot_spmv_kernel) -- the solver's SpMV on every stencil
//                 configuration.
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "pipeline.cuh"
#include "reduce.cuh"
#include "runtime.h"

namespace cbgx {

namespace {

constexpr int kDThreads = 256;
constexpr int kDWarps = kDThreads / 32;
constexpr uint32_t kSlots = 1024;         // open-addressing hash tables (keys are u64)
constexpr uint32_t kDictMax = 255;        // entries per dictionary (index 255 unused)
constexpr uint16_t kPad = 0xFFFF;
constexpr unsigned long long kEmpty = ~0ull;

__device__ __forceinline__ uint32_t hslot(unsigned long long key) {
    return static_cast<uint32_t>((key * 0x9E3779B97F4A7C15ull) >> 54);  // 10 bits
}
// column offsets are stored biased by 2^32 (never equal to kEmpty)
__device__ __forceinline__ unsigned long long off_key(int64_t off) {
    return static_cast<unsigned long long>(off + (1ll << 32));
}

// Insert `key` (idempotent). false: the table already holds kDictMax keys.
__device__ bool table_insert(unsigned long long* tab, unsigned long long key, unsigned* count) {
    uint32_t h = hslot(key);
    for (uint32_t p = 0; p < kSlots; ++p) {
        unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(tab + h);
        if (cur == key) return true;
        if (cur == kEmpty) {
            cur = atomicCAS(tab + h, kEmpty, key);
            if (cur == kEmpty) return atomicAdd(count, 1u) < kDictMax;
            if (cur == key) return true;
        }
        h = (h + 1) & (kSlots - 1);
    }
    return false;
}

__device__ __forceinline__ uint32_t table_find(const unsigned long long* tab, unsigned long long key) {
    uint32_t h = hslot(key);
    while (tab[h] != key) h = (h + 1) & (kSlots - 1);
    return h;
}

// Pass 1: the distinct column offsets and values. Every CTA dedups into its
// own shared tables (warp-level match first), then merges them into the
// global ones; any overflow (or an offset outside int32, or a value whose
// bits equal the empty marker) sets *bad and the matrix keeps CSR.
template <typename RP>
__global__ void __launch_bounds__(kDThreads)
dict_scan_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ ci, const double* __restrict__ va,
                 uint64_t n_rows, unsigned long long* __restrict__ g_off, unsigned long long* __restrict__ g_val,
                 unsigned* __restrict__ g_cnt, unsigned* __restrict__ bad) {
    __shared__ unsigned long long s_off[kSlots], s_val[kSlots];
    __shared__ unsigned s_cnt[2];
    for (uint32_t i = threadIdx.x; i < kSlots; i += kDThreads) s_off[i] = s_val[i] = kEmpty;
    if (threadIdx.x < 2) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    // Warp-uniform loops (the lanes of a warp share the row base; rows past
    // n and entries past a row's end take part as inactive lanes), so every
    // __match_any_sync below is reached by all 32 lanes together.
    bool ok = true;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kDThreads;
    const int lane = threadIdx.x & 31;
    for (uint64_t r0 = blockIdx.x * static_cast<uint64_t>(kDThreads) + (threadIdx.x & ~31u); r0 < n_rows;
         r0 += stride) {
        if (!__all_sync(0xFFFFFFFFu, ok) || *reinterpret_cast<volatile unsigned*>(bad)) {
            ok = false;
            break;
        }
        const uint64_t r = r0 + lane;
        const bool row = r < n_rows;
        const uint64_t k0 = row ? static_cast<uint64_t>(rp[r]) : 0, k1 = row ? static_cast<uint64_t>(rp[r + 1]) : 0;
        const unsigned len = static_cast<unsigned>(k1 - k0);
        const unsigned wlen = __reduce_max_sync(0xFFFFFFFFu, len);
        for (unsigned k = 0; k < wlen; ++k) {
            bool act = k < len;
            unsigned long long ko = kEmpty, kv = kEmpty;
            if (act) {
                const int64_t off = static_cast<int64_t>(ci[k0 + k]) - static_cast<int64_t>(r);
                ko = off_key(off);
                kv = static_cast<unsigned long long>(__double_as_longlong(va[k0 + k]));
                if (off < INT32_MIN || off > INT32_MAX || kv == kEmpty) {
                    ok = false;
                    act = false;
                    ko = kv = kEmpty;
                }
            }
            // inactive lanes carry the empty key: they group together and
            // never insert
            const unsigned mo = __match_any_sync(0xFFFFFFFFu, ko), mv = __match_any_sync(0xFFFFFFFFu, kv);
            if (act && __ffs(mo) - 1 == lane) ok = table_insert(s_off, ko, &s_cnt[0]) && ok;
            if (act && __ffs(mv) - 1 == lane) ok = table_insert(s_val, kv, &s_cnt[1]) && ok;
        }
    }
    if (!ok) atomicExch(bad, 1u);
    __syncthreads();
    if (*reinterpret_cast<volatile unsigned*>(bad)) return;
    for (uint32_t i = threadIdx.x; i < kSlots; i += kDThreads) {
        bool fine = true;
        if (s_off[i] != kEmpty) fine = table_insert(g_off, s_off[i], &g_cnt[0]);
        if (s_val[i] != kEmpty) fine = fine && table_insert(g_val, s_val[i], &g_cnt[1]);
        if (!fine) atomicExch(bad, 1u);
    }
}

// Per-slice width (longest row of the 32) in entries * 32.
template <typename RP>
__global__ void dict_slice_kernel(const RP* __restrict__ rp, uint64_t n, uint64_t nslices, uint64_t* __restrict__ slen,
                                  unsigned* __restrict__ max_w) {
    for (uint64_t sl = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) / 32; sl < nslices + 1;
         sl += static_cast<uint64_t>(gridDim.x) * blockDim.x / 32) {
        const int lane = threadIdx.x & 31;
        const uint64_t r = sl * 32 + lane;
        const unsigned len = (sl < nslices && r < n) ? static_cast<unsigned>(rp[r + 1] - rp[r]) : 0u;
        const unsigned m = __reduce_max_sync(0xFFFFFFFFu, len);
        if (lane == 0) {
            slen[sl] = static_cast<uint64_t>(m) * 32;
            atomicMax(max_w, m);
        }
    }
}

// Pass 2: the codes, slice-major (entry k of row 32s+lane at soff[s]+32k+lane).
template <typename RP>
__global__ void __launch_bounds__(kDThreads)
dict_fill_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ ci, const double* __restrict__ va,
                 uint64_t n_rows, const uint64_t* __restrict__ soff, const unsigned long long* __restrict__ g_off,
                 const unsigned long long* __restrict__ g_val, const uint8_t* __restrict__ off_idx,
                 const uint8_t* __restrict__ val_idx, uint32_t ell4, uint16_t* __restrict__ codes,
                 unsigned* __restrict__ too_long) {
    __shared__ unsigned long long s_off[kSlots], s_val[kSlots];
    __shared__ uint8_t s_oi[kSlots], s_vi[kSlots];
    for (uint32_t i = threadIdx.x; i < kSlots; i += kDThreads) {
        s_off[i] = g_off[i];
        s_val[i] = g_val[i];
        s_oi[i] = off_idx[i];
        s_vi[i] = val_idx[i];
    }
    __syncthreads();
    const uint64_t padded = (n_rows + 31) / 32 * 32;
    for (uint64_t r = blockIdx.x * static_cast<uint64_t>(kDThreads) + threadIdx.x; r < padded;
         r += static_cast<uint64_t>(gridDim.x) * kDThreads) {
        const uint64_t sl = r / 32, lane = r % 32;
        const uint64_t base = ell4 ? 0 : soff[sl], width = ell4 ? 4ull * ell4 : (soff[sl + 1] - base) / 32;
        const uint64_t k0 = r < n_rows ? static_cast<uint64_t>(rp[r]) : 0;
        const uint64_t len = r < n_rows ? static_cast<uint64_t>(rp[r + 1]) - k0 : 0;
        // a row longer than the slice width (an understated max_row_nnz
        // hint) would be cut short: the build is refused instead
        if (len > width) atomicExch(too_long, 1u);
        for (uint64_t k = 0; k < width; ++k) {
            uint16_t code = kPad;
            if (k < len) {
                const int64_t off = static_cast<int64_t>(ci[k0 + k]) - static_cast<int64_t>(r);
                const uint32_t oi = s_oi[table_find(s_off, off_key(off))];
                const uint32_t vi = s_vi[table_find(s_val, static_cast<unsigned long long>(__double_as_longlong(va[k0 + k])))];
                code = static_cast<uint16_t>(vi << 8 | oi);
            }
            // SELL: entry k at base + 32 k + lane; ELL4: groups of 4 entries
            // of a row contiguous (one 8-byte load per group), group g at
            // ((s * ell4 + g) * 32 + lane) * 4
            codes[ell4 ? ((sl * ell4 + k / 4) * 32 + lane) * 4 + (k & 3) : base + k * 32 + lane] = code;
        }
    }
}

// MODE 0: y = A x.  MODE 1: y = b - A x. One warp per slice (persistent
// grid, one wave); kEll: every slice has the same width W (no offset table
// to read before the codes). The first 8 codes of a warp's NEXT slice are
// loaded before the current slice's x gathers, so the code stream of one
// slice overlaps the gathers of the previous one. Per batch of 8 entries:
// dictionary lookups (shared), x gathers, then the in-order multiply-adds
// (sparse.cpp:50-52: separate roundings from +0.0).
// SELL layout (ragged slices): one warp per slice, the first 8 codes of
// the warp's NEXT slice are requested before the current slice's x gathers.
__device__ __forceinline__ void sell_head(uint64_t sl, const uint64_t* __restrict__ soff,
                                          const uint16_t* __restrict__ codes, int lane, uint64_t& base,
                                          uint32_t& width, uint16_t (&cc)[8]) {
    base = __ldg(soff + sl);
    width = static_cast<uint32_t>((__ldg(soff + sl + 1) - base) / 32);
#pragma unroll
    for (int i = 0; i < 8; ++i) cc[i] = i < static_cast<int>(width) ? __ldcs(codes + base + 32 * i + lane) : kPad;
}

// Per batch of 8 entries: dictionary lookups (shared), x gathers, then the
// in-order multiply-adds (sparse.cpp:50-52: separate roundings from +0.0).
__device__ __forceinline__ double batch8(const uint16_t (&c)[8], int32_t r, const int32_t* s_o, const double* s_v,
                                         const double* __restrict__ x, double s) {
    double xv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) xv[i] = c[i] != kPad ? __ldg(x + (r + s_o[c[i] & 0xFF])) : 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
        if (c[i] != kPad) s = __dadd_rn(s, __dmul_rn(s_v[c[i] >> 8], xv[i]));
    return s;
}

__device__ __forceinline__ void unpack8(uint2 a, uint2 b, uint16_t (&c)[8]) {
    c[0] = a.x & 0xFFFF; c[1] = a.x >> 16; c[2] = a.y & 0xFFFF; c[3] = a.y >> 16;
    c[4] = b.x & 0xFFFF; c[5] = b.x >> 16; c[6] = b.y & 0xFFFF; c[7] = b.y >> 16;
}

// MODE 0: y = A x.  MODE 1: y = b - A x. Persistent grid (one wave), one
// warp per 32-row slice. kEll: ELL4 layout (uniform width, 8-byte groups of
// 4 codes, no offset table).
#ifndef DSELL_SPMV_THREADS
#define DSELL_SPMV_THREADS 256
#endif
// the codes stream once per SpMV: evict-first loads (L1-cached __ldg measured neutral)
#define CLD(p) __ldcs(p)
constexpr int kST = DSELL_SPMV_THREADS;
constexpr int kSW = kST / 32;
#ifndef DSELL_MIN_BLOCKS
#define DSELL_MIN_BLOCKS 5  // with the pad-free batches: 160 vs 192 us at 7-pt 256^3, 82 vs 96 convdiff 192^3 (scripts/ab_spmv.sh)
#endif
// (ELL4 instantiations; the ragged SELL path: 4 CTAs, its former 64-register budget)
#define DSELL_BOUNDS __launch_bounds__(kST, kEll && DSELL_MIN_BLOCKS ? DSELL_MIN_BLOCKS : 4)
template <int MODE, bool kEll>
__global__ void DSELL_BOUNDS
dsell_spmv_kernel(uint64_t n_rows, const uint64_t* __restrict__ soff, uint32_t ell_w, const uint16_t* __restrict__ codes,
                  const int32_t* __restrict__ d_off, const double* __restrict__ d_val, const double* __restrict__ x,
                  const double* __restrict__ b, double* __restrict__ y, int with_norm,
                  double* __restrict__ partials, unsigned* __restrict__ ticket, double* __restrict__ norm_out) {
    __shared__ int32_t s_o[256];
    __shared__ double s_v[256];
    __shared__ double red[kSW];
    for (uint32_t i = threadIdx.x; i < 256; i += kST) {
        // index 255 never occurs in a real code: the padding code 0xFFFF
        // decodes to offset 0, value +0.0
        s_o[i] = i == 255 ? 0 : d_off[i];
        s_v[i] = i == 255 ? 0.0 : d_val[i];
    }
    __syncthreads();
    pdl_trigger();
    const int lane = threadIdx.x & 31;
    // warps of the grid interleaved over the slices (measured on B200: a
    // contiguous slice range per CTA, for L1 reuse of the small offsets'
    // x lines, is 3-18% slower)
    const uint64_t nsl = (n_rows + 31) / 32;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * kSW;
    uint64_t sl = (blockIdx.x * static_cast<uint64_t>(kST) + threadIdx.x) / 32;
    double acc = 0.0;
    if constexpr (kEll) {
        const uint32_t g4 = ell_w / 4;  // 8-byte groups per row
        const uint2* c4 = reinterpret_cast<const uint2*>(codes);
        uint2 n0 = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu), n1 = n0;
        // the codes do not depend on the predecessor grid
        if (sl < nsl) {
            n0 = CLD(c4 + sl * g4 * 32 + lane);
            if (g4 > 1) n1 = CLD(c4 + (sl * g4 + 1) * 32 + lane);
        }
        pdl_wait();
        for (; sl < nsl; sl += nw) {
            const int32_t r = static_cast<int32_t>(sl * 32 + lane);
            uint2 a0 = n0, a1 = n1;
            const uint64_t nx = sl + nw;
            if (nx < nsl) {
                n0 = CLD(c4 + nx * g4 * 32 + lane);
                if (g4 > 1) n1 = CLD(c4 + (nx * g4 + 1) * 32 + lane);
            }
            double s = 0.0;
            // Padding codes decode to (offset 0, value +0.0): the gather reads
            // x[r] (clamped into range for the rows past n) and adds 0 * x[r]
            // = +-0, which leaves s unchanged (s starts at +0.0 and is never
            // -0.0), so the batches need no per-entry predicates. A NaN sum
            // (which a non-finite x[r] under a padding code could cause) is
            // recomputed exactly below.
            const int32_t rc = static_cast<uint64_t>(r) < n_rows ? r : static_cast<int32_t>(n_rows - 1);
            for (uint32_t g = 0; g < g4; g += 2) {
                if (g) {
                    a0 = CLD(c4 + (sl * g4 + g) * 32 + lane);
                    a1 = g + 1 < g4 ? CLD(c4 + (sl * g4 + g + 1) * 32 + lane) : make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
                } else if (g4 == 1) {
                    a1 = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
                }
                uint16_t c[8];
                unpack8(a0, a1, c);
                double xv[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) xv[i] = __ldg(x + (rc + s_o[c[i] & 0xFF]));
#pragma unroll
                for (int i = 0; i < 8; ++i) s = __dadd_rn(s, __dmul_rn(s_v[c[i] >> 8], xv[i]));
            }
            if (isnan(s) && static_cast<uint64_t>(r) < n_rows) {
                s = 0.0;
                for (uint32_t g = 0; g < g4; g += 2) {
                    const uint2 e0 = CLD(c4 + (sl * g4 + g) * 32 + lane);
                    const uint2 e1 = g + 1 < g4 ? CLD(c4 + (sl * g4 + g + 1) * 32 + lane)
                                                : make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
                    uint16_t c[8];
                    unpack8(e0, e1, c);
                    s = batch8(c, r, s_o, s_v, x, s);
                }
            }
            if (static_cast<uint64_t>(r) < n_rows) {
                if (MODE == 1) s = __dsub_rn(__ldg(b + r), s);
                y[r] = s;
                if (with_norm) acc = __dadd_rn(acc, __dmul_rn(s, s));
            }
        }
    } else {
        uint16_t cc[8];
        uint64_t base = 0;
        uint32_t width = 0;
        if (sl < nsl) sell_head(sl, soff, codes, lane, base, width, cc);
        pdl_wait();
        for (; sl < nsl; sl += nw) {
            const int64_t r = static_cast<int64_t>(sl * 32 + lane);
            uint16_t cur[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) cur[i] = cc[i];
            const uint64_t cbase = base;
            const uint32_t cw = width;
            if (sl + nw < nsl) sell_head(sl + nw, soff, codes, lane, base, width, cc);
            double s = 0.0;
            for (uint32_t k = 0; k < cw; k += 8) {
                if (k) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) cur[i] = k + i < cw ? __ldcs(codes + cbase + 32 * (k + i) + lane) : kPad;
                }
                double xv[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) xv[i] = cur[i] != kPad ? __ldg(x + (r + s_o[cur[i] & 0xFF])) : 0.0;
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    if (cur[i] != kPad) s = __dadd_rn(s, __dmul_rn(s_v[cur[i] >> 8], xv[i]));
            }
            if (static_cast<uint64_t>(r) < n_rows) {
                if (MODE == 1) s = __dsub_rn(__ldg(b + r), s);
                y[r] = s;
                if (with_norm) acc = __dadd_rn(acc, __dmul_rn(s, s));
            }
        }
    }
    if (!with_norm) return;
    acc = warp_sum(acc);
    if (lane == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    block_finalize(red, kSW, 1, partials, ticket, norm_out);
}

// ---------------------------------------------------- pair-coded ELL8
// Structured-grid matrices hold few distinct (value, column offset) PAIRS
// (a constant-coefficient stencil: one per offset). When there are at most
// 255, each entry becomes ONE byte indexing a pair table {value, offset} in
// shared memory: half the code bytes of the 2-byte (value, offset) codes,
// and per entry one 16-byte shared load instead of two lookups plus field
// extraction (the SpMV is instruction-bound: ~190 instructions per 32-row
// slice with 2-byte codes on B200). Rows are padded to a multiple of 8
// entries (one 8-byte code load per 8 entries); 0xFF = padding = (+0.0,
// offset 0), unpredicated as in dsell_spmv_kernel.

// Which 2-byte codes occur: a per-CTA shared bitmap, merged with atomicOr.
__global__ void __launch_bounds__(256) pair_mark_kernel(const uint16_t* __restrict__ codes, uint64_t count,
                                                        unsigned* __restrict__ bitmap) {
    __shared__ unsigned sb[2048];
    for (uint32_t i = threadIdx.x; i < 2048; i += 256) sb[i] = 0u;
    __syncthreads();
    const uint4* c8 = reinterpret_cast<const uint4*>(codes);
    for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < count / 8; i += gridDim.x * 256ull) {
        const uint4 q = __ldcs(c8 + i);
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t c = (w[k / 2] >> (16 * (k & 1))) & 0xFFFFu;
            if (c != kPad) {
                const unsigned bit = 1u << (c & 31);
                if (!(sb[c >> 5] & bit)) atomicOr(sb + (c >> 5), bit);
            }
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < 2048; i += 256)
        if (sb[i]) atomicOr(bitmap + i, sb[i]);
}

// ELL4 2-byte codes -> ELL8 pair bytes (entry k of row 32s+lane at byte
// ((s * g8 + k / 8) * 32 + lane) * 8 + k % 8).
__global__ void __launch_bounds__(256) pair_convert_kernel(const uint16_t* __restrict__ codes, uint64_t nslices,
                                                           uint32_t g4, uint32_t g8, const uint8_t* __restrict__ map8,
                                                           uint8_t* __restrict__ out) {
    const uint64_t total = nslices * 32 * g8;  // 8-byte output groups
    for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < total; i += gridDim.x * 256ull) {
        const uint64_t lane = i % 32, sg = i / 32, sl = sg / g8, g = sg % g8;
        uint32_t lo = 0, hi = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t e = static_cast<uint32_t>(g) * 8 + k;  // entry index in the row
            uint32_t b = 0xFFu;
            if (e < 4 * g4) {
                const uint16_t c = codes[((sl * g4 + e / 4) * 32 + lane) * 4 + (e & 3)];
                if (c != kPad) b = map8[c];
            }
            if (k < 4) lo |= b << (8 * k);
            else hi |= b << (8 * (k - 4));
        }
        reinterpret_cast<uint2*>(out)[i] = make_uint2(lo, hi);
    }
}

// 4 CTAs/SM: 7-pt 128^3 SpMV phase 0.975 vs 0.993 ms per solve at 5 (48
// registers), 1.007 at 6, 1.072 at 8; two slices per warp iteration (both
// slices' gathers in flight) was slower (24.6 vs 22.5 us).
#ifndef PELL_MIN_BLOCKS
#define PELL_MIN_BLOCKS 4
#endif
// Row r's result: a NaN sum (a non-finite x[rc] under a padding entry) is
// recomputed over the real entries only; then y[r] (or b[r] - ...) and the
// norm partial.
template <int MODE>
__device__ __forceinline__ void pell_finish(double s, int32_t r, uint64_t n_rows, uint32_t g8, const uint2* cp,
                                            const double2* tab, const double* __restrict__ x,
                                            const double* __restrict__ b, double* __restrict__ y, int with_norm,
                                            double& acc) {
    if (static_cast<uint64_t>(r) >= n_rows) return;
    if (isnan(s)) {
        s = 0.0;
        for (uint32_t g = 0; g < g8; ++g) {
            const uint2 q = __ldcs(cp + 32 * g);
            for (int k = 0; k < 8; ++k) {
                const uint32_t idx = ((k < 4 ? q.x : q.y) >> (8 * (k & 3))) & 0xFFu;
                if (idx != 0xFFu)
                    s = __dadd_rn(s, __dmul_rn(tab[idx].x, __ldg(x + r + __double2loint(tab[idx].y) / 8)));
            }
        }
    }
    if (MODE == 1) s = __dsub_rn(__ldg(b + r), s);
    y[r] = s;
    if (with_norm) acc = __dadd_rn(acc, __dmul_rn(s, s));
}
// MODE 0: y = A x.  MODE 1: y = b - A x. One warp per 32-row slice, lane =
// row; products and sums in row order from +0.0 (sparse.cpp:50-52), padding
// entries add +-0 (see dsell_spmv_kernel) and a NaN sum is recomputed
// exactly; bit-identical to spmv().
// G1: every row fits one 8-byte code word (g8 == 1, <= 8 entries per row:
// 7-point stencils): the row's 8 table offsets are read first, all 8
// gathers issued back to back (32-bit byte offsets from x), then the values
// and the row-order sum -- fewer live registers than holding 8 (value,
// offset) pairs across the gathers, so the loads are not serialised.
#ifndef PELL_G1
#define PELL_G1 1
#endif
template <int MODE, int G1>
__global__ void __launch_bounds__(256, PELL_MIN_BLOCKS)
pell_spmv_kernel(uint64_t n_rows, uint32_t g8, const uint8_t* __restrict__ codes, const int32_t* __restrict__ p_off,
                 const double* __restrict__ p_val, const double* __restrict__ x, const double* __restrict__ b,
                 double* __restrict__ y, int with_norm, double* __restrict__ partials, unsigned* __restrict__ ticket,
                 double* __restrict__ norm_out, uint64_t s_begin, uint64_t s_end, int accumulate, uint32_t n_pair) {
    // pair table: .x = value, .y = the column offset in BYTES (off * 8) in
    // the low word -- one 16-byte shared load per entry, and the gather
    // address is the slice's row pointer plus a sign-extended 32-bit offset
    __shared__ double2 tab[256];
    __shared__ double red[8];
    // only the n_pair used entries and the padding entry 255 are read
    if (threadIdx.x < n_pair)
        tab[threadIdx.x] = make_double2(p_val[threadIdx.x], __hiloint2double(0, 8 * p_off[threadIdx.x]));
    else if (threadIdx.x == 255)
        tab[255] = make_double2(0.0, __hiloint2double(0, 0));
    pdl_trigger();
    const int lane = threadIdx.x & 31;
    const uint64_t nsl = s_end;  // slices [s_begin, s_end)
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * 8;
    uint64_t sl = s_begin + (blockIdx.x * 256ull + threadIdx.x) / 32;
    // running pointers: the warp's slice advances by nw slices per iteration
    const uint64_t cstep = nw * g8 * 32;  // in 8-byte groups
    const uint2* cp = reinterpret_cast<const uint2*>(codes) + sl * g8 * 32 + lane;
    int32_t r = static_cast<int32_t>(sl * 32 + lane);
    const int32_t rstep = static_cast<int32_t>(nw * 32);
    const int32_t rlast = static_cast<int32_t>(n_rows - 1);
    double acc = 0.0;
    uint2 nxt = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
    if (sl < nsl) nxt = __ldcs(cp);  // codes do not depend on the predecessor
    __syncthreads();
    pdl_wait();
    for (; sl < nsl; sl += nw, cp += cstep, r += rstep) {
        const int32_t rc = min(r, rlast);
        const char* xr = reinterpret_cast<const char*>(x + rc);
        uint2 cur = nxt;
        if (sl + nw < nsl) nxt = __ldcs(cp + cstep);
        double s = 0.0;
        if constexpr (G1) {
            const uint32_t* tw = reinterpret_cast<const uint32_t*>(tab);
            const uint32_t rb = static_cast<uint32_t>(rc) * 8u;
            uint32_t idx[8];
            double xv[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) idx[k] = ((k < 4 ? cur.x : cur.y) >> (8 * (k & 3))) & 0xFFu;
#pragma unroll
            for (int k = 0; k < 8; ++k)
                xv[k] = __ldg(reinterpret_cast<const double*>(reinterpret_cast<const char*>(x) +
                                                              static_cast<uint64_t>(rb + tw[4 * idx[k] + 2])));
#pragma unroll
            for (int k = 0; k < 8; ++k) s = __dadd_rn(s, __dmul_rn(tab[idx[k]].x, xv[k]));
            pell_finish<MODE>(s, r, n_rows, g8, cp, tab, x, b, y, with_norm, acc);
            continue;
        }
        for (uint32_t g = 0; g < g8; ++g) {
            if (g) cur = __ldcs(cp + 32 * g);
            double v[8], xv[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t idx = ((k < 4 ? cur.x : cur.y) >> (8 * (k & 3))) & 0xFFu;
                const double2 t = tab[idx];
                v[k] = t.x;
                xv[k] = __ldg(reinterpret_cast<const double*>(xr + __double2loint(t.y)));
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) s = __dadd_rn(s, __dmul_rn(v[k], xv[k]));
        }
        pell_finish<MODE>(s, r, n_rows, g8, cp, tab, x, b, y, with_norm, acc);
    }
    if (!with_norm) return;
    acc = warp_sum(acc);
    if (lane == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (with_norm == 2) {
        // per-CTA partials only (warps in order): the consumer sums them
        // after the kernel boundary -- no fence, ticket or last-block tail
        if (threadIdx.x == 0) {
            double t = red[0];
            for (int w = 1; w < 8; ++w) t = __dadd_rn(t, red[w]);
            partials[blockIdx.x] = t;
        }
        return;
    }
    block_finalize(red, 8, 1, partials, ticket, norm_out, accumulate != 0);
}

// ---------------------------------------------------------------------------
// Row-pattern coded SpMV. A constant-coefficient stencil has very few distinct
// ROWS of pair codes (7-point on a box: 27 -- interior, faces, edges,
// corners). When the matrix holds <= 255 distinct rows of the pair-coded
// copy, every row becomes ONE byte (its pattern id) and the table
// {8G element offsets (int32), 8G values (fp64)} of each pattern sits in
// shared memory: per row 2G + 4G 16-byte shared loads instead of one shared
// load and a byte extraction per entry, and per entry one 32-bit add plus one
// IMAD.WIDE for the gather address. Padding entries are (offset 0, +0.0):
// same bit-identity argument as the pair-coded kernel, a NaN sum recomputed
// over the pattern's real entries. Products and sums in row order:
// bit-identical to spmv() (sparse.cpp:50-52).
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
// hash of one row's G code words (never 0: 0 marks an empty slot)
__device__ __forceinline__ unsigned long long row_key(const uint2* __restrict__ cp, uint32_t g8) {
    unsigned long long h = 0x632BE59BD9B4E019ull;
    for (uint32_t g = 0; g < g8; ++g) {
        const uint2 q = cp[32 * g];
        h = mix64(h ^ (static_cast<unsigned long long>(q.y) << 32 | q.x));
    }
    return h ? h : 1ull;
}
constexpr uint32_t kPatSlots = 1024;  // global table; per-CTA table below
constexpr uint32_t kPatLocal = 512;
constexpr uint32_t kPatTabMax = 40u * 1024u;  // dynamic shared memory of the pattern tables
// offset of a padding entry: a gather of x[r] times +0.0 (a NaN sum is
// recomputed over the pattern's leading real entries). Predicating padding
// entries off instead measured no faster (L1 requests saved, issue lost).
constexpr int32_t kPatPad = 0;

// Pass 1: the distinct row patterns, deduplicated per CTA in shared memory,
// then merged into the global table; the CTA that claims a global slot writes
// the row's code words next to it. *bad: a table overflowed.
__global__ void __launch_bounds__(256) pat_scan_kernel(const uint2* __restrict__ codes8, uint64_t rows, uint32_t g8,
                                                       unsigned long long* __restrict__ gkeys,
                                                       uint2* __restrict__ gwords, unsigned* __restrict__ bad) {
    __shared__ unsigned long long sk[kPatLocal];
    __shared__ uint32_t srow[kPatLocal];
    for (uint32_t i = threadIdx.x; i < kPatLocal; i += 256) sk[i] = 0ull;
    __syncthreads();
    bool over = false;
    for (uint64_t r = blockIdx.x * 256ull + threadIdx.x; r < rows; r += gridDim.x * 256ull) {
        const uint2* cp = codes8 + (r / 32) * g8 * 32 + (r % 32);
        const unsigned long long h = row_key(cp, g8);
        uint32_t s = static_cast<uint32_t>(h) & (kPatLocal - 1), p = 0;
        for (; p < kPatLocal; ++p, s = (s + 1) & (kPatLocal - 1)) {
            unsigned long long k = *reinterpret_cast<volatile unsigned long long*>(sk + s);
            if (k == h) break;
            if (k == 0ull) {
                k = atomicCAS(sk + s, 0ull, h);
                if (k == 0ull) { srow[s] = static_cast<uint32_t>(r); break; }
                if (k == h) break;
            }
        }
        over |= p == kPatLocal;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < kPatLocal; i += 256) {
        const unsigned long long h = sk[i];
        if (!h) continue;
        uint32_t s = static_cast<uint32_t>(h >> 32) & (kPatSlots - 1), p = 0;
        for (; p < kPatSlots; ++p, s = (s + 1) & (kPatSlots - 1)) {
            unsigned long long k = *reinterpret_cast<volatile unsigned long long*>(gkeys + s);
            if (k == h) break;
            if (k == 0ull) {
                k = atomicCAS(gkeys + s, 0ull, h);
                if (k == 0ull) {
                    const uint64_t r = srow[i];
                    const uint2* cp = codes8 + (r / 32) * g8 * 32 + (r % 32);
                    for (uint32_t g = 0; g < g8; ++g) gwords[s * 4 + g] = cp[32 * g];
                    break;
                }
                if (k == h) break;
            }
        }
        over |= p == kPatSlots;
    }
    if (over) atomicOr(bad, 1u);
}

// Pass 2: every row's pattern id, verified word by word against the pattern
// (a hash collision sets *bad and the matrix keeps the pair-coded kernel).
__global__ void __launch_bounds__(256) pat_map_kernel(const uint2* __restrict__ codes8, uint64_t rows, uint32_t g8,
                                                      const unsigned long long* __restrict__ gkeys,
                                                      const uint8_t* __restrict__ slot_id,
                                                      const uint2* __restrict__ pwords, uint8_t* __restrict__ pid,
                                                      unsigned* __restrict__ bad) {
    __shared__ unsigned long long sk[kPatSlots];
    __shared__ uint8_t sid[kPatSlots];
    for (uint32_t i = threadIdx.x; i < kPatSlots; i += 256) {
        sk[i] = gkeys[i];
        sid[i] = slot_id[i];
    }
    __syncthreads();
    bool wrong = false;
    for (uint64_t r = blockIdx.x * 256ull + threadIdx.x; r < rows; r += gridDim.x * 256ull) {
        const uint2* cp = codes8 + (r / 32) * g8 * 32 + (r % 32);
        const unsigned long long h = row_key(cp, g8);
        uint32_t s = static_cast<uint32_t>(h >> 32) & (kPatSlots - 1), p = 0;
        while (p < kPatSlots && sk[s] != h && sk[s] != 0ull) { s = (s + 1) & (kPatSlots - 1); ++p; }
        if (p == kPatSlots || sk[s] != h) { wrong = true; continue; }
        const uint32_t id = sid[s];
        for (uint32_t g = 0; g < g8; ++g) {
            const uint2 a = cp[32 * g], b = pwords[id * g8 + g];
            wrong |= a.x != b.x || a.y != b.y;
        }
        pid[r] = static_cast<uint8_t>(id);
    }
    if (wrong) atomicOr(bad, 1u);
}

template <int MODE, int G>
__global__ void __launch_bounds__(256, PELL_MIN_BLOCKS)
ppat_spmv_kernel(uint64_t n_rows, const uint8_t* __restrict__ pid, const uint4* __restrict__ ptab, uint32_t ptab_u4,
                 const uint8_t* __restrict__ pcnt, const double* __restrict__ x, const double* __restrict__ b, double* __restrict__ y, int with_norm,
                 double* __restrict__ partials, unsigned* __restrict__ ticket, double* __restrict__ norm_out,
                 uint64_t s_begin, uint64_t s_end, int accumulate) {
    // pattern p: int32 off[8G] at p * 96G (kPatPad = padding), then fp64 val[8G]
    extern __shared__ uint4 stab[];
    __shared__ double red[8];
    for (uint32_t i = threadIdx.x; i < ptab_u4; i += 256) stab[i] = ptab[i];
    pdl_trigger();
    const int lane = threadIdx.x & 31;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * 8;
    const uint64_t sl = s_begin + (blockIdx.x * 256ull + threadIdx.x) / 32;
    const uint32_t iters = sl < s_end ? static_cast<uint32_t>((s_end - sl + nw - 1) / nw) : 0u;
    int32_t r = static_cast<int32_t>(sl * 32 + lane);
    const int32_t rstep = static_cast<int32_t>(nw * 32);
    const int32_t nr = static_cast<int32_t>(n_rows);
    double acc = 0.0;
    uint32_t nxt = 0;
    if (iters) nxt = __ldcs(pid + r);  // ids do not depend on the predecessor
    __syncthreads();
    pdl_wait();
    const char* tb = reinterpret_cast<const char*>(stab);
    for (uint32_t it = 0; it < iters; ++it, r += rstep) {
        const uint32_t p = nxt;
        if (it + 1 < iters) nxt = __ldcs(pid + r + rstep);
        const char* pb = tb + p * (96u * G);
        // rows past n_rows (the last slice's fill) are all padding: they
        // gather x[n_rows - 1]
        const double* xb = x + min(r, nr - 1);
        // opaque row pointer: each gather address is then ONE IMAD.WIDE of
        // the entry's offset (ptxas would otherwise re-associate r + off in
        // 64 bits: four instructions per gather)
        asm("" : "+l"(xb));
        double s = 0.0;
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int4 o0 = *reinterpret_cast<const int4*>(pb + 32 * g);
            const int4 o1 = *reinterpret_cast<const int4*>(pb + 32 * g + 16);
            const int32_t o[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
            double xv[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) xv[k] = __ldg(xb + o[k]);
#pragma unroll
            for (int k = 0; k < 8; k += 2) {
                const double2 v = *reinterpret_cast<const double2*>(pb + 32 * G + 64 * g + 8 * k);
                s = __dadd_rn(s, __dmul_rn(v.x, xv[k]));
                s = __dadd_rn(s, __dmul_rn(v.y, xv[k + 1]));
            }
        }
        if (isnan(s) && r < nr) {
            // a padding entry (offset 0, +0.0; real entries come first)
            // multiplied a non-finite x[r]: recompute over the real entries
            const uint32_t cnt = __ldg(pcnt + p);
            s = 0.0;
#pragma unroll 1
            for (uint32_t e = 0; e < cnt; ++e) {
                const int32_t oe = reinterpret_cast<const int32_t*>(pb + 32 * (e / 8))[e % 8];
                const double ve = reinterpret_cast<const double*>(pb + 32 * G + 64 * (e / 8))[e % 8];
                s = __dadd_rn(s, __dmul_rn(ve, __ldg(xb + oe)));
            }
        }
        if (r >= nr) continue;
        if (MODE == 1) s = __dsub_rn(__ldg(b + r), s);
        y[r] = s;
        if (with_norm) acc = __dadd_rn(acc, __dmul_rn(s, s));
    }
    if (!with_norm) return;
    acc = warp_sum(acc);
    if (lane == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (with_norm == 2) {
        if (threadIdx.x == 0) {
            double t = red[0];
            for (int w = 1; w < 8; ++w) t = __dadd_rn(t, red[w]);
            partials[blockIdx.x] = t;
        }
        return;
    }
    block_finalize(red, 8, 1, partials, ticket, norm_out, accumulate != 0);
}

// Uniform-slot patterns (a constant-coefficient stencil): the real column
// offsets of every row pattern, in row order, embed into ONE sorted list of
// S <= 32 slots, and every slot carries one value whatever the pattern. A
// row is then its pattern's slot mask: per slot present, one gather of
// x[r + off[u]] and one multiply-add by val[u] -- offsets and values are
// kernel parameters (constant bank operands, no shared-memory table loads).
// An absent slot gathers nothing and multiplies +0.0: with every slot value
// finite (checked at build) that adds +-0, which leaves the row sum unchanged
// (it starts at +0.0 and is never -0.0), so the row sums its real entries in
// row order: bit-identical to spmv() (sparse.cpp:50-52) for any x.
struct USlots {
    int32_t off[32];
    double val[32];
};
// 2 slices per warp iteration, 5 CTAs/SM (scripts/ab_uslot.sh, one box):
// 7-pt 128^3 solve-like 16.4 -> 14.3 us, 27-pt 256^3 182 -> 150 us, bench
// SpMV phase 0.72 -> 0.64 ms; 3 slices or 3 CTAs/SM no better.
#ifndef USLOT_U
#define USLOT_U 2
#endif
#ifndef USLOT_MIN_BLOCKS
#define USLOT_MIN_BLOCKS 5
#endif

template <int MODE, int S>
__global__ void __launch_bounds__(256, USLOT_MIN_BLOCKS)
uslot_spmv_kernel(uint64_t n_rows, uint64_t n_cols, const uint8_t* __restrict__ pid, const uint32_t* __restrict__ pmask,
                  uint32_t n_pat, const __grid_constant__ USlots us, const double* __restrict__ x,
                  const double* __restrict__ b, double* __restrict__ y, int with_norm,
                  double* __restrict__ partials, unsigned* __restrict__ ticket, double* __restrict__ norm_out,
                  uint64_t s_begin, uint64_t s_end, int accumulate) {
    __shared__ uint32_t smask[256];
    __shared__ double red[8];
    if (threadIdx.x < n_pat) smask[threadIdx.x] = pmask[threadIdx.x];
    pdl_trigger();
    const int lane = threadIdx.x & 31;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * 8;
    const uint64_t sl = s_begin + (blockIdx.x * 256ull + threadIdx.x) / 32;
    const uint32_t iters = sl < s_end ? static_cast<uint32_t>((s_end - sl + nw - 1) / nw) : 0u;
    int32_t r = static_cast<int32_t>(sl * 32 + lane);
    const int32_t rstep = static_cast<int32_t>(nw * 32);
    const int32_t nr = static_cast<int32_t>(n_rows);
    double acc = 0.0;
    // USLOT_U slices per iteration (their gathers in flight together); ids
    // prefetched one iteration ahead
    constexpr int U = USLOT_U;
    uint32_t nxt[U];
    const uint8_t* pp = pid + r;  // running pointer to the next iteration's ids
#pragma unroll
    for (int u = 0; u < U; ++u) nxt[u] = static_cast<uint32_t>(u) < iters ? __ldcs(pp + u * rstep) : 0u;
    __syncthreads();
    pdl_wait();
    for (uint32_t it = 0; it < iters; it += U, r += U * rstep) {
        uint32_t m[U];
        const double* xb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            m[u] = it + u < iters ? smask[nxt[u]] : 0u;
            xb[u] = x + min(r + u * rstep, nr - 1);
            asm("" : "+l"(xb[u]));  // one IMAD.WIDE per gather (see ppat_spmv_kernel)
        }
        pp += U * rstep;
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (it + U + u < iters) nxt[u] = __ldcs(pp + u * rstep);
        double sum[U];
#pragma unroll
        for (int u = 0; u < U; ++u) sum[u] = 0.0;
#pragma unroll
        for (int g = 0; g < S; g += 8) {
            constexpr int kMax = 8;
            double xv[U][kMax];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int k = 0; k < kMax; ++k) {
                    xv[u][k] = 0.0;
                    if (g + k < S && (m[u] >> (g + k) & 1u)) xv[u][k] = __ldg(xb[u] + us.off[g + k]);
                }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int k = 0; k < kMax; ++k)
                    if (g + k < S) sum[u] = __dadd_rn(sum[u], __dmul_rn(us.val[g + k], xv[u][k]));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t ru = r + u * rstep;
            if (it + u >= iters || ru >= nr) continue;
            double sv = sum[u];
            if (MODE == 1) sv = __dsub_rn(__ldg(b + ru), sv);
            y[ru] = sv;
            if (with_norm) acc = __dadd_rn(acc, __dmul_rn(sv, sv));
        }
    }
    if (!with_norm) return;
    acc = warp_sum(acc);
    if (lane == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (with_norm == 2) {
        if (threadIdx.x == 0) {
            double t = red[0];
            for (int w = 1; w < 8; ++w) t = __dadd_rn(t, red[w]);
            partials[blockIdx.x] = t;
        }
        return;
    }
    block_finalize(red, 8, 1, partials, ticket, norm_out, accumulate != 0);
}

int dict_grid(uint64_t rows) {
    const uint64_t want = (rows + kDThreads - 1) / kDThreads;
    const uint64_t cap = static_cast<uint64_t>(sm_count()) * 8;
    return static_cast<int>(std::max<uint64_t>(1, std::min(want, cap)));
}

// Pair-coded ELL8 SpMV switch (A/B: CBGX_PELL=0 keeps the 2-byte codes).
bool pell_enabled() {
    static const bool v = [] {
        const char* e = getenv("CBGX_PELL");
        return !e || atoi(e) != 0;
    }();
    return v;
}

template <typename T>
void ensure(T*& p, uint64_t& cap, uint64_t need) {
    if (p && cap >= need) return;
    if (p) CBGX_CUDA(cudaFree(p));
    p = nullptr;
    CBGX_CUDA(cudaMalloc(reinterpret_cast<void**>(&p), std::max<uint64_t>(need, 1) * sizeof(T)));
    cap = need;
}

// Row-pattern switch (A/B: CBGX_PPAT=0 keeps the pair-coded kernel).
bool ppat_enabled() {
    static const bool v = [] {
        const char* e = getenv("CBGX_PPAT");
        return !e || atoi(e) != 0;
    }();
    return v;
}

// The row-pattern copy from the pair codes (see ppat_spmv_kernel): a scan
// collects the distinct rows (one 40 KB host round trip), the host builds the
// pattern tables, a map pass writes one id byte per row and verifies it (one
// more 4-byte round trip). D.n_pat stays 0 on more than 255 patterns.
void build_patterns(DictSell& D, const std::vector<int32_t>& po, const std::vector<double>& pv, cudaStream_t st) {
    D.n_pat = 0;
    D.n_slots = 0;
    const uint32_t g8 = D.ell8_w / 8;
    if (!ppat_enabled() || D.max_level < 2 || g8 < 1 || g8 > 4) return;
    uint64_t cap = 0;
    if (!D.pkeys) {
        ensure(D.pkeys, cap, kPatSlots);
        ensure(D.pwords, cap, kPatSlots * 4);
        ensure(D.pslot, cap, kPatSlots);
    }
    const uint64_t rows = D.nslices * 32;
    CBGX_CUDA(cudaMemsetAsync(D.pkeys, 0, kPatSlots * sizeof(unsigned long long), st));
    CBGX_CUDA(cudaMemsetAsync(D.flags, 0, sizeof(unsigned), st));
    const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((rows + 255) / 256, sm_count() * 2ull)));
    const uint2* c8 = reinterpret_cast<const uint2*>(D.codes8);
    CBGX_K(pat_scan_kernel<<<grid, 256, 0, st>>>(c8, rows, g8, D.pkeys, D.pwords, D.flags));
    CBGX_CUDA(cudaGetLastError());
    std::vector<unsigned long long> keys(kPatSlots);
    std::vector<uint2> words(kPatSlots * 4);
    unsigned bad = 0;
    CBGX_CUDA(cudaMemcpyAsync(keys.data(), D.pkeys, kPatSlots * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CBGX_CUDA(cudaMemcpyAsync(words.data(), D.pwords, kPatSlots * 4 * sizeof(uint2), cudaMemcpyDeviceToHost, st));
    CBGX_CUDA(cudaMemcpyAsync(&bad, D.flags, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    CBGX_CUDA(cudaStreamSynchronize(st));
    if (bad) return;
    std::vector<uint8_t> slot(kPatSlots, 0);
    std::vector<uint2> pw;
    uint32_t np = 0;
    for (uint32_t i = 0; i < kPatSlots; ++i) {
        if (!keys[i]) continue;
        if (np == 255) return;
        slot[i] = static_cast<uint8_t>(np++);
        for (uint32_t g = 0; g < g8; ++g) pw.push_back(words[i * 4 + g]);
    }
    const uint32_t stride = 96 * g8;  // bytes per pattern
    if (np * stride > kPatTabMax) return;
    if (np == 0) return;
    std::vector<uint8_t> tab(static_cast<size_t>(np) * stride, 0);
    std::vector<uint8_t> cnt(np, 0);
    for (uint32_t p = 0; p < np; ++p) {
        int32_t* off = reinterpret_cast<int32_t*>(tab.data() + p * stride);
        double* val = reinterpret_cast<double*>(tab.data() + p * stride + 32 * g8);
        for (uint32_t e = 0; e < 8 * g8; ++e) {
            const uint2 w = pw[p * g8 + e / 8];
            const uint32_t k = e % 8;
            const uint32_t c = ((k < 4 ? w.x : w.y) >> (8 * (k & 3))) & 0xFFu;
            off[e] = c == 0xFFu ? kPatPad : po[c];
            val[e] = c == 0xFFu ? 0.0 : pv[c];
            // real entries first, then padding (dict_fill_kernel, pair_convert_kernel)
            if (c != 0xFFu) cnt[p] = static_cast<uint8_t>(e + 1);
        }
    }
    if (!D.ptab) CBGX_CUDA(cudaMalloc(reinterpret_cast<void**>(&D.ptab), kPatTabMax));
    if (!D.pcnt) CBGX_CUDA(cudaMalloc(reinterpret_cast<void**>(&D.pcnt), 256));
    CBGX_CUDA(cudaMemcpyAsync(D.pcnt, cnt.data(), np, cudaMemcpyHostToDevice, st));
    ensure(D.pid, D.pid_cap, rows);
    uint2* d_pw = D.pwords;  // dense pattern words reuse the scratch (after the copy back)
    CBGX_CUDA(cudaMemcpyAsync(D.ptab, tab.data(), tab.size(), cudaMemcpyHostToDevice, st));
    CBGX_CUDA(cudaMemcpyAsync(D.pslot, slot.data(), kPatSlots, cudaMemcpyHostToDevice, st));
    CBGX_CUDA(cudaMemcpyAsync(d_pw, pw.data(), pw.size() * sizeof(uint2), cudaMemcpyHostToDevice, st));
    CBGX_K(pat_map_kernel<<<grid, 256, 0, st>>>(c8, rows, g8, D.pkeys, D.pslot, d_pw, D.pid, D.flags));
    CBGX_CUDA(cudaGetLastError());
    CBGX_CUDA(cudaMemcpyAsync(&bad, D.flags, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    // the host vectors above are read by the async copies: finish them here
    CBGX_CUDA(cudaStreamSynchronize(st));
    if (bad) return;
    D.ptab_u4 = static_cast<uint32_t>(tab.size() / 16);
    D.n_pat = np;
    // uniform slots: every pattern's real offsets increasing, their union
    // <= 32 slots, one value per slot
    D.n_slots = 0;
    if (D.max_level < 3) return;
    std::vector<int32_t> u;
    for (uint32_t p = 0; p < np; ++p) {
        const int32_t* off = reinterpret_cast<const int32_t*>(tab.data() + p * stride);
        for (uint32_t e = 0; e < cnt[p]; ++e) {
            if (e && off[e] <= off[e - 1]) return;
            u.push_back(off[e]);
        }
    }
    std::sort(u.begin(), u.end());
    u.erase(std::unique(u.begin(), u.end()), u.end());
    if (u.empty() || u.size() > 32) return;
    USlots us{};
    std::vector<bool> seen(u.size(), false);
    std::vector<uint32_t> mask(np, 0u);
    for (uint32_t p = 0; p < np; ++p) {
        const int32_t* off = reinterpret_cast<const int32_t*>(tab.data() + p * stride);
        const double* val = reinterpret_cast<const double*>(tab.data() + p * stride + 32 * g8);
        for (uint32_t e = 0; e < cnt[p]; ++e) {
            const uint32_t k = static_cast<uint32_t>(std::lower_bound(u.begin(), u.end(), off[e]) - u.begin());
            if (seen[k] && std::memcmp(&us.val[k], &val[e], 8) != 0) return;
            if (!std::isfinite(val[e])) return;  // absent slots multiply +0.0
            us.val[k] = val[e];
            seen[k] = true;
            mask[p] |= 1u << k;
        }
    }
    for (size_t k = 0; k < u.size(); ++k) us.off[k] = u[k];
    if (!D.pmask) CBGX_CUDA(cudaMalloc(reinterpret_cast<void**>(&D.pmask), 256 * sizeof(uint32_t)));
    CBGX_CUDA(cudaMemcpyAsync(D.pmask, mask.data(), np * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    CBGX_CUDA(cudaStreamSynchronize(st));
    static_assert(sizeof(USlots) <= sizeof(D.uslots), "USlots storage");
    std::memcpy(D.uslots, &us, sizeof(USlots));
    D.n_slots = static_cast<uint32_t>(u.size());
}

// The pair-coded ELL8 copy from the ELL4 2-byte codes (see pell_spmv_kernel):
// one pass marks the 2-byte codes present, the host numbers them (one round
// trip of 8 KB), one pass rewrites the codes as bytes. D.ell8_w stays 0 (the
// 2-byte kernel is used) for SELL layouts or more than 255 pairs.
void build_pairs(DictSell& D, const std::vector<int32_t>& d_off, const std::vector<double>& d_val, cudaStream_t st) {
    D.ell8_w = 0;
    D.n_pat = 0;
    D.n_slots = 0;
    if (!D.ell_w || !pell_enabled() || D.max_level < 1) return;
    uint64_t cap = 0;
    if (!D.bitmap) {
        ensure(D.bitmap, cap, 2048);
        ensure(D.map8, cap, 65536);
        ensure(D.pair_val, cap, 256);
        ensure(D.pair_off, cap, 256);
    }
    CBGX_CUDA(cudaMemsetAsync(D.bitmap, 0, 2048 * sizeof(unsigned), st));
    const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((D.entries / 8 + 255) / 256, sm_count() * 4ull)));
    CBGX_K(pair_mark_kernel<<<grid, 256, 0, st>>>(D.codes, D.entries, D.bitmap));
    CBGX_CUDA(cudaGetLastError());
    std::vector<unsigned> bm(2048);
    CBGX_CUDA(cudaMemcpyAsync(bm.data(), D.bitmap, 2048 * sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    CBGX_CUDA(cudaStreamSynchronize(st));
    std::vector<uint8_t> map(65536, 0xFF);
    std::vector<double> pv(256, 0.0);
    std::vector<int32_t> po(256, 0);
    uint32_t np = 0;
    for (uint32_t c = 0; c < 65536; ++c) {
        if (!(bm[c >> 5] >> (c & 31) & 1u)) continue;
        if (np == 255) return;  // more than 255 pairs: keep the 2-byte codes
        map[c] = static_cast<uint8_t>(np);
        pv[np] = d_val[c >> 8];
        po[np] = d_off[c & 0xFF];
        ++np;
    }
    const uint32_t g4 = D.ell_w / 4, g8 = (D.ell_w + 7) / 8;
    const uint64_t bytes = D.nslices * 32 * 8ull * g8;
    if (bytes > D.codes8_cap) {
        if (D.codes8) CBGX_CUDA(cudaFree(D.codes8));
        D.codes8 = nullptr;
        D.codes8_cap = 0;
        size_t free_b = 0, total_b = 0;
        CBGX_CUDA(cudaMemGetInfo(&free_b, &total_b));
        if (static_cast<double>(bytes) > 0.5 * static_cast<double>(free_b)) return;
        ensure(D.codes8, D.codes8_cap, bytes);
    }
    CBGX_CUDA(cudaMemcpyAsync(D.map8, map.data(), 65536, cudaMemcpyHostToDevice, st));
    CBGX_CUDA(cudaMemcpyAsync(D.pair_val, pv.data(), 256 * sizeof(double), cudaMemcpyHostToDevice, st));
    CBGX_CUDA(cudaMemcpyAsync(D.pair_off, po.data(), 256 * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    const uint64_t groups = D.nslices * 32 * g8;
    const int g2 = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((groups + 255) / 256, sm_count() * 8ull)));
    CBGX_K(pair_convert_kernel<<<g2, 256, 0, st>>>(D.codes, D.nslices, g4, g8, D.map8, D.codes8));
    CBGX_CUDA(cudaGetLastError());
    // the host vectors above are read by the async copies: finish them here
    CBGX_CUDA(cudaStreamSynchronize(st));
    D.entries8 = bytes;
    D.ell8_w = 8 * g8;
    D.n_pair = np;
    build_patterns(D, po, pv, st);
}

// Builds (or rebuilds, reusing D's buffers) the dictionary copy of A. One
// host round trip (the dictionaries); a second only for ragged matrices that
// need the per-slice offset table. Stream-ordered otherwise.
template <typename RP>
bool dict_build(const cbgx_csr& A, double reserve_bytes, cudaStream_t st, DictSell& D) {
    D.ready = false;
    const RP* rp = static_cast<const RP*>(A.d_row_ptr);
    uint64_t cap = 0;
    if (!D.tabs) {
        ensure(D.tabs, cap, 2ull * kSlots);
        ensure(D.flags, cap, 4);
        ensure(D.idx, cap, 2ull * kSlots);
        ensure(D.off, cap, 256);
        ensure(D.val, cap, 256);
    }
    // pass 1: dictionaries
    CBGX_CUDA(cudaMemsetAsync(D.tabs, 0xFF, 2 * kSlots * sizeof(unsigned long long), st));
    CBGX_CUDA(cudaMemsetAsync(D.flags, 0, 4 * sizeof(unsigned), st));
    CBGX_K(dict_scan_kernel<RP><<<dict_grid(A.n_rows), kDThreads, 0, st>>>(rp, A.d_col_idx, A.d_values, A.n_rows, D.tabs,
                                                                            D.tabs + kSlots, D.flags, D.flags + 2));
    CBGX_CUDA(cudaGetLastError());
    std::vector<unsigned long long> h_tabs(2 * kSlots);
    unsigned h_flags[4];
    CBGX_CUDA(cudaMemcpyAsync(h_tabs.data(), D.tabs, h_tabs.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CBGX_CUDA(cudaMemcpyAsync(h_flags, D.flags, sizeof h_flags, cudaMemcpyDeviceToHost, st));
    CBGX_CUDA(cudaStreamSynchronize(st));
    if (h_flags[2] || h_flags[0] > kDictMax || h_flags[1] > kDictMax) return false;
    // dense dictionaries + slot -> index maps
    std::vector<int32_t> d_off(256, 0);
    std::vector<double> d_val(256, 0.0);
    std::vector<uint8_t> idx(2 * kSlots, 0);
    uint32_t no = 0, nv = 0;
    for (uint32_t i = 0; i < kSlots; ++i) {
        if (h_tabs[i] != kEmpty) {
            d_off[no] = static_cast<int32_t>(static_cast<int64_t>(h_tabs[i]) - (1ll << 32));
            idx[i] = static_cast<uint8_t>(no++);
        }
        if (h_tabs[kSlots + i] != kEmpty) {
            const unsigned long long bits = h_tabs[kSlots + i];
            std::memcpy(&d_val[nv], &bits, 8);
            idx[kSlots + i] = static_cast<uint8_t>(nv++);
        }
    }
    D.nslices = (A.n_rows + 31) / 32;
    D.n_off = no;
    D.n_val = nv;
    D.ell_w = 0;
    // Uniform width padded to groups of 4 (ELL4) when that pads by <= 1/4
    // (7-point rows: 8, 27-point: 28): no offset table and one 8-byte code
    // load per 4 entries in the SpMV. Decided from the known longest row and
    // nnz when available (no pass over the row offsets).
    uint64_t total = 0;
    uint32_t max_w = A.max_row_nnz;
    const bool small = A.n_rows < (1ull << 31) - (1ull << 30);  // 32-bit row indices in the ELL4 kernel
    auto ell_fits = [&](uint32_t w, uint64_t entries) {
        const uint64_t t = D.nslices * 128 * static_cast<uint64_t>((w + 3) / 4);
        return w > 0 && small && t <= entries + entries / 4;
    };
    if (max_w > 0 && ell_fits(max_w, A.nnz)) {
        D.ell_w = 4 * ((max_w + 3) / 4);
        total = D.nslices * 32 * static_cast<uint64_t>(D.ell_w);
    } else {
        ensure(D.soff, D.soff_cap, D.nslices + 1);
        const int g1 = static_cast<int>(std::min<uint64_t>((D.nslices + 1 + 7) / 8 + 1, sm_count() * 16ull));
        CBGX_K(dict_slice_kernel<RP><<<g1, 256, 0, st>>>(rp, A.n_rows, D.nslices, D.soff, D.flags + 3));
        size_t tmp_bytes = 0;
        CBGX_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, D.soff, D.soff, D.nslices + 1, st));
        void* tmp = nullptr;
        CBGX_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
        CBGX_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, D.soff, D.soff, D.nslices + 1, st));
        CBGX_CUDA(cudaFreeAsync(tmp, st));
        unsigned mw = 0;
        CBGX_CUDA(cudaMemcpyAsync(&total, D.soff + D.nslices, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
        CBGX_CUDA(cudaMemcpyAsync(&mw, D.flags + 3, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        CBGX_CUDA(cudaStreamSynchronize(st));
        if (ell_fits(mw, total)) {
            D.ell_w = 4 * ((mw + 3) / 4);
            total = D.nslices * 32 * static_cast<uint64_t>(D.ell_w);
        }
    }
    if (total > D.codes_cap) {
        if (D.codes) CBGX_CUDA(cudaFree(D.codes));
        D.codes = nullptr;
        D.codes_cap = 0;
        size_t free_b = 0, total_b = 0;
        CBGX_CUDA(cudaMemGetInfo(&free_b, &total_b));
        if (static_cast<double>(total) * 2.0 > 0.8 * (static_cast<double>(free_b) - reserve_bytes)) return false;
        ensure(D.codes, D.codes_cap, total);
    }
    D.entries = total;
    CBGX_CUDA(cudaMemcpyAsync(D.idx, idx.data(), idx.size(), cudaMemcpyHostToDevice, st));
    CBGX_CUDA(cudaMemcpyAsync(D.off, d_off.data(), 256 * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    CBGX_CUDA(cudaMemcpyAsync(D.val, d_val.data(), 256 * sizeof(double), cudaMemcpyHostToDevice, st));
    CBGX_K(dict_fill_kernel<RP><<<dict_grid(D.nslices * 32), kDThreads, 0, st>>>(
        rp, A.d_col_idx, A.d_values, A.n_rows, D.soff, D.tabs, D.tabs + kSlots, D.idx, D.idx + kSlots, D.ell_w / 4,
        D.codes, D.flags + 2));  // flags[2] (scan failure) is 0 here
    CBGX_CUDA(cudaGetLastError());
    if (max_w == A.max_row_nnz && max_w > 0) {
        // the ELL width came from the caller's max_row_nnz hint (cbgx.h:
        // "0 = unknown"), not from a pass over the row offsets: verify it
        unsigned long_rows = 0;
        CBGX_CUDA(cudaMemcpyAsync(&long_rows, D.flags + 2, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
        CBGX_CUDA(cudaStreamSynchronize(st));
        if (long_rows) return false;
    }
    build_pairs(D, d_off, d_val, st);
    D.ready = true;
    return true;
}

}  // namespace

DictSell::~DictSell() {
    for (void* p : {static_cast<void*>(codes), static_cast<void*>(soff), static_cast<void*>(off), static_cast<void*>(val),
                    static_cast<void*>(tabs), static_cast<void*>(flags), static_cast<void*>(idx),
                    static_cast<void*>(codes8), static_cast<void*>(pair_val), static_cast<void*>(pair_off),
                    static_cast<void*>(map8), static_cast<void*>(bitmap), static_cast<void*>(pid),
                    static_cast<void*>(ptab), static_cast<void*>(pkeys), static_cast<void*>(pwords),
                    static_cast<void*>(pslot), static_cast<void*>(pcnt), static_cast<void*>(pmask)})
        if (p) cudaFree(p);
}

bool build_dict_sell(const cbgx_csr& A, double reserve_bytes, cudaStream_t st, DictSell& D) {
    D.ready = false;
    if (A.n_rows == 0 || A.nnz == 0) return false;
    // padding codes gather x[min(r, n_rows - 1)]: x must hold n_rows values
    if (A.n_cols < A.n_rows) return false;
    return A.row_ptr_bits == 32 ? dict_build<int32_t>(A, reserve_bytes, st, D)
                                : dict_build<int64_t>(A, reserve_bytes, st, D);
}

template <int MODE, bool kEll>
static void dict_launch(const cbgx_csr& A, const DictSell& D, const double* x, const double* b, double* y, int fused,
                        double* norm, Workspace* ws, cudaStream_t st, bool pdl) {
    static int per_sm = -1;  // per instantiation; one device geometry
    if (per_sm < 0) {
        CBGX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dsell_spmv_kernel<MODE, kEll>, kST, 0));
        per_sm = std::max(per_sm, 1);
    }
    const uint64_t want = (D.nslices + kSW - 1) / kSW;
    const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(want, static_cast<uint64_t>(sm_count()) * per_sm)));
    // fused == 2: per-CTA omega^2 partials into ws->omega_parts (no ticket)
    double* partials = fused == 2 ? ws->get_omega_parts(grid) : fused ? ws->get_partials(grid) : nullptr;
    unsigned* ticket = fused == 1 ? ws->get_counter() : nullptr;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(kST);
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = pdl ? 1 : 0;
    note_launch();
    CBGX_CUDA(cudaLaunchKernelEx(&lc, dsell_spmv_kernel<MODE, kEll>, A.n_rows, static_cast<const uint64_t*>(D.soff),
                                 D.ell_w, static_cast<const uint16_t*>(D.codes), static_cast<const int32_t*>(D.off),
                                 static_cast<const double*>(D.val), x, b, y, fused, partials, ticket, norm));
}

template <int MODE>
static uint32_t pell_launch(const cbgx_csr& A, const DictSell& D, const double* x, const double* b, double* y, int fused,
                        double* norm, Workspace* ws, cudaStream_t st, bool pdl, uint64_t s_begin = 0,
                        uint64_t s_end = ~0ull, bool accumulate = false) {
    static int per_sm = -1, per_sm_u = -1;  // pair/pattern kernels (PELL_MIN_BLOCKS); uniform slots
    if (per_sm < 0) {
        CBGX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pell_spmv_kernel<MODE, 0>, 256, 0));
        per_sm = std::max(per_sm, 1);
        CBGX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_u, uslot_spmv_kernel<MODE, 7>, 256, 0));
        per_sm_u = std::max(per_sm_u, 1);
    }
    // 32-bit row arithmetic: r + U * rstep stays below 2^31
    const bool uslot = D.n_slots && std::max(A.n_rows, A.n_cols) < (1ull << 31) - (1ull << 24);
    s_end = std::min<uint64_t>(s_end, D.nslices);
    if (s_begin >= s_end) return 0;
    const uint64_t want = (s_end - s_begin + 7) / 8;
    const int grid = static_cast<int>(std::max<uint64_t>(
        1, std::min<uint64_t>(want, static_cast<uint64_t>(sm_count()) * (uslot ? per_sm_u : per_sm))));
    // fused == 2: per-CTA omega^2 partials into ws->omega_parts (no ticket)
    double* partials = fused == 2 ? ws->get_omega_parts(grid) : fused ? ws->get_partials(grid) : nullptr;
    unsigned* ticket = fused == 1 ? ws->get_counter() : nullptr;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(256);
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = pdl ? 1 : 0;
    note_launch();
    if (uslot) {
        const uint32_t S = D.n_slots;
        auto k = S == 7 ? uslot_spmv_kernel<MODE, 7> : S == 27 ? uslot_spmv_kernel<MODE, 27>
               : S <= 8 ? uslot_spmv_kernel<MODE, 8> : S <= 16 ? uslot_spmv_kernel<MODE, 16>
               : S <= 24 ? uslot_spmv_kernel<MODE, 24> : uslot_spmv_kernel<MODE, 32>;
        USlots us;
        std::memcpy(&us, D.uslots, sizeof(USlots));
        CBGX_CUDA(cudaLaunchKernelEx(&lc, k, A.n_rows, A.n_cols, static_cast<const uint8_t*>(D.pid),
                                     static_cast<const uint32_t*>(D.pmask), D.n_pat, us, x, b, y, fused, partials,
                                     ticket, norm, s_begin, s_end, static_cast<int>(accumulate)));
        return static_cast<uint32_t>(grid);
    }
    if (D.n_pat && std::max(A.n_rows, A.n_cols) < (1ull << 31)) {
        const uint32_t G = D.ell8_w / 8;
        auto k = G == 1 ? ppat_spmv_kernel<MODE, 1> : G == 2 ? ppat_spmv_kernel<MODE, 2>
               : G == 3 ? ppat_spmv_kernel<MODE, 3> : ppat_spmv_kernel<MODE, 4>;
        lc.dynamicSmemBytes = static_cast<size_t>(D.ptab_u4) * 16;
        CBGX_CUDA(cudaLaunchKernelEx(&lc, k, A.n_rows, static_cast<const uint8_t*>(D.pid),
                                     static_cast<const uint4*>(D.ptab), D.ptab_u4,
                                     static_cast<const uint8_t*>(D.pcnt), x, b, y, fused, partials, ticket,
                                     norm, s_begin, s_end, static_cast<int>(accumulate)));
        return static_cast<uint32_t>(grid);
    }
    // G1's gather offsets are 32-bit byte offsets into x
    const bool g1 = PELL_G1 && D.ell8_w == 8 && std::max(A.n_rows, A.n_cols) * 8 < (1ull << 32);
    CBGX_CUDA(cudaLaunchKernelEx(&lc, g1 ? pell_spmv_kernel<MODE, 1> : pell_spmv_kernel<MODE, 0>, A.n_rows, D.ell8_w / 8,
                                 static_cast<const uint8_t*>(D.codes8), static_cast<const int32_t*>(D.pair_off),
                                 static_cast<const double*>(D.pair_val), x, b, y, fused, partials, ticket, norm,
                                 s_begin, s_end, static_cast<int>(accumulate), D.n_pair));
    return static_cast<uint32_t>(grid);
}

uint32_t launch_spmv_pell_parts(const cbgx_csr& A, const DictSell& D, const double* x, double* y, Workspace* ws,
                                cudaStream_t st, bool pdl) {
    if (!D.ell8_w) return 0;
    return pell_launch<0>(A, D, x, nullptr, y, 2, nullptr, ws, st, pdl);
}

void launch_spmv_pell_range(const cbgx_csr& A, const DictSell& D, const double* x, double* y, double* norm,
                            uint64_t s_begin, uint64_t s_end, bool accumulate, Workspace* ws, cudaStream_t st) {
    if (!D.ell8_w) throw Error(CBGX_EINTERNAL, "spmv: pair-coded copy missing");
    pell_launch<0>(A, D, x, nullptr, y, norm ? 1 : 0, norm, ws, st, false, s_begin, s_end, accumulate);
}

namespace {
template <typename RP>
__global__ void ghost_rows_kernel(const RP* __restrict__ rp, const int32_t* __restrict__ ci, uint64_t n, int64_t lo,
                                  unsigned long long* __restrict__ out) {
    for (uint64_t r = blockIdx.x * 256ull + threadIdx.x; r < n; r += gridDim.x * 256ull) {
        bool below = false, above = false;
        for (uint64_t k = static_cast<uint64_t>(rp[r]); k < static_cast<uint64_t>(rp[r + 1]); ++k) {
            const int64_t c = ci[k];
            below |= c < lo;
            above |= c >= lo + static_cast<int64_t>(n);
        }
        if (below) atomicMax(out, static_cast<unsigned long long>(r + 1));
        if (above) atomicMin(out + 1, static_cast<unsigned long long>(r));
    }
}
}  // namespace

void ghost_row_bounds(const cbgx_csr& A, uint64_t lo, uint64_t out[2], cudaStream_t st) {
    unsigned long long* d = nullptr;
    CBGX_CUDA(cudaMalloc(reinterpret_cast<void**>(&d), 2 * sizeof(unsigned long long)));
    const unsigned long long init[2] = {0ull, static_cast<unsigned long long>(A.n_rows)};
    CBGX_CUDA(cudaMemcpyAsync(d, init, sizeof(init), cudaMemcpyHostToDevice, st));
    const int grid = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((A.n_rows + 255) / 256, sm_count() * 8ull)));
    if (A.row_ptr_bits == 32)
        CBGX_K(ghost_rows_kernel<int32_t><<<grid, 256, 0, st>>>(static_cast<const int32_t*>(A.d_row_ptr), A.d_col_idx,
                                                                  A.n_rows, static_cast<int64_t>(lo), d));
    else
        CBGX_K(ghost_rows_kernel<int64_t><<<grid, 256, 0, st>>>(static_cast<const int64_t*>(A.d_row_ptr), A.d_col_idx,
                                                                  A.n_rows, static_cast<int64_t>(lo), d));
    unsigned long long h[2];
    CBGX_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
    CBGX_CUDA(cudaStreamSynchronize(st));
    CBGX_CUDA(cudaFree(d));
    out[0] = h[0];
    out[1] = h[1];
}

void launch_spmv_dict(const cbgx_csr& A, const DictSell& D, const double* x, const double* b, double* y, double* norm,
                      int reduction, Workspace* ws, cudaStream_t st, bool pdl) {
    const int fused = norm && reduction == CBGX_REDUCE_TREE;
    if (D.ell8_w) {
        if (b) pell_launch<1>(A, D, x, b, y, fused, norm, ws, st, pdl);
        else pell_launch<0>(A, D, x, b, y, fused, norm, ws, st, pdl);
    } else if (D.ell_w) {
        if (b) dict_launch<1, true>(A, D, x, b, y, fused, norm, ws, st, pdl);
        else dict_launch<0, true>(A, D, x, b, y, fused, norm, ws, st, pdl);
    } else {
        if (b) dict_launch<1, false>(A, D, x, b, y, fused, norm, ws, st, pdl);
        else dict_launch<0, false>(A, D, x, b, y, fused, norm, ws, st, pdl);
    }
    if (norm && !fused) launch_dot(y, y, A.n_rows, CBGX_REDUCE_REFERENCE, norm, ws, st);
}

}  // namespace cbgx

using namespace cbgx;

struct cbgx_dict_csr {
    std::unique_ptr<DictSell> d;
};

extern "C" {

int cbgx_csr_dict_create(const cbgx_csr* A, cbgx_dict_csr** out, void* stream) {
    return cbgx_csr_dict_create2(A, 3, out, stream);
}

int cbgx_csr_dict_create2(const cbgx_csr* A, uint32_t max_level, cbgx_dict_csr** out, void* stream) {
    return guard([&] {
        if (!A || !out) throw Error(CBGX_EINVAL, "dict: null argument");
        if (A->row_ptr_bits != 32 && A->row_ptr_bits != 64) throw Error(CBGX_EINVAL, "csr: row_ptr_bits must be 32 or 64");
        *out = nullptr;
        if (A->n_cols < A->n_rows) throw Error(CBGX_EINVAL, "dict: needs n_cols >= n_rows");
        if (max_level > 3) throw Error(CBGX_EINVAL, "dict: max_level must be 0, 1, 2 or 3");
        auto D = std::make_unique<DictSell>();
        D->max_level = max_level;
        if (!build_dict_sell(*A, 0.0, as_stream(stream), *D))
            throw Error(CBGX_EINVAL, "dict: matrix does not fit the dictionary format (more than 255 distinct values or column offsets, or a row longer than max_row_nnz)");
        CBGX_CUDA(cudaStreamSynchronize(as_stream(stream)));
        *out = new cbgx_dict_csr{std::move(D)};
    });
}

int cbgx_csr_dict_info(const cbgx_dict_csr* D, uint32_t* n_offsets, uint32_t* n_values, uint64_t* entries) {
    return guard([&] {
        if (!D) throw Error(CBGX_EINVAL, "dict: null handle");
        if (n_offsets) *n_offsets = D->d->n_off;
        if (n_values) *n_values = D->d->n_val;
        if (entries) *entries = D->d->entries;
    });
}

int cbgx_csr_dict_layout(const cbgx_dict_csr* D, uint32_t* level, uint32_t* n_pairs, uint32_t* n_patterns) {
    return guard([&] {
        if (!D) throw Error(CBGX_EINVAL, "dict: null handle");
        const DictSell& d = *D->d;
        if (level) *level = d.n_slots ? 4u : d.n_pat ? 3u : d.ell8_w ? 2u : d.ell_w ? 1u : 0u;
        if (n_pairs) *n_pairs = d.ell8_w ? d.n_pair : 0u;
        if (n_patterns) *n_patterns = d.n_pat;
    });
}

int cbgx_csr_dict_spmv(const cbgx_csr* A, const cbgx_dict_csr* D, const double* d_x, const double* d_b, double* d_y,
                       double* d_ynorm2, int reduction, cbgx_workspace* ws, void* stream) {
    return guard([&] {
        if (!A || !D) throw Error(CBGX_EINVAL, "dict: null argument");
        if (d_ynorm2 && !ws) throw Error(CBGX_EINVAL, "spmv: fused norm needs a workspace");
        launch_spmv_dict(*A, *D->d, d_x, d_b, d_y, d_ynorm2, reduction, ws_of(ws), as_stream(stream), false);
    });
}

void cbgx_csr_dict_destroy(cbgx_dict_csr* D) { delete D; }

}  // extern "C"
