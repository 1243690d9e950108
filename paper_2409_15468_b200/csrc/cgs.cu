// cgs.cu -- decompress-fused classical Gram-Schmidt kernels and the basis
// write/read kernels.
//
// Reference: KrylovBasis::dot / subtract_scaled (basis.cpp:168-205) called
// column by column from arnoldi_orthogonalize (gmres.cpp:36-71) and
// accumulate_solution (gmres.cpp:134-139). Here ONE launch handles all
// `cols` columns: a persistent CTA owns row tiles of kTileRows rows, keeps
// that tile of w in registers, and streams the tile's segment of every
// compressed column with 128-bit loads (double-buffered one column ahead),
// decoding in registers. w is read once per pass instead of once per
// column, and no decompressed basis value ever touches memory.
//
//   dot:    h_j = sum_i v_j[i] w[i]      (+ <w,w> fused when requested)
//   update: w[i] = w[i] - h_j v_j[i] for j in column order, two roundings,
//           bit-identical to the reference (+ <w_new,w_new> fused)
//
// Reductions are deterministic: per-warp partials per column accumulate in
// shared memory in tile order, CTAs write partial rows in CTA order, and the
// last CTA to finish (device ticket) sums the rows in CTA order.
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <map>
#include <set>
#include <tuple>
#include <utility>

#include "basis.cuh"
#include "pipeline.cuh"
#include "codec.cuh"
#include "common.cuh"
#include "reduce.cuh"
#include "runtime.h"

#ifndef FUSED_CTAS_PER_SM
#define FUSED_CTAS_PER_SM 2
#endif

namespace cbgx {

namespace {

// ---- geometry -------------------------------------------------------------
// Consumers: 8 warps; a step is 1024 rows (4 consecutive rows per thread);
// a sub-tile is up to Geo<F>::sub steps whose w stays in registers while every
// column's segment streams through a kStages-deep shared-memory ring filled
// by one producer thread with cp.async.bulk.
constexpr int kConsumerWarps = 8;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kThreads = kConsumers + 32;   // + producer warp
constexpr int kWarps = kConsumerWarps;      // reduction slots
constexpr uint32_t kStepRows = 4 * kConsumers;  // 1024

// Per format: payload / exponent bytes per 1024-row step, steps per
// sub-tile (w of a sub-tile lives in registers: sub * 4 doubles per thread)
// and ring depth. A ring stage holds one column's segment of a sub-tile.
template <int F> struct Geo;
template <> struct Geo<kZ32> { static constexpr uint32_t pay = 4096, ex = 128; static constexpr int sub = 4, stages = 4; };
#ifndef SPLIT_SUB_SMALL
#define SPLIT_SUB_SMALL 4
#endif
#ifndef SPLIT_STAGES_Z16
#define SPLIT_STAGES_Z16 6
#endif
#ifndef SPLIT_STAGES_Z21
#define SPLIT_STAGES_Z21 5
#endif
template <> struct Geo<kZ16> { static constexpr uint32_t pay = 2048, ex = 128; static constexpr int sub = SPLIT_SUB_SMALL, stages = SPLIT_STAGES_Z16; };
template <> struct Geo<kZ21> { static constexpr uint32_t pay = 2688, ex = 128; static constexpr int sub = SPLIT_SUB_SMALL, stages = SPLIT_STAGES_Z21; };
template <> struct Geo<kF64> { static constexpr uint32_t pay = 8192, ex = 0; static constexpr int sub = 4, stages = 3; };
template <> struct Geo<kF32> { static constexpr uint32_t pay = 4096, ex = 0; static constexpr int sub = 4, stages = 4; };
template <> struct Geo<kF16> { static constexpr uint32_t pay = 2048, ex = 0; static constexpr int sub = 4, stages = 6; };
static_assert(kRowAlign % (kStepRows * 8) == 0, "sub-tiles must divide the row padding");

template <int F>
__host__ __device__ constexpr uint32_t stage_bytes() {
    return Geo<F>::sub * (Geo<F>::pay + Geo<F>::ex) + 16;  // +16: l=21 loader reads one word past
}

// Split [s0, s1) into ceil(len/sub) sub-tiles of near-equal size (so no CTA
// ends with a 1-step remainder that costs a full ring round per column):
// the first `rem` tiles hold base + 1 steps, the others base. One division
// per launch; the per-tile bounds are multiply-adds (the per-stage 64-bit
// divisions of len * i / count showed up in the consumer loops).
struct SubTiles {
    uint64_t s0, count, base, rem;
    __device__ __forceinline__ uint64_t begin(uint64_t i) const { return s0 + i * base + min(i, rem); }
    __device__ __forceinline__ uint64_t end(uint64_t i) const { return begin(i + 1); }
};
template <int F>
__device__ __forceinline__ SubTiles sub_tiles(uint64_t s0, uint64_t s1) {
    const uint64_t len = s1 - s0;
    const uint64_t count = (len + Geo<F>::sub - 1) / Geo<F>::sub;
    return SubTiles{s0, count, count ? len / count : 0, count ? len % count : 0};
}

// ---- shared-memory step loaders (r = local row of the thread's 4 rows) ----
template <int F>
__device__ __forceinline__ void step_lds(Step<F>& st, const unsigned char* pay, const uint32_t* ex, uint32_t r);

template <>
__device__ __forceinline__ void step_lds<kZ32>(Step<kZ32>& st, const unsigned char* pay, const uint32_t* ex, uint32_t r) {
    st.c = *reinterpret_cast<const uint4*>(pay + 4u * r);
    st.e = ex[r / 32];
}
template <>
__device__ __forceinline__ void step_lds<kZ16>(Step<kZ16>& st, const unsigned char* pay, const uint32_t* ex, uint32_t r) {
    st.c = *reinterpret_cast<const uint2*>(pay + 2u * r);
    st.e = ex[r / 32];
}
template <>
__device__ __forceinline__ void step_lds<kZ21>(Step<kZ21>& st, const unsigned char* pay, const uint32_t* ex, uint32_t r) {
    const uint32_t* p = reinterpret_cast<const uint32_t*>(pay);
    const uint32_t bit = (r & 31u) * 21u;
    const uint32_t q = (r / 32) * 21 + (bit >> 5);
    st.sh = bit & 31u;
    st.w0 = p[q]; st.w1 = p[q + 1]; st.w2 = p[q + 2]; st.w3 = p[q + 3];
    st.e = ex[r / 32];
}
// Payload only (the exponent was read by the caller for the stage vote).
template <int F>
__device__ __forceinline__ void step_lds_pay(Step<F>& st, const unsigned char* pay, uint32_t r) {
    if constexpr (F == kZ32) {
        st.c = *reinterpret_cast<const uint4*>(pay + 4u * r);
    } else if constexpr (F == kZ16) {
        st.c = *reinterpret_cast<const uint2*>(pay + 2u * r);
    } else if constexpr (F == kZ21) {
        const uint32_t* p = reinterpret_cast<const uint32_t*>(pay);
        const uint32_t bit = (r & 31u) * 21u;
        const uint32_t q = (r / 32) * 21 + (bit >> 5);
        st.sh = bit & 31u;
        st.w0 = p[q]; st.w1 = p[q + 1]; st.w2 = p[q + 2]; st.w3 = p[q + 3];
    } else {
        step_lds<F>(st, pay, nullptr, r);
    }
}

template <>
__device__ __forceinline__ void step_lds<kF64>(Step<kF64>& st, const unsigned char* pay, const uint32_t*, uint32_t r) {
    const double2* p = reinterpret_cast<const double2*>(pay + 8u * r);
    st.a = p[0];
    st.b = p[1];
}
template <>
__device__ __forceinline__ void step_lds<kF32>(Step<kF32>& st, const unsigned char* pay, const uint32_t*, uint32_t r) {
    st.c = *reinterpret_cast<const float4*>(pay + 4u * r);
}
template <>
__device__ __forceinline__ void step_lds<kF16>(Step<kF16>& st, const unsigned char* pay, const uint32_t*, uint32_t r) {
    st.c = *reinterpret_cast<const uint2*>(pay + 2u * r);
}

// Per-thread offsets into a ring stage, constant for the whole launch: step s
// of the stage sits at + s * PAY bytes (payload) and + 32 s words (exponents),
// so the per-step addresses fold into immediates.
template <int F> struct StageOff {
    uint32_t pay;  // bytes
    uint32_t ex;   // words
    uint32_t sh;   // l=21: bit offset of the thread's first code in its window
    __device__ __forceinline__ StageOff() {
        const uint32_t t = threadIdx.x;
        if constexpr (F == kZ21) {
            const uint32_t bit = (t & 7u) * 84u;  // rows 4t..4t+3 of block t/8
            pay = ((t >> 3) * 21u + (bit >> 5)) * 4u;
            sh = bit & 31u;
        } else {
            pay = t * (Geo<F>::pay / kConsumers);  // 4 rows per thread
            sh = 0;
        }
        ex = t >> 3;
    }
};

// pay / ex: the stage base plus the thread's StageOff; step s at + s * PAY
// bytes and + s * EXW exponent words (defaults: the split kernels' 1024-row
// steps).
template <int F, uint32_t PAY = Geo<F>::pay, uint32_t EXW = 32>
__device__ __forceinline__ void step_lds_at(Step<F>& st, const unsigned char* pay, const uint32_t* ex, const StageOff<F>& o,
                                            int s, bool with_exp = true) {
    const unsigned char* p = pay + s * PAY;
    if constexpr (FmtInfo<F>::frsz) {
        if (with_exp) st.e = ex[EXW * s];
    }
    if constexpr (F == kZ32) {
        st.c = *reinterpret_cast<const uint4*>(p);
    } else if constexpr (F == kZ16) {
        st.c = *reinterpret_cast<const uint2*>(p);
    } else if constexpr (F == kZ21) {
        const uint32_t* q = reinterpret_cast<const uint32_t*>(p);
        st.sh = o.sh;
        st.w0 = q[0]; st.w1 = q[1]; st.w2 = q[2]; st.w3 = q[3];
    } else if constexpr (F == kF64) {
        st.a = reinterpret_cast<const double2*>(p)[0];
        st.b = reinterpret_cast<const double2*>(p)[1];
    } else if constexpr (F == kF32) {
        st.c = *reinterpret_cast<const float4*>(p);
    } else {
        st.c = *reinterpret_cast<const uint2*>(p);
    }
}

// One column's stage of a sub-tile. The exponents of all steps are read
// first and ONE warp vote decides the fast decode for the whole stage (the
// exact per-step path only when some block of the stage needs it); payloads
// are read step by step (reading them all up front spills at 3 CTAs/SM:
// slower for every format on B200). kFull: all Geo<F>::sub steps are present
// (every tile but the last), no per-step bounds checks.

template <int F, bool kFull>
__device__ __forceinline__ double stage_dot(const unsigned char* pay, const uint32_t* ex, const StageOff<F>& o,
                                            uint32_t steps, const double (&wv)[Geo<F>::sub][4]) {
    constexpr int SUB = Geo<F>::sub;
    Step<F> st[SUB];
    double acc = 0.0;
    if constexpr (FmtInfo<F>::frsz) {
        bool ok = true;
#pragma unroll
        for (int s = 0; s < SUB; ++s)
            if (kFull || s < steps) {
                st[s].e = ex[32 * s];
                ok &= st[s].fast();
            }
        if (__builtin_expect(__all_sync(0xFFFFFFFFu, ok), 1)) {
#pragma unroll
            for (int s = 0; s < SUB; ++s)
                if (kFull || s < steps) {
                    step_lds_at<F>(st[s], pay, ex, o, s, false);
                    acc = __dadd_rn(acc, st[s].dot_fast(wv[s]));
                }
            return acc;
        }
    }
#pragma unroll
    for (int s = 0; s < SUB; ++s)
        if (kFull || s < steps) {
            step_lds_at<F>(st[s], pay, ex, o, s);
            acc = __dadd_rn(acc, st[s].dot(wv[s]));
        }
    return acc;
}

template <int F, bool kFull>
__device__ __forceinline__ void stage_update(const unsigned char* pay, const uint32_t* ex, const StageOff<F>& o,
                                             uint32_t steps, double hj, int he, double (&wv)[Geo<F>::sub][4],
                                             bool colfast) {
    constexpr int SUB = Geo<F>::sub;
    Step<F> st[SUB];
    if constexpr (FmtInfo<F>::frsz) {
        if (colfast) {
            // the column's exponent range proves the fast update exact for
            // every block (col_upd_fast): no stage vote
#pragma unroll
            for (int s = 0; s < SUB; ++s)
                if (kFull || s < steps) {
                    step_lds_at<F>(st[s], pay, ex, o, s);
                    st[s].update_fast(hj, he, wv[s]);
                }
            return;
        }
        bool ok = true;
#pragma unroll
        for (int s = 0; s < SUB; ++s)
            if (kFull || s < steps) {
                st[s].e = ex[32 * s];
                ok &= st[s].upd_ok(hj, he);
            }
        if (__builtin_expect(__all_sync(0xFFFFFFFFu, ok), 1)) {
#pragma unroll
            for (int s = 0; s < SUB; ++s)
                if (kFull || s < steps) {
                    step_lds_at<F>(st[s], pay, ex, o, s, false);
                    st[s].update_fast(hj, he, wv[s]);
                }
            return;
        }
    }
#pragma unroll
    for (int s = 0; s < SUB; ++s)
        if (kFull || s < steps) {
            step_lds_at<F>(st[s], pay, ex, o, s);
            st[s].update(hj, he, wv[s]);
        }
}

// Per-column fast-update flags of a split update launch (shared memory,
// one byte per column; nullptr: no exponent ranges kept): col_upd_fast of
// the column's range and its coefficient (hs = the signed coefficients).
template <int F>
__device__ __forceinline__ void set_colfast(const BasisView& B, uint64_t first, uint32_t cols, const double* hs,
                                            uint8_t* cfl) {
    if constexpr (FmtInfo<F>::frsz) {
        if (!B.erange) return;
        for (uint32_t k = threadIdx.x; k < cols; k += blockDim.x) {
            const double hk = hs[k];
            cfl[k] = col_upd_fast<FmtInfo<F>::L>(B.erange[2 * (first + k)], B.erange[2 * (first + k) + 1], hk,
                                                 static_cast<int>(exp_field(hk)));
        }
    }
}
__device__ __forceinline__ bool colfast(const uint8_t* cfl, uint32_t j) { return cfl && cfl[j]; }

__device__ __forceinline__ void load_w(const double* __restrict__ w, uint64_t n, uint64_t r, double out[4]) {
    if (r + 3 < n) {
        load4(w + r, out);
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) out[k] = r + k < n ? w[r + k] : 0.0;
    }
}

// This CTA's step range: steps are split evenly over the grid (balanced to
// one 1024-row step), so no CTA owns a whole extra tile.
__device__ __forceinline__ void cta_steps(uint64_t n, uint64_t& s0, uint64_t& s1) {
    const uint64_t steps = (n + kStepRows - 1) / kStepRows;
    s0 = steps * blockIdx.x / gridDim.x;
    s1 = steps * (blockIdx.x + 1) / gridDim.x;
}

struct Ring {
    unsigned char* stages;
    uint64_t* full;
    uint64_t* empty;
};

template <int F>
__device__ __forceinline__ Ring ring_setup(unsigned char* smem) {
    constexpr int S = Geo<F>::stages;
    Ring r;
    r.stages = smem;
    r.full = reinterpret_cast<uint64_t*>(smem + S * stage_bytes<F>());
    r.empty = r.full + S;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(r.full + s, 1);
            mbar_init(r.empty + s, kConsumerWarps);
        }
        fence_barrier_init();
    }
    return r;
}

// Producer (one elected thread): for every sub-tile and column, wait for a
// free stage and bulk-copy the column's payload (+ exponent) segment.
template <int F>
__device__ __forceinline__ void produce(const Ring& R, const BasisView& B, uint64_t first, uint32_t cols,
                                        uint64_t s0, uint64_t s1, bool reverse) {
    constexpr int S = Geo<F>::stages;
    constexpr uint32_t PAY = Geo<F>::pay, EX = Geo<F>::ex;
    const uint64_t policy = policy_evict_normal();
    uint32_t it = 0;
    const SubTiles T = sub_tiles<F>(s0, s1);
    for (uint64_t t = 0; t < T.count; ++t) {
        const uint64_t sb = T.begin(t);
        const uint32_t steps = static_cast<uint32_t>(T.end(t) - sb);
        const uint32_t pb = steps * PAY, eb = steps * EX;
        for (uint32_t jj = 0; jj < cols; ++jj, ++it) {
            const uint32_t j = reverse ? cols - 1 - jj : jj;
            const int stage = it % S;
            mbar_wait(R.empty + stage, ((it / S) & 1) ^ 1);
            mbar_arrive_expect_tx(R.full + stage, pb + eb);
            unsigned char* dst = R.stages + stage * stage_bytes<F>();
            const unsigned char* col = B.data + (first + j) * B.col_stride_bytes;
            bulk_g2s(dst, col + sb * PAY, pb, R.full + stage, policy);
            if constexpr (EX > 0) {
                const unsigned char* ecol = reinterpret_cast<const unsigned char*>(B.exp + (first + j) * B.exp_col_stride);
                bulk_g2s(dst + Geo<F>::sub * PAY, ecol + sb * EX, eb, R.full + stage, policy);
            }
        }
    }
}

// ------------------------------------------------------------------ dot
// Resident CTAs per SM the split kernels are register-budgeted for (w of a
// sub-tile lives in registers: sub * 4 doubles per thread).
template <int F>
constexpr int split_min_blocks() { return Geo<F>::sub > 4 ? 2 : 3; }

template <int F>
__global__ void __launch_bounds__(kThreads, split_min_blocks<F>())
cgs_dot_kernel(BasisView B, uint64_t first, uint32_t cols, const double* __restrict__ w,
               int with_wnorm, double* __restrict__ partials, unsigned* __restrict__ ticket,
               double* __restrict__ h_out, GateArg gate) {
    if (!gate.open()) return;  // re-orthogonalisation pass not needed
    constexpr int S = Geo<F>::stages;
    constexpr uint32_t PAY = Geo<F>::pay;
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t ncol = cols + (with_wnorm ? 1 : 0);
    const Ring R = ring_setup<F>(smem);
    double* red = reinterpret_cast<double*>(R.empty + S);  // [kWarps][ncol]
    for (uint32_t k = threadIdx.x; k < kWarps * ncol; k += kThreads) red[k] = 0.0;
    __syncthreads();
    uint64_t s0, s1;
    cta_steps(B.n, s0, s1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == kConsumerWarps) {
        if (lane == 0) produce<F>(R, B, first, cols, s0, s1, true);
    } else {
        const StageOff<F> off;
        uint32_t it = 0;
        const SubTiles T = sub_tiles<F>(s0, s1);
        for (uint64_t t = 0; t < T.count; ++t) {
            const uint64_t sb = T.begin(t);
            const uint32_t steps = static_cast<uint32_t>(T.end(t) - sb);
            double wv[Geo<F>::sub][4];
#pragma unroll
            for (int s = 0; s < Geo<F>::sub; ++s) {
                if (s < steps) load_w(w, B.n, (sb + s) * kStepRows + 4u * threadIdx.x, wv[s]);
                else wv[s][0] = wv[s][1] = wv[s][2] = wv[s][3] = 0.0;
            }
            if (with_wnorm) {
                double acc = 0.0;
#pragma unroll
                for (int s = 0; s < Geo<F>::sub; ++s)
#pragma unroll
                    for (int k = 0; k < 4; ++k) acc = fma(wv[s][k], wv[s][k], acc);
                acc = warp_sum(acc);
                if (lane == 0) red[warp * ncol + cols] += acc;
            }
            // Columns stream last-to-first: the preceding update pass ended on
            // the high columns, so they are still in L2 (and the following
            // update starts on the low columns this pass ends with).
            for (uint32_t jj = 0; jj < cols; ++jj, ++it) {
                const uint32_t j = cols - 1 - jj;
                const int stage = it % S;
                mbar_wait(R.full + stage, (it / S) & 1);
                const unsigned char* pay = R.stages + stage * stage_bytes<F>();
                const uint32_t* ex = reinterpret_cast<const uint32_t*>(pay + Geo<F>::sub * PAY);
                double acc = steps == Geo<F>::sub ? stage_dot<F, true>(pay + off.pay, ex + off.ex, off, steps, wv)
                                                  : stage_dot<F, false>(pay + off.pay, ex + off.ex, off, steps, wv);
                __syncwarp();
                if (lane == 0) mbar_arrive(R.empty + stage);
                acc = warp_sum(acc);
                if (lane == 0) red[warp * ncol + j] += acc;
            }
        }
    }
    __syncthreads();
    block_finalize(red, kWarps, ncol, partials, ticket, h_out);
}

// --------------------------------------------------------------- update
template <int F>
__global__ void __launch_bounds__(kThreads, split_min_blocks<F>())
cgs_update_kernel(BasisView B, uint64_t first, uint32_t cols, const double* __restrict__ h,
                  double h_sign, double* __restrict__ w, int with_norm,
                  double* __restrict__ partials, unsigned* __restrict__ ticket,
                  double* __restrict__ norm_out, GateArg gate) {
    if (!gate.open()) return;
    constexpr int S = Geo<F>::stages;
    constexpr uint32_t PAY = Geo<F>::pay;
    extern __shared__ __align__(128) unsigned char smem[];
    const Ring R = ring_setup<F>(smem);
    double* hs = reinterpret_cast<double*>(R.empty + S);  // [cols]
    double* red = hs + cols;                               // [kWarps]
    uint8_t* cfl = B.erange ? reinterpret_cast<uint8_t*>(red + kWarps) : nullptr;  // [cols]
    for (uint32_t k = threadIdx.x; k < cols; k += kThreads) hs[k] = h_sign * h[k];
    set_colfast<F>(B, first, cols, hs, cfl);
    if (threadIdx.x < kWarps) red[threadIdx.x] = 0.0;
    __syncthreads();
    uint64_t s0, s1;
    cta_steps(B.n, s0, s1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == kConsumerWarps) {
        if (lane == 0) produce<F>(R, B, first, cols, s0, s1, false);
    } else {
        const StageOff<F> off;
        uint32_t it = 0;
        double nacc = 0.0;
        const SubTiles T = sub_tiles<F>(s0, s1);
        for (uint64_t t = 0; t < T.count; ++t) {
            const uint64_t sb = T.begin(t);
            const uint32_t steps = static_cast<uint32_t>(T.end(t) - sb);
            double wv[Geo<F>::sub][4];
#pragma unroll
            for (int s = 0; s < Geo<F>::sub; ++s) {
                if (s < steps) load_w(w, B.n, (sb + s) * kStepRows + 4u * threadIdx.x, wv[s]);
                else wv[s][0] = wv[s][1] = wv[s][2] = wv[s][3] = 0.0;
            }
            for (uint32_t j = 0; j < cols; ++j, ++it) {
                const int stage = it % S;
                mbar_wait(R.full + stage, (it / S) & 1);
                const unsigned char* pay = R.stages + stage * stage_bytes<F>();
                const uint32_t* ex = reinterpret_cast<const uint32_t*>(pay + Geo<F>::sub * PAY);
                const double hj = hs[j];
                const int he = static_cast<int>(exp_field(hj));
                const bool cf = colfast(cfl, j);
                if (steps == Geo<F>::sub) stage_update<F, true>(pay + off.pay, ex + off.ex, off, steps, hj, he, wv, cf);
                else stage_update<F, false>(pay + off.pay, ex + off.ex, off, steps, hj, he, wv, cf);
                __syncwarp();
                if (lane == 0) mbar_arrive(R.empty + stage);
            }
#pragma unroll
            for (int s = 0; s < Geo<F>::sub; ++s) {
                if (s >= steps) break;
                const uint64_t r = (sb + s) * kStepRows + 4u * threadIdx.x;
                if (r + 3 < B.n) {
                    store4(w + r, wv[s]);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (r + k < B.n) w[r + k] = wv[s][k];
                }
                if (with_norm) {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (r + k < B.n) nacc = fma(wv[s][k], wv[s][k], nacc);
                }
            }
        }
        if (with_norm) {
            nacc = warp_sum(nacc);
            if (lane == 0) red[warp] = nacc;
        }
    }
    __syncthreads();
    if (with_norm) block_finalize(red, kWarps, 1, partials, ticket, norm_out);
}

// ------------------------------------------------ update, dynamic tiles
// Same pass as cgs_update_kernel, but the sub-tiles are handed out through a
// device counter (the producer takes the next one when it has a free stage),
// so faster SMs take more tiles: the static split leaves every launch waiting
// for the slowest CTA (per-SM throughput differs by ~10% on B200). Rows are
// still updated exactly once in column order (bit-identical); the optional
// <w, w> is summed per tile and the tiles in tile order -- deterministic
// whatever the assignment.
constexpr uint32_t kTileEnd = 0xFFFFFFFFu;
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Poll with relaxed loads and acquire once the target is seen: an acquire
// load at gpu scope invalidates the SM's L1 (CCTL.IVALL) on every spin,
// under the co-resident CTA's feet.
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void wait_count(const unsigned* p, unsigned target) {
    while (ld_relaxed_u32(p) < target) {
    }
    (void)ld_acquire_u32(p);
}

__device__ __forceinline__ void split_consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
}



template <int F>
__global__ void __launch_bounds__(kThreads, split_min_blocks<F>())
cgs_update_dyn_kernel(BasisView B, uint64_t first, uint32_t cols, const double* __restrict__ h,
                      double h_sign, double* __restrict__ w, int with_norm,
                      double* __restrict__ tile_norms, unsigned* __restrict__ counters,
                      double* __restrict__ norm_out, GateArg gate) {
    if (!gate.open()) return;
    constexpr int S = Geo<F>::stages;
    constexpr uint32_t PAY = Geo<F>::pay, EX = Geo<F>::ex;
    extern __shared__ __align__(128) unsigned char smem[];
    const Ring R = ring_setup<F>(smem);
    double* hs = reinterpret_cast<double*>(R.empty + S);  // [cols]
    double* red = hs + cols;                               // [kWarps]
    uint32_t* tid_ring = reinterpret_cast<uint32_t*>(red + kWarps);  // [S]
    uint8_t* cfl = B.erange ? reinterpret_cast<uint8_t*>(tid_ring + S) : nullptr;  // [cols]
    __shared__ bool s_last;
    for (uint32_t k = threadIdx.x; k < cols; k += kThreads) hs[k] = h_sign * h[k];
    set_colfast<F>(B, first, cols, hs, cfl);
    __syncthreads();
    const uint64_t nsteps = (B.n + kStepRows - 1) / kStepRows;
    const uint32_t ntiles = static_cast<uint32_t>((nsteps + Geo<F>::sub - 1) / Geo<F>::sub);
    unsigned* tile_ctr = counters + 2;
    unsigned* ticket = counters + 3;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == kConsumerWarps) {
        if (lane == 0) {
            const uint64_t policy = policy_evict_normal();
            uint32_t it = 0;
            for (;;) {
                const uint32_t tile = atomicAdd(tile_ctr, 1u);
                if (tile >= ntiles) break;
                const uint64_t sb = static_cast<uint64_t>(tile) * Geo<F>::sub;
                const uint32_t steps = static_cast<uint32_t>(min(static_cast<uint64_t>(Geo<F>::sub), nsteps - sb));
                const uint32_t pb = steps * PAY, eb = steps * EX;
                for (uint32_t j = 0; j < cols; ++j, ++it) {
                    const int stage = it % S;
                    mbar_wait(R.empty + stage, ((it / S) & 1) ^ 1);
                    tid_ring[stage] = tile;
                    mbar_arrive_expect_tx(R.full + stage, pb + eb);
                    unsigned char* dst = R.stages + stage * stage_bytes<F>();
                    bulk_g2s(dst, B.data + (first + j) * B.col_stride_bytes + sb * PAY, pb, R.full + stage, policy);
                    if constexpr (EX > 0)
                        bulk_g2s(dst + Geo<F>::sub * PAY,
                                 reinterpret_cast<const unsigned char*>(B.exp + (first + j) * B.exp_col_stride) + sb * EX,
                                 eb, R.full + stage, policy);
                }
            }
            // sentinel stage: no data, tells the consumers to stop
            const int stage = it % S;
            mbar_wait(R.empty + stage, ((it / S) & 1) ^ 1);
            tid_ring[stage] = kTileEnd;
            mbar_arrive(R.full + stage);
        }
    } else {
        const StageOff<F> off;
        uint32_t it = 0;
        for (;;) {
            const int stage0 = it % S;
            mbar_wait(R.full + stage0, (it / S) & 1);
            const uint32_t tile = tid_ring[stage0];
            if (tile == kTileEnd) break;
            const uint64_t sb = static_cast<uint64_t>(tile) * Geo<F>::sub;
            const uint32_t steps = static_cast<uint32_t>(min(static_cast<uint64_t>(Geo<F>::sub), nsteps - sb));
            double wv[Geo<F>::sub][4];
#pragma unroll
            for (int s = 0; s < Geo<F>::sub; ++s) {
                if (s < steps) load_w(w, B.n, (sb + s) * kStepRows + 4u * threadIdx.x, wv[s]);
                else wv[s][0] = wv[s][1] = wv[s][2] = wv[s][3] = 0.0;
            }
            for (uint32_t j = 0; j < cols; ++j, ++it) {
                const int stage = it % S;
                if (j) mbar_wait(R.full + stage, (it / S) & 1);
                const unsigned char* pay = R.stages + stage * stage_bytes<F>();
                const uint32_t* ex = reinterpret_cast<const uint32_t*>(pay + Geo<F>::sub * PAY);
                const double hj = hs[j];
                const int he = static_cast<int>(exp_field(hj));
                const bool cf = colfast(cfl, j);
                if (steps == Geo<F>::sub) stage_update<F, true>(pay + off.pay, ex + off.ex, off, steps, hj, he, wv, cf);
                else stage_update<F, false>(pay + off.pay, ex + off.ex, off, steps, hj, he, wv, cf);
                __syncwarp();
                if (lane == 0) mbar_arrive(R.empty + stage);
            }
            double nacc = 0.0;
#pragma unroll
            for (int s = 0; s < Geo<F>::sub; ++s) {
                if (s >= steps) break;
                const uint64_t r = (sb + s) * kStepRows + 4u * threadIdx.x;
                if (r + 3 < B.n) {
                    store4(w + r, wv[s]);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (r + k < B.n) w[r + k] = wv[s][k];
                }
                if (with_norm) {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (r + k < B.n) nacc = fma(wv[s][k], wv[s][k], nacc);
                }
            }
            if (with_norm) {
                // this tile's <w, w>: warps in order
                nacc = warp_sum(nacc);
                split_consumer_sync();
                if (lane == 0) red[warp] = nacc;
                split_consumer_sync();
                if (threadIdx.x == 0) {
                    double t = red[0];
                    for (int k = 1; k < kWarps; ++k) t = __dadd_rn(t, red[k]);
                    tile_norms[tile] = t;
                }
            }
        }
    }
    // last CTA: reset the tile counter; sum the tile norms in tile order
    __syncthreads();
    __threadfence();
    if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x == 0) {
        *tile_ctr = 0u;
        *ticket = 0u;
    }
    if (with_norm && warp == 0) {
        double v = 0.0;
        for (uint32_t t0 = lane; t0 < ntiles; t0 += 32) v = __dadd_rn(v, __ldcg(tile_norms + t0));
        v = warp_sum(v);
        if (lane == 0) *norm_out = v;
    }
}

// --------------------------------------------------- dot, dynamic tiles
// Tiles handed out as in cgs_update_dyn_kernel. Partial sums are kept per
// TILE (column-major table part[col * ntiles + tile], warps of the tile in
// order), so the grouping never depends on which CTA took which tile; after a
// grid barrier (cooperative launch: every CTA is resident) each CTA reduces
// its share of the columns over the tiles in one fixed order.
template <int F>
__global__ void __launch_bounds__(kThreads, split_min_blocks<F>())
cgs_dot_dyn_kernel(BasisView B, uint64_t first, uint32_t cols, const double* __restrict__ w,
                   int with_wnorm, double* __restrict__ part, unsigned* __restrict__ counters,
                   double* __restrict__ h_out, GateArg gate) {
    if (!gate.open()) return;  // re-orthogonalisation pass not needed
    constexpr int S = Geo<F>::stages;
    constexpr uint32_t PAY = Geo<F>::pay, EX = Geo<F>::ex;
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t ncol = cols + (with_wnorm ? 1 : 0);
    const Ring R = ring_setup<F>(smem);
    double* red = reinterpret_cast<double*>(R.empty + S);  // [kWarps][ncol]
    uint32_t* tid_ring = reinterpret_cast<uint32_t*>(red + kWarps * ncol);  // [S]
    __syncthreads();
    const uint64_t nsteps = (B.n + kStepRows - 1) / kStepRows;
    const uint32_t ntiles = static_cast<uint32_t>((nsteps + Geo<F>::sub - 1) / Geo<F>::sub);
    unsigned* tile_ctr = counters + 4;
    unsigned* arrive = counters + 5;
    unsigned* ticket = counters + 6;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == kConsumerWarps) {
        if (lane == 0) {
            const uint64_t policy = policy_evict_normal();
            uint32_t it = 0;
            for (;;) {
                const uint32_t tile = atomicAdd(tile_ctr, 1u);
                if (tile >= ntiles) break;
                const uint64_t sb = static_cast<uint64_t>(tile) * Geo<F>::sub;
                const uint32_t steps = static_cast<uint32_t>(min(static_cast<uint64_t>(Geo<F>::sub), nsteps - sb));
                const uint32_t pb = steps * PAY, eb = steps * EX;
                for (uint32_t jj = 0; jj < cols; ++jj, ++it) {
                    const uint32_t j = cols - 1 - jj;  // last-to-first (L2 reuse after an update pass)
                    const int stage = it % S;
                    mbar_wait(R.empty + stage, ((it / S) & 1) ^ 1);
                    tid_ring[stage] = tile;
                    mbar_arrive_expect_tx(R.full + stage, pb + eb);
                    unsigned char* dst = R.stages + stage * stage_bytes<F>();
                    bulk_g2s(dst, B.data + (first + j) * B.col_stride_bytes + sb * PAY, pb, R.full + stage, policy);
                    if constexpr (EX > 0)
                        bulk_g2s(dst + Geo<F>::sub * PAY,
                                 reinterpret_cast<const unsigned char*>(B.exp + (first + j) * B.exp_col_stride) + sb * EX,
                                 eb, R.full + stage, policy);
                }
                if (cols == 0) {  // <w, w> only: one empty stage per tile
                    const int stage = it % S;
                    mbar_wait(R.empty + stage, ((it / S) & 1) ^ 1);
                    tid_ring[stage] = tile;
                    mbar_arrive(R.full + stage);
                    ++it;
                }
            }
            const int stage = it % S;
            mbar_wait(R.empty + stage, ((it / S) & 1) ^ 1);
            tid_ring[stage] = kTileEnd;
            mbar_arrive(R.full + stage);
        }
    } else {
        const StageOff<F> off;
        uint32_t it = 0;
        const uint32_t per_tile = cols ? cols : 1u;
        for (;;) {
            const int stage0 = it % S;
            mbar_wait(R.full + stage0, (it / S) & 1);
            const uint32_t tile = tid_ring[stage0];
            if (tile == kTileEnd) break;
            const uint64_t sb = static_cast<uint64_t>(tile) * Geo<F>::sub;
            const uint32_t steps = static_cast<uint32_t>(min(static_cast<uint64_t>(Geo<F>::sub), nsteps - sb));
            double wv[Geo<F>::sub][4];
#pragma unroll
            for (int s = 0; s < Geo<F>::sub; ++s) {
                if (s < steps) load_w(w, B.n, (sb + s) * kStepRows + 4u * threadIdx.x, wv[s]);
                else wv[s][0] = wv[s][1] = wv[s][2] = wv[s][3] = 0.0;
            }
            if (with_wnorm) {
                double acc = 0.0;
#pragma unroll
                for (int s = 0; s < Geo<F>::sub; ++s)
#pragma unroll
                    for (int k = 0; k < 4; ++k) acc = fma(wv[s][k], wv[s][k], acc);
                acc = warp_sum(acc);
                if (lane == 0) red[warp * ncol + cols] = acc;
            }
            // one column's stage: wait (the tile's first stage was waited on
            // above), the lane's partial, release the stage
            auto column = [&](uint32_t jj) -> double {
                const int stage = it % S;
                if (jj) mbar_wait(R.full + stage, (it / S) & 1);
                const unsigned char* pay = R.stages + stage * stage_bytes<F>();
                const uint32_t* ex = reinterpret_cast<const uint32_t*>(pay + Geo<F>::sub * PAY);
                const double acc = steps == Geo<F>::sub
                                       ? stage_dot<F, true>(pay + off.pay, ex + off.ex, off, steps, wv)
                                       : stage_dot<F, false>(pay + off.pay, ex + off.ex, off, steps, wv);
                __syncwarp();
                if (lane == 0) mbar_arrive(R.empty + stage);
                ++it;
                return acc;
            };
            if (cols) {
                uint32_t jj = 0;
                for (; jj < cols; ++jj) {
                    const double v = warp_sum(column(jj));
                    if (lane == 0) red[warp * ncol + cols - 1 - jj] = v;
                }
            } else {
                const int stage = it % S;
                __syncwarp();
                if (lane == 0) mbar_arrive(R.empty + stage);
                ++it;
            }
            // this tile's partials: warps in order, column-major table
            split_consumer_sync();
            for (uint32_t k = threadIdx.x; k < ncol; k += kConsumers) {
                double t = red[k];
                for (int q = 1; q < kWarps; ++q) t = __dadd_rn(t, red[q * ncol + k]);
                part[static_cast<uint64_t>(k) * ntiles + tile] = t;
            }
            split_consumer_sync();
        }
    }
    // grid barrier (all CTAs resident: cooperative launch)
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(arrive, 1u);
        wait_count(arrive, gridDim.x);
    }
    __syncthreads();
    // columns k = blockIdx.x, blockIdx.x + gridDim.x, ...: every thread sums
    // the tiles t, t + kThreads, ... of the column, then warp 0 adds the
    // kThreads partials lane-strided and a butterfly (fixed shape)
    double* csum = red;  // the per-tile scratch is free now (>= kThreads doubles, see the launcher)
    for (uint32_t k = blockIdx.x; k < ncol; k += gridDim.x) {
        const double* col = part + static_cast<uint64_t>(k) * ntiles;
        double v = 0.0, x[8];
        for (uint32_t t0 = threadIdx.x; t0 < ntiles; t0 += kThreads * 8) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint32_t t = t0 + kThreads * q;
                x[q] = t < ntiles ? __ldcg(col + t) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (t0 + kThreads * q < ntiles) v = __dadd_rn(v, x[q]);
        }
        __syncthreads();
        csum[threadIdx.x] = v;
        __syncthreads();
        if (warp == 0) {
            double u = 0.0;
            for (uint32_t i = lane; i < static_cast<uint32_t>(kThreads); i += 32) u = __dadd_rn(u, csum[i]);
            u = warp_sum(u);
            if (lane == 0) h_out[k] = u;
        }
    }
    // the last CTA out resets the counters for the next launch
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(ticket, 1u) == gridDim.x - 1) {
            *tile_ctr = 0u;
            *arrive = 0u;
            *ticket = 0u;
            __threadfence();
        }
    }
}

// ------------------------------------------------- reference-order dot
// One thread per column, the exact order of KrylovBasis::dot: per 32-block
// partial from +0.0 left to right, then a running total over blocks
// (basis.cpp:176-186). Thread `cols` (if with_wnorm) does norm2's
// sequential <w,w> (sparse.cpp:62-66).
template <int F>
__global__ void serial_dot_kernel(BasisView B, uint64_t first, uint32_t cols,
                                  const double* __restrict__ w, int with_wnorm,
                                  double* __restrict__ h_out, GateArg gate) {
    if (!gate.open()) return;
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < cols) {
        double total = 0.0;
        const uint64_t nb = (B.n + 31) / 32;
        for (uint64_t b = 0; b < nb; ++b) {
            double part = 0.0;
            const uint64_t have = (B.n - b * 32) < 32 ? (B.n - b * 32) : 32;
            for (uint64_t r = 0; r < have; ++r) {
                const uint64_t i = b * 32 + r;
                part = __dadd_rn(part, __dmul_rn(basis_value<F>(B, first + j, i), w[i]));
            }
            total = __dadd_rn(total, part);
        }
        h_out[j] = total;
    } else if (j == cols && with_wnorm) {
        double s = 0.0;
        for (uint64_t i = 0; i < B.n; ++i) s = __dadd_rn(s, __dmul_rn(w[i], w[i]));
        h_out[cols] = s;
    }
}

// --------------------------------------------------------- write / read
template <int F>
__global__ void write_plain_kernel(unsigned char* __restrict__ col, const double* __restrict__ x,
                                   uint64_t n, uint64_t n_pad, ScaleArg scale, double* __restrict__ v_out) {
    const double s = scale.value();
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n_pad;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        double v = 0.0;
        if (i < n) {
            v = x[i];
            if (scale.src) v = __dmul_rn(v, s);
            if (v_out) v_out[i] = v;
        }
        if constexpr (F == kF64) reinterpret_cast<double*>(col)[i] = v;
        else if constexpr (F == kF32) reinterpret_cast<float*>(col)[i] = __double2float_rn(v);
        else reinterpret_cast<uint16_t*>(col)[i] = double_to_half_bits(v);
    }
}

template <int F>
__global__ void read_kernel(BasisView B, uint64_t col, uint64_t first, uint64_t count,
                            double* __restrict__ out) {
    for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < count;
         k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t i = first + k;
        out[k] = i < B.n ? basis_value<F>(B, col, i) : 0.0;
    }
}

template <template <int> class K, class... A>
void dispatch_fmt(int f, A&&... a) {
    switch (f) {
    case kF64: K<kF64>::run(a...); break;
    case kF32: K<kF32>::run(a...); break;
    case kF16: K<kF16>::run(a...); break;
    case kZ16: K<kZ16>::run(a...); break;
    case kZ21: K<kZ21>::run(a...); break;
    default: K<kZ32>::run(a...); break;
    }
}

// Persistent grid: as many CTAs as fit (smem-limited), never more than
// there are 1024-row steps.
// Persistent grid: all CTAs that can be co-resident (registers and shared
// memory via the occupancy calculator), never more than 1024-row steps.
// Occupancy query cached per (device, kernel, smem): it costs host time on
// every launch otherwise.
template <class K>
int occupancy(K kernel, size_t smem) {
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, size_t>, int> cache;
    const auto key = std::make_tuple(current_device(), reinterpret_cast<const void*>(kernel), smem);
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int per_sm = 0;
    CBGX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, smem));
    cache.emplace(key, per_sm);
    return per_sm;
}

template <class K>
int ring_grid(K kernel, uint64_t n, size_t smem) {
    const int per_sm = occupancy(kernel, smem);
    const uint64_t steps = (n + kStepRows - 1) / kStepRows;
    const uint64_t cap = static_cast<uint64_t>(sm_count()) * std::max(per_sm, 1);
    return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(steps, cap)));
}

template <int F>
size_t ring_smem(size_t extra_doubles) {
    return Geo<F>::stages * (stage_bytes<F>() + 16) + extra_doubles * sizeof(double);
}

// Raise the dynamic shared-memory limit once per kernel (per device).
template <class K>
void allow_smem(K kernel) {
    static std::mutex mu;
    static std::set<std::pair<int, const void*>> done;
    const auto key = std::make_pair(current_device(), reinterpret_cast<const void*>(kernel));
    std::lock_guard<std::mutex> lock(mu);
    if (done.count(key)) return;
    CBGX_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    done.insert(key);
}

// ------------------------------------------------------------ read sweep
// The device analogue of the reference's read benchmark (bench.cpp:55-96,
// the paper's Fig. 3) on the CGS decode path: a producer lane bulk-copies
// the column's sub-tiles (Geo<F>::sub steps of 1024 rows, payload +
// exponents) into the split kernels' ring; the consumer warps read a
// stage's exponents first, take ONE warp vote for the fast decode, decode 4
// values per thread per step from shared memory, apply `intensity`
// multiply-adds (buf = buf * mul + add, two roundings as the reference's
// -ffp-contract=off build) and fold them into a per-thread sum. Static,
// balanced step ranges per CTA, so the checksum's tree (CTA partials in CTA
// order) depends only on the grid -- deterministic.
template <int F, bool kFull>
__device__ __forceinline__ double stage_sweep(const unsigned char* pay, const uint32_t* ex, const StageOff<F>& o,
                                              uint32_t steps, uint64_t row0, uint64_t n, int intensity, double mul,
                                              double add, bool fold_ok, uint32_t e_lo, uint32_t e_span) {
    constexpr int SUB = Geo<F>::sub;
    Step<F> st[SUB];
    bool fast = true;
    if constexpr (FmtInfo<F>::frsz) {
#pragma unroll
        for (int s = 0; s < SUB; ++s)
            if (kFull || s < static_cast<int>(steps)) {
                st[s].e = ex[32 * s];
                fast &= st[s].fast();
            }
        fast = __all_sync(0xFFFFFFFFu, fast);
    }
    // decode the whole stage, then ONE multiply-add loop over its 4 * SUB
    // values (the loop control amortised over the stage). FRSZ2 fast path:
    // the first multiply is folded into the decode (+-mag * RN(scale * mul),
    // bit-identical to RN(decode * mul) when scale * mul is exact -- voted
    // with the decode path), saving one FP64 multiply per value.
    double v[SUB][4];
    bool folded = false;
    if constexpr (FmtInfo<F>::frsz) {
        // scale * mul is exact iff it stays normal: a range of block
        // exponents fixed by mul's exponent (integer check on e, no FP test)
        bool ok = fast && fold_ok;
        if (ok) {
#pragma unroll
            for (int s = 0; s < SUB; ++s)
                if (kFull || s < static_cast<int>(steps)) ok &= st[s].e - e_lo <= e_span;
        }
        folded = __all_sync(0xFFFFFFFFu, ok);
        if (__builtin_expect(folded, 1)) {
#pragma unroll
            for (int s = 0; s < SUB; ++s) {
                if (!kFull && s >= static_cast<int>(steps)) {
                    v[s][0] = v[s][1] = v[s][2] = v[s][3] = 0.0;
                    continue;
                }
                step_lds_at<F>(st[s], pay, ex, o, s, false);
                st[s].decode_mul(st[s].smul(mul), v[s]);
#pragma unroll
                for (int k = 0; k < 4; ++k) v[s][k] = __dadd_rn(v[s][k], add);
            }
        }
    }
    if (!folded) {
#pragma unroll
        for (int s = 0; s < SUB; ++s) {
            if (!kFull && s >= static_cast<int>(steps)) {
                v[s][0] = v[s][1] = v[s][2] = v[s][3] = 0.0;
                continue;
            }
            if constexpr (FmtInfo<F>::frsz) {
                step_lds_at<F>(st[s], pay, ex, o, s, false);
                if (__builtin_expect(fast, 1)) st[s].decode_fast(v[s]);
                else st[s].decode(v[s]);
            } else {
                step_lds_at<F>(st[s], pay, ex, o, s);
                st[s].decode(v[s]);
            }
        }
    }
#pragma unroll 1
    for (int t = folded ? 1 : 0; t < intensity; ++t)
#pragma unroll
        for (int s = 0; s < SUB; ++s)
#pragma unroll
            for (int k = 0; k < 4; ++k) v[s][k] = __dadd_rn(__dmul_rn(v[s][k], mul), add);
    // n % 32 == 0: a thread's 4 rows are all inside or all past n
    double acc = 0.0;
    const bool all_in = kFull && row0 + (SUB - 1) * static_cast<uint64_t>(kStepRows) < n;
#pragma unroll
    for (int s = 0; s < SUB; ++s)
        if (all_in || ((kFull || s < static_cast<int>(steps)) && row0 + static_cast<uint64_t>(s) * kStepRows < n))
            acc = __dadd_rn(acc, __dadd_rn(__dadd_rn(v[s][0], v[s][1]), __dadd_rn(v[s][2], v[s][3])));
    return acc;
}

// The read sweep's common case, streamed step by step: an FRSZ2 stage whose
// rows are all below n, intensity 1, and every block exponent inside the
// folded-multiply range (one vote). No decoded-stage array and no per-step
// bounds: ~8 instructions per value instead of ~13. Otherwise the general
// stage_sweep.
template <int F>
__device__ __forceinline__ double stage_sweep1(const unsigned char* pay, const uint32_t* ex, const StageOff<F>& o,
                                               uint64_t row0, uint64_t n, double mul, double add, bool fold_ok,
                                               uint32_t e_lo, uint32_t e_span, uint32_t e_span1) {
    constexpr int SUB = Geo<F>::sub;
    Step<F> st[SUB];
    bool ok = fold_ok;
#pragma unroll
    for (int s = 0; s < SUB; ++s) {
        st[s].e = ex[32 * s];
        // implies the fast decode (e_lo > L - 2) and 2^52 * scale * mul finite
        ok &= st[s].e - e_lo <= e_span1;
    }
    if (__builtin_expect(!__all_sync(0xFFFFFFFFu, ok), 0))
        return stage_sweep<F, true>(pay, ex, o, SUB, row0, n, 1, mul, add, fold_ok, e_lo, e_span);
    double acc = 0.0;
#pragma unroll
    for (int s = 0; s < SUB; ++s) {
        step_lds_at<F>(st[s], pay, ex, o, s, false);
        double v[4];
        const double sm = st[s].smul(mul);
        st[s].decode_mul_fma(sm, __dmul_rn(sm, -0x1p52), v);
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = __dadd_rn(v[k], add);
        acc = __dadd_rn(acc, __dadd_rn(__dadd_rn(v[0], v[1]), __dadd_rn(v[2], v[3])));
    }
    return acc;
}

template <int F>
__global__ void __launch_bounds__(kThreads, split_min_blocks<F>())
read_sweep_kernel(BasisView B, uint64_t col, uint64_t n, int intensity, double mul, double add,
                  double* __restrict__ partials, unsigned* __restrict__ ticket, double* __restrict__ out) {
    constexpr int S = Geo<F>::stages;
    constexpr uint32_t PAY = Geo<F>::pay;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ double red[kWarps + 1];
    const Ring R = ring_setup<F>(smem);
    __syncthreads();
    uint64_t s0, s1;
    cta_steps(n, s0, s1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double acc = 0.0;
    if (warp == kConsumerWarps) {
        if (lane == 0) produce<F>(R, B, col, 1, s0, s1, false);
    } else {
        const StageOff<F> off;
        const SubTiles T = sub_tiles<F>(s0, s1);
        // Block exponents e for which scale(e) * mul is exact (normal):
        // scale = 2^(e - 1023 - (L - 2)), mul = m 2^(E - 1023) with m in
        // [1, 2) -> biased exponent of the product E + e - 1023 - (L - 2)
        // must lie in [1, 2046]. Only for a normal, nonzero mul.
        constexpr int L = FmtInfo<F>::L;
        const int E = static_cast<int>((__double_as_longlong(mul) >> 52) & 0x7FF);
        const int lo = max(1 - E + 1023 + (L - 2), L - 1);  // also the fast decode's e > L - 2
        const int hi = min(2046 - E + 1023 + (L - 2), 2046);
        const bool fold_ok = FmtInfo<F>::frsz && E >= 1 && E <= 2046 && hi >= lo;
        const uint32_t e_lo = static_cast<uint32_t>(lo);
        const uint32_t e_span = hi >= lo ? static_cast<uint32_t>(hi - lo) : 0u;
        // the streamed path's FMA decode also needs 2^52 * scale * mul finite
        const bool fold1 = fold_ok && hi - 52 >= lo;
        const uint32_t e_span1 = fold1 ? static_cast<uint32_t>(hi - 52 - lo) : 0u;
        // ring position as 32-bit counters (a 64-bit t % S costs ~20
        // instructions per stage)
        uint32_t stage = 0, phase = 0;
        for (uint64_t t = 0; t < T.count; ++t) {
            mbar_wait(R.full + stage, phase);
            const uint64_t sb = T.begin(t);
            const uint32_t steps = static_cast<uint32_t>(T.end(t) - sb);
            const unsigned char* pay = R.stages + stage * stage_bytes<F>();
            const uint32_t* ex = reinterpret_cast<const uint32_t*>(pay + Geo<F>::sub * PAY);
            const uint64_t row0 = sb * kStepRows + 4u * threadIdx.x;
            const bool full = steps == static_cast<uint32_t>(Geo<F>::sub);
            double a;
            bool streamed = false;
            if constexpr (FmtInfo<F>::frsz) {
                if (full && intensity == 1 && fold1 && (sb + Geo<F>::sub) * kStepRows <= n) {
                    a = stage_sweep1<F>(pay + off.pay, ex + off.ex, off, row0, n, mul, add, fold_ok, e_lo, e_span,
                                        e_span1);
                    streamed = true;
                }
            }
            if (streamed) {
            } else if (full)
                a = stage_sweep<F, true>(pay + off.pay, ex + off.ex, off, steps, row0, n, intensity, mul, add, fold_ok,
                                         e_lo, e_span);
            else
                a = stage_sweep<F, false>(pay + off.pay, ex + off.ex, off, steps, row0, n, intensity, mul, add,
                                          fold_ok, e_lo, e_span);
            acc = __dadd_rn(acc, a);
            __syncwarp();
            if (lane == 0) mbar_arrive(R.empty + stage);
            if (++stage == S) {
                stage = 0;
                phase ^= 1u;
            }
        }
    }
    acc = warp_sum(acc);
    if (lane == 0) red[warp] = acc;  // the producer warp contributes +0.0
    __syncthreads();
    block_finalize(red, kWarps + 1, 1, partials, ticket, out);
}

// Dynamic tile scheduling for the split CGS kernels (measured on B200:
// update at n = 2^26, k = 100 0.85 -> 1.03 of the HBM peak).
template <int F> struct DotLaunch {
    static void run(const BasisView& B, uint64_t first, uint32_t cols, const double* w, int wn,
                    int reduction, double* h, Workspace* ws, cudaStream_t st, const GateArg& gate, bool coop) {
        const uint32_t ncol = cols + (wn ? 1 : 0);
        if (ncol == 0) return;
        if (reduction == CBGX_REDUCE_REFERENCE) {
            const uint32_t threads = ncol;
            CBGX_K(serial_dot_kernel<F><<<(threads + 63) / 64, 64, 0, st>>>(B, first, cols, w, wn, h, gate));
            return;
        }
        if (coop) {
            // reduction scratch: kWarps x ncol per tile, kThreads for the
            // final column sums
            const size_t smem = ring_smem<F>(std::max<size_t>(static_cast<size_t>(kWarps) * ncol, kThreads)) + 64;
            allow_smem(cgs_dot_dyn_kernel<F>);
            const int grid = ring_grid(cgs_dot_dyn_kernel<F>, B.n, smem);
            const uint64_t nsteps = (B.n + kStepRows - 1) / kStepRows;
            const uint64_t ntiles = (nsteps + Geo<F>::sub - 1) / Geo<F>::sub;
            double* part = ws->get_partials(static_cast<size_t>(ntiles) * ncol);
            unsigned* ctr = ws->get_counter();
            void* args[] = {const_cast<BasisView*>(&B), &first, &cols, &w, &wn, &part, &ctr, &h,
                            const_cast<GateArg*>(&gate)};
            note_launch();
            CBGX_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(cgs_dot_dyn_kernel<F>), dim3(grid),
                                                  dim3(kThreads), args, smem, st));
            return;
        }
        const size_t smem = ring_smem<F>(static_cast<size_t>(kWarps) * ncol);
        allow_smem(cgs_dot_kernel<F>);
        const int grid = ring_grid(cgs_dot_kernel<F>, B.n, smem);
        double* partials = ws->get_partials(static_cast<size_t>(grid) * ncol);
        CBGX_K(cgs_dot_kernel<F><<<grid, kThreads, smem, st>>>(B, first, cols, w, wn, partials,
                                                        ws->get_counter(), h, gate));
    }
};

template <int F> struct UpdateLaunch {
    static void run(const BasisView& B, uint64_t first, uint32_t cols, const double* h, double sign,
                    double* w, double* norm, int reduction, Workspace* ws, cudaStream_t st,
                    const GateArg& gate) {
        const bool fused_norm = norm && reduction == CBGX_REDUCE_TREE;
        if (cols > 0 || fused_norm) {
            const size_t smem = ring_smem<F>(cols + kWarps) + 64 + cols;
            allow_smem(cgs_update_dyn_kernel<F>);
            const int grid = ring_grid(cgs_update_dyn_kernel<F>, B.n, smem);
            const uint64_t nsteps = (B.n + kStepRows - 1) / kStepRows;
            double* tn = fused_norm ? ws->get_partials((nsteps + Geo<F>::sub - 1) / Geo<F>::sub) : nullptr;
            CBGX_K(cgs_update_dyn_kernel<F><<<grid, kThreads, smem, st>>>(B, first, cols, h, sign, w, fused_norm, tn,
                                                                   ws->get_counter(), norm, gate));
            if (norm && !fused_norm) launch_dot(w, w, B.n, CBGX_REDUCE_REFERENCE, norm, ws, st, gate);
            return;
        }
        if (cols > 0 || fused_norm) {
            const size_t smem = ring_smem<F>(cols + kWarps) + cols;
            allow_smem(cgs_update_kernel<F>);
            const int grid = ring_grid(cgs_update_kernel<F>, B.n, smem);
            double* partials = fused_norm ? ws->get_partials(grid) : nullptr;
            CBGX_K(cgs_update_kernel<F><<<grid, kThreads, smem, st>>>(B, first, cols, h, sign, w, fused_norm,
                                                               partials, ws->get_counter(), norm, gate));
        }
        if (norm && !fused_norm) launch_dot(w, w, B.n, CBGX_REDUCE_REFERENCE, norm, ws, st, gate);
    }
};

template <int F> struct WriteLaunch {
    static void run(const cbgx_basis& V, uint64_t j, const double* x, const ScaleArg& scale,
                    double* v_out, uint64_t* bad, cudaStream_t st) {
        unsigned char* col = static_cast<unsigned char*>(V.d_data) + j * V.col_stride_bytes;
        if constexpr (FmtInfo<F>::frsz) {
            // the column's exponent range for the vote-free fast decode,
            // folded by the compress kernel itself
            uint32_t* er = V.d_erange ? V.d_erange + 2 * j : nullptr;
            if (er) CBGX_CUDA(cudaMemsetAsync(er, 0, 2 * sizeof(uint32_t), st));
            launch_compress(x, V.n, V.n_pad / 32, 32, FmtInfo<F>::L,
                            V.d_exp + j * V.exp_col_stride, reinterpret_cast<uint32_t*>(col),
                            scale, v_out, bad, st, er);
        } else {
            const uint64_t blocks = std::min<uint64_t>((V.n_pad + 255) / 256, static_cast<uint64_t>(sm_count()) * 16);
            CBGX_K(write_plain_kernel<F><<<static_cast<int>(std::max<uint64_t>(blocks, 1)), 256, 0, st>>>(
                col, x, V.n, V.n_pad, scale, v_out));
        }
    }
};

template <int F> struct SweepLaunch {
    static void run(const BasisView& B, uint64_t col, uint64_t n, int intensity, double mul, double add,
                    double* out, Workspace* ws, cudaStream_t st) {
        const size_t smem = ring_smem<F>(0) + 64;
        allow_smem(read_sweep_kernel<F>);
        const int grid = ring_grid(read_sweep_kernel<F>, n, smem);
        CBGX_K(read_sweep_kernel<F><<<grid, kThreads, smem, st>>>(B, col, n, intensity, mul, add,
                                                                 ws->get_partials(grid), ws->get_counter(), out));
    }
};
template <int F> struct ReadLaunch {
    static void run(const BasisView& B, uint64_t j, uint64_t first, uint64_t count, double* out,
                    cudaStream_t st) {
        const uint64_t blocks = std::min<uint64_t>((count + 255) / 256, static_cast<uint64_t>(sm_count()) * 16);
        CBGX_K(read_kernel<F><<<static_cast<int>(std::max<uint64_t>(blocks, 1)), 256, 0, st>>>(B, j, first, count, out));
    }
};

// ============================================================================
// Fused single-GPU Arnoldi orthogonalisation (persistent, co-resident grid).
//
// One launch replaces dot -> update -> [gated dot -> update] -> scaled write
// of the next basis column (gmres.cpp:211-234 minus the host Givens). One CTA
// per SM (16 consumer warps + 1 producer warp) owns a fixed, contiguous row
// range for the whole launch, so w stays in registers across all passes;
// passes are separated by grid all-reductions among the consumer warps while
// the producer warp keeps streaming the next pass's columns through the
// shared-memory ring (the basis does not depend on the reduction). Dot passes
// run last-to-first and update passes first-to-last, so each pass starts on
// the columns the previous one left in L2.
//
// Rows are split over the CTAs in 128-row units (16-B aligned segments for
// every format), so CTAs differ by at most one unit (<1% at 128^3) and every
// grid reduction waits on a balanced grid. Geometry (build-time, measured on
// B200 with scripts/ab_fused.sh): FUSED_CTAS CTAs per SM of FUSED_WARPS
// consumer warps, each thread holding 4 rows x FUSED_STEPS steps of w in
// registers. 2 x 12 warps x 5 steps (1536-row steps) beat 2 x 8 x 8 (7.94 vs
// 8.19 ms per 128^3 solve) and 2 x 10 x 6: more warps hide the decode and
// shared-memory latency of the column passes. Eligible when every
// CTA's rows fit (n <= 4 * 32 * FUSED_WARPS * FUSED_STEPS * CTAs).
#ifndef FUSED_WARPS
#define FUSED_WARPS 12
#endif
#ifndef FUSED_STEPS
#define FUSED_STEPS 5
#endif
constexpr int kFusedMaxSteps = FUSED_STEPS;
constexpr int kFCtasPerSM = FUSED_CTAS_PER_SM;
constexpr int kFWarps = FUSED_WARPS;            // consumer warps
constexpr int kFConsumers = kFWarps * 32;
constexpr int kFThreads = kFConsumers + 32;     // + producer warp
constexpr uint32_t kFStepRows = 4 * kFConsumers;
constexpr uint32_t kUnitRows = 128;
static_assert(kColTail >= kFStepRows, "column tail must cover one fused step");
static_assert(kFStepRows % kUnitRows == 0, "steps are whole 128-row units");

// payload / exponent bytes per step and per 128-row unit
template <int F> struct FBytes {
    static constexpr uint32_t pay = Geo<F>::pay * kFStepRows / 1024, ex = Geo<F>::ex * kFStepRows / 1024;
    static constexpr uint32_t upay = Geo<F>::pay / 8, uex = Geo<F>::ex / 8;
};

// Ring stage = one column's segment of `chunk` steps (~32 KB), `stages` deep
// (~100 KB of shared memory per CTA at two CTAs per SM).
#ifndef FUSED_CHUNK_BYTES
#define FUSED_CHUNK_BYTES 32768
#endif
#ifndef FUSED_RING_BYTES
#define FUSED_RING_BYTES 100000
#endif

template <int F> struct FGeo {
    static constexpr int chunk_raw = static_cast<int>(FUSED_CHUNK_BYTES / (FBytes<F>::pay + FBytes<F>::ex));
    static constexpr int chunk = chunk_raw < 1 ? 1 : (chunk_raw > kFusedMaxSteps ? kFusedMaxSteps : chunk_raw);
    static constexpr uint32_t basis_bytes = chunk * (FBytes<F>::pay + FBytes<F>::ex) + 16;
    static constexpr uint32_t stage_bytes = basis_bytes / 16 * 16 + 16;
    static constexpr int stages_raw = static_cast<int>((kFCtasPerSM == 1 ? 170000 : FUSED_RING_BYTES) / (stage_bytes + 16));
    static constexpr int stages = stages_raw < 2 ? 2 : stages_raw;
};

template <int F>
__host__ __device__ constexpr uint32_t fstage_bytes() {
    return FGeo<F>::stage_bytes;
}

struct FusedArgs {
    BasisView B;
    uint32_t cols;             // columns 0..cols-1 orthogonalise w; column `cols` is written
    unsigned char* out_pay;    // column `cols` payload / values
    uint32_t* out_exp;         // column `cols` exponents (FRSZ2)
    uint32_t* out_erange;      // column `cols` exponent range (nullptr: not kept)
    unsigned long long* fx;      // this launch's fixed-point accumulators: 2 regions + flag
    unsigned long long* fx_next; // the next launch's set: zeroed here (CTA 0)
    uint32_t fx_region;          // words per region (fx_at(max_cols + 2))
    const double* w;           // SpMV output (rows [0, n))
    double* v_out;             // next SpMV input
    double* slot;              // [hn1, hn2, omega2, h[0..m], u[0..m]]; omega2 set by the SpMV
    const double* om_parts;    // the SpMV's per-CTA omega^2 partials (nullptr: omega2 from slot[2])
    uint32_t om_count;
    uint32_t u_off;            // index of u in slot
    double eta;
    double* partials;          // kRegions regions of (cols + 1) x gs doubles (value-major)
    uint32_t gs;               // gridDim.x rounded up to even
    uint32_t rot;              // diagnostic rotation of the row ranges (cbgx_debug_fused_rotation)
    unsigned* bar;             // this launch's arrival counter (zero at launch)
    unsigned* bar_next;        // the next launch's counter: zeroed here (CTA 0)
    unsigned* gate_hist;       // previous launch's gate: 0 open (speculate), 1 closed
    double* host_slot;         // optional mapped pinned copy of the slot (read by the host)
    unsigned long long* trace; // optional: CTA 0 phase timestamps (debug)
};

// Partial regions, one per grid reduction of a launch, so a CTA that runs
// ahead never overwrites partials a slower CTA is still reading.
constexpr int kRegions = 4;

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// phase timestamps of every CTA: trace[kTraceBase + phase * 1024 + cta]
constexpr int kTraceBase = 32, kTracePhases = 24;
// Compiled in only for diagnostic builds (CBGX_NVFLAGS_EXTRA=-DCBGX_FUSED_TRACE=1,
// scripts/fused_phases.py): the timer reads are not free.
#ifndef CBGX_FUSED_TRACE
#define CBGX_FUSED_TRACE 0
#endif
#if CBGX_FUSED_TRACE
#define FTRACE(i) do { if (a.trace && threadIdx.x == 0) a.trace[kTraceBase + (i) * 1024 + blockIdx.x] = global_ns(); } while (0)
#else
#define FTRACE(i) do { } while (0)
#endif

__device__ __forceinline__ void consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(kFConsumers) : "memory");
}

__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}


// Row shares of the fused grid: equal shares of 128-row units. (Weighted
// shares -- fewer rows for the second CTA of an SM, which streams ~10%
// slower -- measured 0.5-0.7% slower: the two CTAs share the SM's
// throughput.)
__host__ __device__ __forceinline__ void fused_unit_range(uint64_t units, uint64_t G, uint64_t slot, uint64_t& u0,
                                                          uint64_t& u1) {
    u0 = units * slot / G;
    u1 = units * (slot + 1) / G;
}

// This CTA's rows: [r0, r1) in 128-row units, weighted over the grid.
__device__ __forceinline__ void fused_rows(uint64_t n, uint32_t rot, uint64_t& r0, uint64_t& r1) {
    const uint64_t units = (n + kUnitRows - 1) / kUnitRows;
    const uint64_t slot = (blockIdx.x + rot) % gridDim.x;  // rot: diagnostic only (0 in production)
    uint64_t u0, u1;
    fused_unit_range(units, gridDim.x, slot, u0, u1);
    r0 = u0 * kUnitRows;
    r1 = u1 * kUnitRows;
}

// ------------------------------------------- fixed-point grid reductions
// The fused kernel's two grid reductions (h; u and hn1) are also accumulated
// as exact fixed-point sums: a CTA partial p becomes the integer
// X = p * 2^(kFxF - e) (truncated below the resolution 2^(e - kFxF), e a
// per-value scale exponent fixed before the launch from omega), split into
// three signed 42-bit chunks, each added with one red.global.add.u64 into its
// own 64-bit word (296 chunks < 2^51: no word overflows). Integer addition is
// associative, so the sums are exact, deterministic and independent of the
// arrival order; after the barrier every CTA reads 3 words per value (ONE
// load batch instead of the value-major table's 2-19, by k) and rounds the
// 126-bit integer to double once. A partial >= 2^(e+6), a non-finite
// partial, a non-positive or non-finite omega^2, or an hn1 too small for 50
// significant bits sends every CTA (uniformly: the same flag and sums) to
// the value-major table path, which is always written too.
constexpr int kFxF = 110;
constexpr unsigned long long kFxM = (1ull << 42) - 1;

__device__ __forceinline__ bool fx_split(double p, int e, long long c[3]) {
    const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(p));
    c[0] = c[1] = c[2] = 0;
    if (p == 0.0) return true;
    int ex = static_cast<int>((bits >> 52) & 0x7FF);
    if (ex == 0x7FF) return false;
    unsigned long long m = bits & ((1ull << 52) - 1);
    if (ex) m |= 1ull << 52;
    else ex = 1;
    const int sh = ex - 1075 + kFxF - e;  // X = m * 2^sh, X < 2^116 for sh <= 63
    if (sh > 63) return false;
    unsigned long long lo = 0, hi = 0;
    if (sh >= 0) {
        lo = m << sh;
        hi = sh ? m >> (64 - sh) : 0ull;
    } else if (sh > -64) {
        lo = m >> (-sh);
    }
    const long long q0 = static_cast<long long>(lo & kFxM), q1 = static_cast<long long>(((lo >> 42) | (hi << 22)) & kFxM),
                    q2 = static_cast<long long>(hi >> 20);
    const bool neg = bits >> 63;
    c[0] = neg ? -q0 : q0;
    c[1] = neg ? -q1 : q1;
    c[2] = neg ? -q2 : q2;
    return true;
}

// w0 + w1 2^42 + w2 2^84, rounded to nearest-even, times 2^(e - kFxF).
// Sets *small when |X| < 2^60 (fewer than 50 significant bits above the
// truncation noise of 296 partials).
__device__ __forceinline__ double fx_join(long long w0, long long w1, long long w2, int e, bool* small) {
    const __int128 X = static_cast<__int128>(w0) + (static_cast<__int128>(w1) << 42) + (static_cast<__int128>(w2) << 84);
    if (X == 0) {
        *small = true;
        return 0.0;
    }
    const bool neg = X < 0;
    const unsigned __int128 M = neg ? -static_cast<unsigned __int128>(X) : static_cast<unsigned __int128>(X);
    const unsigned long long hi = static_cast<unsigned long long>(M >> 64), lo = static_cast<unsigned long long>(M);
    const int top = hi ? 127 - __clzll(static_cast<long long>(hi)) : 63 - __clzll(static_cast<long long>(lo));
    *small = top < 60;
    double v;
    if (top <= 52) {
        v = static_cast<double>(lo);  // exact
        v = ldexp(v, e - kFxF);
    } else {
        const int shift = top - 52;
        unsigned long long mant = static_cast<unsigned long long>(M >> shift);
        const unsigned __int128 rem = M & ((static_cast<unsigned __int128>(1) << shift) - 1);
        const unsigned __int128 half = static_cast<unsigned __int128>(1) << (shift - 1);
        if (rem > half || (rem == half && (mant & 1ull))) ++mant;  // 2^53 stays exact
        v = ldexp(static_cast<double>(mant), shift + e - kFxF);
    }
    return neg ? -v : v;
}

// Accumulator words kFxStride apart (16: one 128-byte line per word): every
// CTA adds into the same words, and same-line atomics serialise in their L2
// slice -- spread over lines, the adds proceed in parallel (ortho phase
// 4.877 -> 4.853 ms per solve at 128^3, four A/B runs each).
#ifndef FX_STRIDE
#define FX_STRIDE 16
#endif
constexpr uint32_t kFxStride = FX_STRIDE;
// value j's three chunk words start at acc + fx_at(j)
__host__ __device__ constexpr uint32_t fx_at(uint32_t j) { return 3u * kFxStride * j; }

__device__ __forceinline__ void fx_red(unsigned long long* w, const long long c[3]) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
        asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(w + i * kFxStride),
                     "l"(static_cast<unsigned long long>(c[i]))
                     : "memory");
}

// Grid all-reduce among the consumer warps of all (co-resident) CTAs, one
// barrier hop. Partials are value-major: value k of CTA c at
// region[k * gs + c]. Thread 0 arrives with a release add on the launch's
// monotonic counter and waits (acquire) until all CTAs of barrier number
// `seq` have arrived; then EVERY CTA sums the partials itself in one fixed
// order -- R = 2^i <= 32 adjacent lanes per value, lane g adding the
// 16-B pairs g, g+R, ... (loads batched so they are all in flight), then a
// butterfly over the R lanes -- so all CTAs hold bit-identical results and
// nobody waits for another CTA to publish them. count <= kFConsumers.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned seq, unsigned long long* trace) {
    consumer_sync();
    if (threadIdx.x == 0) {
        if (CBGX_FUSED_TRACE && trace && blockIdx.x == 0) trace[11 + 2 * seq] = global_ns();
        red_release_add(bar, 1u);
        wait_count(bar, (seq + 1) * gridDim.x);
        if (CBGX_FUSED_TRACE && trace && blockIdx.x == 0) trace[12 + 2 * seq] = global_ns();
    }
    consumer_sync();
}

// The value-major table reduction (after the barrier).
__device__ __forceinline__ void table_reduce(const double* region, uint32_t gs, uint32_t count, double* out_smem) {
    uint32_t R = 32;
    while (R > 1 && R * count > static_cast<uint32_t>(kFConsumers)) R >>= 1;
    const uint32_t t = threadIdx.x, k = t / R, g = t % R;
    const unsigned G = gridDim.x, pairs = (G + 1) / 2;
    double v = 0.0;
    if (k < count) {
        const double2* base = reinterpret_cast<const double2*>(region + static_cast<uint64_t>(k) * gs);
        constexpr int kB = 4;
        for (unsigned p0 = g; p0 < pairs; p0 += R * kB) {
            double2 x[kB];
#pragma unroll
            for (int i = 0; i < kB; ++i) {
                const unsigned p = p0 + R * i;
                x[i] = p < pairs ? __ldcg(base + p) : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int i = 0; i < kB; ++i) {
                const unsigned p = p0 + R * i;
                if (p < pairs) {
                    v = __dadd_rn(v, x[i].x);
                    if (2 * p + 1 < G) v = __dadd_rn(v, x[i].y);
                }
            }
        }
    }
    for (uint32_t off = R >> 1; off >= 1; off >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xFFFFFFFFu, v, off));
    if (g == 0 && k < count) out_smem[k] = v;
    consumer_sync();
}

__device__ __forceinline__ void grid_allreduce(unsigned* bar, unsigned seq, const double* region, uint32_t gs,
                                               uint32_t count, double* out_smem,
                                               unsigned long long* trace = nullptr) {
    grid_barrier(bar, seq, trace);
    table_reduce(region, gs, count, out_smem);
}

// Fixed-point variant: `acc` holds the count x 3 accumulator words, `flag`
// the overflow word (bit `fbit`), values k < count use scale exponent e,
// value `nlast` (if < count) e_last and must keep 50 significant bits.
// fx_ok == false (scales unusable this launch): table path.
__device__ __forceinline__ void grid_allreduce_fx(unsigned* bar, unsigned seq, const double* region, uint32_t gs,
                                                  uint32_t count, double* out_smem, const unsigned long long* acc,
                                                  const unsigned long long* flag, unsigned fbit, bool fx_ok, int e,
                                                  uint32_t nlast, int e_last, volatile int* s_flag,
                                                  unsigned long long* trace = nullptr) {
    grid_barrier(bar, seq, trace);
    if (fx_ok) {
        const uint32_t t = threadIdx.x;
        long long w0 = 0, w1 = 0, w2 = 0;
        unsigned long long f = 0;
        if (t < count) {
            w0 = static_cast<long long>(__ldcg(acc + fx_at(t)));
            w1 = static_cast<long long>(__ldcg(acc + fx_at(t) + kFxStride));
            w2 = static_cast<long long>(__ldcg(acc + fx_at(t) + 2 * kFxStride));
        }
        if (t == count) f = __ldcg(flag);
        bool small = false;
        double v = 0.0;
        if (t < count) v = fx_join(w0, w1, w2, t == nlast ? e_last : e, &small);
        if (t == count) *s_flag = (f >> fbit) & 1ull ? 1 : 0;
        consumer_sync();
        if (t == nlast && small) *s_flag = 1;
        consumer_sync();
        if (*s_flag == 0) {
            if (t < count) out_smem[t] = v;
            consumer_sync();
            return;
        }
    }
    table_reduce(region, gs, count, out_smem);
}

// CTA sum of one value per consumer thread (warp butterflies, then the warp
// sums in order); returned in every thread.
__device__ __forceinline__ double cta_wnorm_sum(double v, double* nred) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    v = warp_sum(v);
    consumer_sync();  // nred may still be read by a previous reduction
    if (lane == 0) nred[warp] = v;
    consumer_sync();
    double s = nred[0];
    for (int w = 1; w < kFWarps; ++w) s = __dadd_rn(s, nred[w]);
    return s;
}

// This CTA's <w, w> over its register-resident rows (fixed order); the
// value is returned in every thread.
__device__ __forceinline__ double cta_wnorm2(double wv[][4], double* nred) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double nacc = 0.0;
#pragma unroll
    for (int s = 0; s < kFusedMaxSteps; ++s)
#pragma unroll
        for (int k = 0; k < 4; ++k) nacc = fma(wv[s][k], wv[s][k], nacc);
    nacc = warp_sum(nacc);
    if (lane == 0) nred[warp] = nacc;
    consumer_sync();
    double s = nred[0];
    for (int w = 1; w < kFWarps; ++w) s = __dadd_rn(s, nred[w]);
    return s;
}

template <int F>
__device__ __forceinline__ void fused_write(const FusedArgs& a, uint64_t r0, uint64_t r1, uint32_t steps,
                                            double wv[][4], double scale, uint32_t* scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t e_inv = 0, e_max = 0;  // the column's exponent range (erange_fold)
#pragma unroll
    for (int s = 0; s < kFusedMaxSteps; ++s) {
        if (s >= static_cast<int>(steps)) break;
        const uint64_t r = r0 + s * kFStepRows + 4u * threadIdx.x;
        if (r >= r1) continue;  // warp-uniform: r1 is a multiple of 128
        double v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = r + k < a.B.n ? __dmul_rn(wv[s][k], scale) : 0.0;
        if (r + 3 < a.B.n) {
            store4(a.v_out + r, v);
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (r + k < a.B.n) a.v_out[r + k] = v[k];
        }
        if constexpr (FmtInfo<F>::frsz) {
            constexpr int L = FmtInfo<F>::L;
            uint32_t e = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) e = max(e, exp_field(v[k]));
            e = max(e, __shfl_xor_sync(0xFFFFFFFFu, e, 1));
            e = max(e, __shfl_xor_sync(0xFFFFFFFFu, e, 2));
            e = max(e, __shfl_xor_sync(0xFFFFFFFFu, e, 4));
            uint32_t c[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) c[k] = encode32<L>(v[k], e);
            if ((lane & 7) == 0) a.out_exp[r / 32] = e;
            erange_fold(e, e_inv, e_max);
            if constexpr (L == 32) {
                reinterpret_cast<uint4*>(a.out_pay)[r / 4] = make_uint4(c[0], c[1], c[2], c[3]);
            } else if constexpr (L == 16) {
                reinterpret_cast<uint2*>(a.out_pay)[r / 4] = make_uint2(c[0] | (c[1] << 16), c[2] | (c[3] << 16));
            } else {
                // 4 blocks (84 words) per warp per step, assembled in smem
                uint32_t* wbuf = scratch + warp * 84;
                for (int i = lane; i < 84; i += 32) wbuf[i] = 0u;
                __syncwarp();
                const uint32_t bit0 = (lane >> 3) * 672u + (lane & 7) * 84u;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t b = bit0 + 21u * k, q = b >> 5, sh = b & 31u;
                    atomicOr(wbuf + q, c[k] << sh);
                    if (sh > 11) atomicOr(wbuf + q + 1, c[k] >> (32 - sh));
                }
                __syncwarp();
                uint32_t* dst = reinterpret_cast<uint32_t*>(a.out_pay) + (r - 4u * lane) / 32 * 21;
                for (int i = lane; i < 84; i += 32) dst[i] = wbuf[i];
                __syncwarp();
            }
        } else if constexpr (F == kF64) {
            reinterpret_cast<double2*>(a.out_pay)[r / 2] = make_double2(v[0], v[1]);
            reinterpret_cast<double2*>(a.out_pay)[r / 2 + 1] = make_double2(v[2], v[3]);
        } else if constexpr (F == kF32) {
            reinterpret_cast<float4*>(a.out_pay)[r / 4] =
                make_float4(__double2float_rn(v[0]), __double2float_rn(v[1]), __double2float_rn(v[2]), __double2float_rn(v[3]));
        } else {
            reinterpret_cast<uint2*>(a.out_pay)[r / 4] =
                make_uint2(double_to_half_bits(v[0]) | (static_cast<uint32_t>(double_to_half_bits(v[1])) << 16),
                           double_to_half_bits(v[2]) | (static_cast<uint32_t>(double_to_half_bits(v[3])) << 16));
        }
    }
    if constexpr (FmtInfo<F>::frsz) {
        if (a.out_erange) {
            // CTA maximum of the warps' ranges, one atomic pair per CTA
            e_inv = __reduce_max_sync(0xFFFFFFFFu, e_inv);
            e_max = __reduce_max_sync(0xFFFFFFFFu, e_max);
            consumer_sync();  // scratch is free (the l=21 assembly is done)
            if (lane == 0) {
                scratch[2 * warp] = e_inv;
                scratch[2 * warp + 1] = e_max;
            }
            consumer_sync();
            if (threadIdx.x == 0) {
                uint32_t ci = 0, cm = 0;
                for (int q = 0; q < kFWarps; ++q) {
                    ci = max(ci, scratch[2 * q]);
                    cm = max(cm, scratch[2 * q + 1]);
                }
                atomicMax(a.out_erange, ci);
                atomicMax(a.out_erange + 1, cm);
            }
        }
    }
}

// Significant bits of a stored basis value (|V^T V - I| <~ 2^-p for the
// decoded columns): FRSZ2-l keeps l - 2 magnitude bits below the block
// maximum; f16 10, f32 22; f64 bounded by the orthogonality of the computed
// basis, taken as 2^-40.
template <int F>
constexpr int kOrthBits = FmtInfo<F>::frsz ? FmtInfo<F>::L - 2 : (F == kF64 ? 40 : (F == kF32 ? 22 : 10));
__host__ __device__ constexpr double pow2(int e) {
    double r = 1.0;
    for (; e > 0; --e) r *= 2.0;
    for (; e < 0; ++e) r *= 0.5;
    return r;
}

// One column's chunks of a pass (dot: partial sums into acc/acc2; update:
// w -= h_j v_j). kFast: the column's exponent range (cbgx_basis.d_erange)
// proves every block decodes exactly on the fast path -- no per-step test;
// otherwise (a rare column, or no ranges kept) every block takes the exact
// decoder, again without a per-step test (measured on B200: the per-step
// warp vote and the two inlined decode paths cost 8% of the fused launch).
template <int F, bool kDot, bool kFull, bool kFast>
__device__ __forceinline__ void fused_column(double hj, int he, uint32_t steps, uint32_t nch, unsigned char* stages,
                                             uint64_t* full, uint64_t* empty, uint32_t& it, double wv[][4],
                                             double& acc, double& acc2) {
    constexpr int S = FGeo<F>::stages;
    constexpr uint32_t PAY = FBytes<F>::pay, SB = fstage_bytes<F>();
    constexpr int kChunkSteps = FGeo<F>::chunk, kChunks = (kFusedMaxSteps + kChunkSteps - 1) / kChunkSteps;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int ch = 0; ch < kChunks; ++ch) {
        if (!kFull && ch >= static_cast<int>(nch)) break;
        const int stage = it % S;
        mbar_wait(full + stage, (it / S) & 1);
        const unsigned char* pay = stages + stage * SB;
        const uint32_t* ex = reinterpret_cast<const uint32_t*>(pay + kChunkSteps * PAY);
        const StageOff<F> off;
        const unsigned char* pay_t = pay + off.pay;
        const uint32_t* ex_t = ex + off.ex;
#pragma unroll
        for (int s = 0; s < kChunkSteps; ++s) {
            const int gs = ch * kChunkSteps + s;
            // whole steps (warp-uniform): rows past the CTA's range hold
            // valid FRSZ2 data of the next range and w = 0 there
            if (gs < kFusedMaxSteps && (kFull || static_cast<uint32_t>(gs) < steps)) {
                Step<F> st;
                step_lds_at<F, FBytes<F>::pay, FBytes<F>::ex / 4>(st, pay_t, ex_t, off, s);
                if constexpr (kDot) {
                    double d;
                    if constexpr (!FmtInfo<F>::frsz) d = st.dot(wv[gs]);
                    else if constexpr (kFast) d = st.dot_fast(wv[gs]);
                    else d = st.dot_exact(wv[gs]);
                    if (s & 1) acc2 = __dadd_rn(acc2, d);
                    else acc = __dadd_rn(acc, d);
                } else {
                    if constexpr (!FmtInfo<F>::frsz) st.update(hj, he, wv[gs]);
                    else if constexpr (kFast) st.update_fast(hj, he, wv[gs]);
                    else st.update_exact(hj, wv[gs]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + stage);
        ++it;
    }
}

// One column pass over the CTA's rows: dot (partials into red[warp][j]) or
// update (w -= h_j v_j) for columns in the given order. `lim` = number of
// the CTA's rows; a thread's 4 rows are skipped past it (its w stays 0).
// kFull: the CTA holds kFusedMaxSteps steps (every CTA but the last few),
// no per-step bounds checks. Per ring stage the shared-memory step loads
// use a per-thread stage base (StageOff), so the per-step offsets are
// immediates. ers: the columns' exponent ranges in shared memory (nullptr:
// the per-step vote decides the decode path).
template <int F, bool kDot, bool kFull>
__device__ __forceinline__ void fused_pass(uint32_t cols, uint32_t lim, uint32_t steps, uint32_t nch, unsigned char* stages,
                                           uint64_t* full, uint64_t* empty, uint32_t& it, double wv[][4],
                                           double* red, const double* hsm, const uint32_t* ers) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (uint32_t jj = 0; jj < cols; ++jj) {
        const uint32_t j = kDot ? cols - 1 - jj : jj;
        const double hj = kDot ? 0.0 : hsm[j];
        const int he = static_cast<int>(exp_field(hj));
        double acc = 0.0, acc2 = 0.0;
        bool fast = false;
        if constexpr (FmtInfo<F>::frsz) {
            if (ers) {
                constexpr int L = FmtInfo<F>::L;
                fast = kDot ? col_dot_fast<L>(ers[2 * j], ers[2 * j + 1])
                            : col_upd_fast<L>(ers[2 * j], ers[2 * j + 1], hj, he);
            }
        }
        // the exact variant without the full-steps specialisation (rare
        // path; less code next to the hot loops)
        if (FmtInfo<F>::frsz && __builtin_expect(fast, 1))
            fused_column<F, kDot, kFull, FmtInfo<F>::frsz>(hj, he, steps, nch, stages, full, empty, it, wv, acc, acc2);
        else
            fused_column<F, kDot, kFull && !FmtInfo<F>::frsz, false>(hj, he, steps, nch, stages, full, empty, it, wv,
                                                                     acc, acc2);
        if constexpr (kDot) {
            acc = warp_sum(__dadd_rn(acc, acc2));
            if (lane == 0) red[warp * cols + j] = acc;
        }
    }
    if constexpr (!kDot) {
        // the update also touched the rows past the CTA's range: w = 0 there
#pragma unroll
        for (int s = 0; s < kFusedMaxSteps; ++s)
            if (static_cast<uint32_t>(s) * kFStepRows + 4u * threadIdx.x >= lim)
                wv[s][0] = wv[s][1] = wv[s][2] = wv[s][3] = 0.0;
    }
}

template <int F, bool kDot>
__device__ __forceinline__ void fused_pass_any(uint32_t cols, uint32_t lim, uint32_t steps, uint32_t nch,
                                               unsigned char* stages, uint64_t* full, uint64_t* empty, uint32_t& it,
                                               double wv[][4], double* red, const double* hsm, const uint32_t* ers) {
    if (steps == static_cast<uint32_t>(kFusedMaxSteps))
        fused_pass<F, kDot, true>(cols, lim, steps, nch, stages, full, empty, it, wv, red, hsm, ers);
    else
        fused_pass<F, kDot, false>(cols, lim, steps, nch, stages, full, empty, it, wv, red, hsm, ers);
}

// This CTA's dot-pass partials (red[warp][j] summed over warps in order)
// into the value-major region: region[j * gs + cta].
__device__ __forceinline__ void dot_partials_out(const double* red, uint32_t cols, double* region, uint32_t gs,
                                                 unsigned long long* acc = nullptr, unsigned long long* flag = nullptr,
                                                 unsigned fbit = 0, int e = 0) {
    consumer_sync();
    for (uint32_t j = threadIdx.x; j < cols; j += kFConsumers) {
        double s = red[j];
        for (int w = 1; w < kFWarps; ++w) s = __dadd_rn(s, red[w * cols + j]);
        region[static_cast<uint64_t>(j) * gs + blockIdx.x] = s;
        if (acc) {
            long long c[3];
            if (fx_split(s, e, c)) fx_red(acc + fx_at(j), c);
            else atomicOr(flag, 1ull << fbit);
        }
    }
}

// Pass schedule (gmres.cpp:36-71, CGS with the reference's gated second
// pass), 3 grid reductions when the second pass runs, 2 when it does not:
//   dot1 -> R0[h] -> update1 -> (speculative dot2) -> R1[u.., hn1] -> gate
//   -> update2 -> R2[hn2] -> scaled write of column `cols`.
// The second dot pass needs only the CTA's own rows of the updated w, so it
// runs before the gate is known when the previous launch's gate was open
// (re-orthogonalisation tends to persist), saving one grid reduction; if
// the gate turns out closed its coefficients are simply not used. With the
// previous gate closed the dot2 pass waits for the gate (R1 = [hn1] only,
// then R2'[u] in region 2).
template <int F>
__global__ void __launch_bounds__(kFThreads, kFCtasPerSM) arnoldi_fused_kernel(FusedArgs a) {
    constexpr int S = FGeo<F>::stages;
    constexpr uint32_t PAY = FBytes<F>::pay, UPAY = FBytes<F>::upay, UEX = FBytes<F>::uex, SB = fstage_bytes<F>();
    extern __shared__ __align__(128) unsigned char smem[];
    const uint32_t cols = a.cols;
    unsigned char* stages = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * SB);
    uint64_t* empty = full + S;
    double* red = reinterpret_cast<double*>(empty + S);        // [kFWarps][cols]
    double* hsm = red + kFWarps * (cols + 1);                   // reduced h / u (+ hn1 at [cols])
    double* scal = hsm + cols + 1;                              // [hn2]
    double* nred = scal + 4;                                    // [kFWarps] norm partials
    uint32_t* scratch = reinterpret_cast<uint32_t*>(nred + kFWarps);  // l=21 write: 16 warps x 84 words
    volatile int* s_gate = reinterpret_cast<volatile int*>(scratch + kFWarps * 84);
    uint32_t* ers_s = reinterpret_cast<uint32_t*>(scratch + kFWarps * 84 + 4);  // [cols][2] exponent ranges
    const uint32_t* ers = FmtInfo<F>::frsz && a.B.erange ? ers_s : nullptr;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kFWarps);
        }
        fence_barrier_init();
        *s_gate = -1;
    }
    // launched as a programmatic dependent of the SpMV: everything below
    // reads what earlier kernels wrote
    pdl_wait();
    // previous launch's gate (written by CTA 0 at its end, after every CTA
    // of that launch had read it); CTA-uniform
    const bool spec = *reinterpret_cast<volatile unsigned*>(a.gate_hist) == 0u;
    if (blockIdx.x == 0 && threadIdx.x == 0) *a.bar_next = 0u;
    if (ers) {
        // exponent ranges of the columns read here; column `cols` (written
        // at the end of this launch, after two grid barriers) is reset
        for (uint32_t k = threadIdx.x; k < 2 * cols; k += kFThreads) ers_s[k] = a.B.erange[k];
        if (blockIdx.x == 0 && threadIdx.x < 2) a.out_erange[threadIdx.x] = 0u;
    }
    // the next launch's fixed-point accumulators (it starts after this grid)
    // (spread over the grid: one or two words per CTA)
    for (uint32_t k = blockIdx.x * kFThreads + threadIdx.x; k < 2 * a.fx_region / kFxStride;
         k += gridDim.x * kFThreads)
        a.fx_next[k * kFxStride] = 0ull;
    if (blockIdx.x == 0 && threadIdx.x == 0) a.fx_next[2 * a.fx_region] = 0ull;
    // omega^2 (from the SpMV epilogue) kept in shared memory: the gate and
    // the fixed-point scales need it (a register would be spilled and a
    // global reload costs an L2 round trip on the critical path)
    if (threadIdx.x == 0 && !a.om_parts) scal[1] = a.slot[2];
    __syncthreads();
    uint64_t r0, r1;
    fused_rows(a.B.n, a.rot, r0, r1);
    const uint32_t lim = static_cast<uint32_t>(r1 - r0);
    const uint32_t steps = (lim + kFStepRows - 1) / kFStepRows;
    constexpr int kChunkSteps = FGeo<F>::chunk;
    constexpr uint32_t kChunkRows = kChunkSteps * kFStepRows;
    const uint32_t nch = (lim + kChunkRows - 1) / kChunkRows;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == kFWarps) {
        // ---------------- producer: [SpMV tiles], dot1 (rev), update1, [dot2 (rev), update2]
        const uint64_t policy = policy_evict_normal();
        uint32_t it = 0;
        if (lane != 0) return;
        const uint64_t u0 = r0 / kUnitRows;
        for (int pass = 0; pass < 4; ++pass) {
            if (pass == (spec ? 3 : 2)) {
                while (*s_gate < 0) __nanosleep(64);
                if (*s_gate == 0) break;
            }
            const bool rev = (pass & 1) == 0;
            for (uint32_t jj = 0; jj < cols; ++jj) {
                const uint32_t j = rev ? cols - 1 - jj : jj;
                const unsigned char* col = a.B.data + j * a.B.col_stride_bytes;
                const unsigned char* ecol = reinterpret_cast<const unsigned char*>(a.B.exp + j * a.B.exp_col_stride);
                for (uint32_t ch = 0; ch < nch; ++ch, ++it) {
                    // whole steps: the last one may run past r1 (into the next
                    // range, or the allocation's slack after the last column)
                    const uint32_t ub = ch * (kChunkRows / kUnitRows);
                    const uint32_t un = min(kChunkSteps, static_cast<int>(steps - ch * kChunkSteps)) * (kFStepRows / kUnitRows);
                    const int stage = it % S;
                    mbar_wait(empty + stage, ((it / S) & 1) ^ 1);
                    mbar_arrive_expect_tx(full + stage, un * (UPAY + UEX));
                    unsigned char* dst = stages + stage * SB;
                    bulk_g2s(dst, col + (u0 + ub) * UPAY, un * UPAY, full + stage, policy);
                    if constexpr (UEX > 0)
                        bulk_g2s(dst + kChunkSteps * PAY, ecol + (u0 + ub) * UEX, un * UEX, full + stage, policy);
                }
            }
        }
        return;
    }

    // ---------------- consumers
    FTRACE(0);
    // the SpMV's omega^2 partials: loads issued before w's, summed after
    double omp = 0.0;
    if (a.om_parts)
        for (uint32_t k = threadIdx.x; k < a.om_count; k += kFConsumers) omp = __dadd_rn(omp, __ldcg(a.om_parts + k));
    uint32_t it = 0;
    double wv[kFusedMaxSteps][4];
    const uint64_t wend = min(r1, a.B.n);
#pragma unroll
    for (int s = 0; s < kFusedMaxSteps; ++s) {
        const uint64_t r = r0 + s * kFStepRows + 4u * threadIdx.x;
        if (s < static_cast<int>(steps)) {
            load_w(a.w, wend, r, wv[s]);
        } else {
            wv[s][0] = wv[s][1] = wv[s][2] = wv[s][3] = 0.0;
        }
    }
    FTRACE(1);
    if (a.om_parts) {
        // the same fixed order in every CTA: bit-identical omega^2 grid-wide
        const double om = cta_wnorm_sum(omp, nred);
        if (threadIdx.x == 0) {
            scal[1] = om;
            if (blockIdx.x == 0) a.slot[2] = om;
        }
        consumer_sync();
    }
    // fixed-point scales from omega (see fx_split): h and u partials at
    // e_h (|p| < 2^(e_h + 6) fits), hn1 partials at e_n
    const double om2 = scal[1];
    const int E2 = static_cast<int>((static_cast<unsigned long long>(__double_as_longlong(om2)) >> 52) & 0x7FF) - 1023;
    const bool fx_ok = om2 > 0.0 && E2 > -1023 && E2 < 1024 && E2 < 700 && E2 > -700;
    const int e_h = ((E2 + 2) >> 1) + 8, e_n = E2 + 1 + 8;
    unsigned long long* const fx0 = fx_ok ? a.fx : nullptr;
    unsigned long long* const fx1 = fx_ok ? a.fx + a.fx_region : nullptr;
    unsigned long long* const fxflag = a.fx + 2 * a.fx_region;
    volatile int* const s_fx = s_gate + 1;
    const uint32_t gs = a.gs;
    const uint64_t region = static_cast<uint64_t>(cols + 1) * gs;
    double* const P = a.partials;
    const bool cta0 = blockIdx.x == 0;
    unsigned seq = 0;

    // dot1 -> h
    fused_pass_any<F, true>(cols, lim, steps, nch, stages, full, empty, it, wv, red, hsm, ers);
    FTRACE(2);
    dot_partials_out(red, cols, P, gs, fx0, fxflag, 0, e_h);
    grid_allreduce_fx(a.bar, seq++, P, gs, cols, hsm, a.fx, fxflag, 0, fx_ok, e_h, ~0u, 0, s_fx, a.trace);
    if (cta0)
        for (uint32_t j = threadIdx.x; j < cols; j += kFConsumers) {
            a.slot[3 + j] = hsm[j];
            if (a.host_slot) a.host_slot[3 + j] = hsm[j];
        }
    FTRACE(3);
    // update1
    fused_pass_any<F, false>(cols, lim, steps, nch, stages, full, empty, it, wv, red, hsm, ers);
    FTRACE(4);
    const double hn1_part = cta_wnorm2(wv, nred);
    double* const P1 = P + region;
    if (spec) {
        // speculative dot2 -> u, reduced together with hn1
        fused_pass_any<F, true>(cols, lim, steps, nch, stages, full, empty, it, wv, red, hsm, ers);
        FTRACE(5);
        dot_partials_out(red, cols, P1, gs, fx1, fxflag, 1, e_h);
    }
    if (threadIdx.x == 0) {
        P1[static_cast<uint64_t>(cols) * gs + blockIdx.x] = hn1_part;
        if (spec && fx1) {
            long long c[3];
            if (fx_split(hn1_part, e_n, c)) fx_red(fx1 + fx_at(cols), c);
            else atomicOr(fxflag, 2ull);
        }
    }
    if (spec) grid_allreduce_fx(a.bar, seq++, P1, gs, cols + 1, hsm, a.fx + a.fx_region, fxflag, 1, fx_ok, e_h, cols, e_n,
                                s_fx, a.trace);
    else grid_allreduce(a.bar, seq++, P1 + static_cast<uint64_t>(cols) * gs, gs, 1, hsm + cols);
    FTRACE(6);
    const double hn1 = hsm[cols];
    const double omega2 = om2;
    // gmres.cpp:51 on the device (same IEEE ops as the host)
    const bool gate = sqrt(hn1) < a.eta * sqrt(omega2);
    if (threadIdx.x == 0) {
        *s_gate = gate ? 1 : 0;
        __threadfence_block();
    }
    if (cta0 && threadIdx.x == 0) {
        a.slot[0] = hn1;
        if (a.host_slot) {
            a.host_slot[0] = hn1;
            a.host_slot[2] = omega2;
        }
    }
    double hn2 = hn1;
    if (gate) {
        if (!spec) {
            fused_pass_any<F, true>(cols, lim, steps, nch, stages, full, empty, it, wv, red, hsm, ers);
            FTRACE(5);
            dot_partials_out(red, cols, P + 2 * region, gs);
            grid_allreduce(a.bar, seq++, P + 2 * region, gs, cols, hsm);
        }
        if (cta0)
            for (uint32_t j = threadIdx.x; j < cols; j += kFConsumers) {
                a.slot[a.u_off + j] = hsm[j];
                if (a.host_slot) a.host_slot[a.u_off + j] = hsm[j];
            }
        FTRACE(7);
        // update2 (u in hsm)
        fused_pass_any<F, false>(cols, lim, steps, nch, stages, full, empty, it, wv, red, hsm, ers);
        FTRACE(8);
        // h_next^2 of the second pass (gmres.cpp:66): ||w1 - V u||^2 =
        // hn1 - 2 u.(V^T w1) + u^T (V^T V) u = hn1 - |u|^2 + u^T E u with
        // u = V^T w1 and V^T V = I + E, |E| <~ 2^-p for a basis stored with
        // p significant bits (kOrthBits). When |u|^2 <= 2^(p-52) hn1 the
        // Pythagorean value hn1 - |u|^2 is within 2^-52 hn1 of the explicit
        // norm -- rounding level, below the tree sum's reduction-order noise
        // -- and the grid all-reduce of ||w2||^2 is skipped. That is the
        // usual case for FRSZ2-32/f32/f64 (u is the rounding residue of the
        // first pass); otherwise (and mostly for FRSZ2-16/21, f16) the
        // explicit norm is reduced. Every CTA holds the same u, so |u|^2
        // (xor butterfly: identical in every lane) and the branch are uniform.
        double uu = 0.0;
        for (uint32_t j = lane; j < cols; j += 32) uu = __dadd_rn(uu, __dmul_rn(hsm[j], hsm[j]));
        uu = warp_sum(uu);
        constexpr double kPyth = pow2(kOrthBits<F> - 52);
        if (uu <= kPyth * hn1) {
            hn2 = __dsub_rn(hn1, uu);
        } else {
            const double p = cta_wnorm2(wv, nred);
            double* const P3 = P + 3 * region;
            if (threadIdx.x == 0) P3[blockIdx.x] = p;
            grid_allreduce(a.bar, seq++, P3, gs, 1, scal, a.trace);
            hn2 = scal[0];
        }
        if (cta0 && threadIdx.x == 0) {
            a.slot[1] = hn2;
            if (a.host_slot) a.host_slot[1] = hn2;
        }
        FTRACE(9);
    }
    if (cta0 && threadIdx.x == 0) *a.gate_hist = gate ? 0u : 1u;
    pdl_trigger();  // the next SpMV may launch (it waits for this grid)
    // v = w / h_next of the last pass, written as the next basis column
    const double scale = 1.0 / sqrt(hn2);
    fused_write<F>(a, r0, r1, steps, wv, scale, scratch);
    FTRACE(10);
}

// Diagnostic: rotate the CTA -> row-range map (are slow CTAs slow because of
// their SM or their rows?). 0 in production.
uint32_t g_fused_rot = 0;

// Debug timeline of the fused kernel (CTA 0): enabled by CBGX_TRACE_FUSED=1,
// read back with cbgx_debug_fused_trace.
unsigned long long* g_trace = nullptr;
unsigned long long* fused_trace_buffer() {
    static const bool on = [] {
        const char* e = getenv("CBGX_TRACE_FUSED");
        return e && e[0] == '1';
    }();
    if (!on || !CBGX_FUSED_TRACE) return nullptr;
    if (!g_trace) {
        CBGX_CUDA(cudaMalloc(&g_trace, (kTraceBase + kTracePhases * 1024) * sizeof(unsigned long long)));
        CBGX_CUDA(cudaMemset(g_trace, 0, (kTraceBase + kTracePhases * 1024) * sizeof(unsigned long long)));
    }
    return g_trace;
}

template <int F>
size_t fused_smem(uint32_t cols) {
    return FGeo<F>::stages * (fstage_bytes<F>() + 16) +
           (kFWarps * (cols + 1) + (cols + 1) + 4 + kFWarps) * sizeof(double) + kFWarps * 84 * 4 + 32 +
           2 * (cols + 1) * sizeof(uint32_t);
}

// Grid size of the fused kernel (0 when not eligible): one CTA per SM,
// every CTA's rows within kFusedMaxSteps steps, cols + 1 <= kFConsumers.
template <int F>
int fused_grid(uint64_t n, uint32_t max_cols) {
    if (max_cols + 1 > static_cast<uint32_t>(kFConsumers)) return 0;
    const size_t smem = fused_smem<F>(max_cols);
    if (smem > 227 * 1024) return 0;
    static std::mutex mu;
    static std::map<std::pair<int, size_t>, int> cache;
    const auto key = std::make_pair(current_device(), smem);
    int per_sm = 0;
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = cache.find(key);
        if (it != cache.end()) {
            per_sm = it->second;
        } else {
            // the attribute is per kernel, not per size: set the maximum once
            CBGX_CUDA(cudaFuncSetAttribute(arnoldi_fused_kernel<F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           227 * 1024));
            CBGX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, arnoldi_fused_kernel<F>, kFThreads, smem));
            int coop = 0;
            CBGX_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, current_device()));
            if (!coop) per_sm = 0;
            cache.emplace(key, per_sm);
        }
    }
    if (per_sm < 1) return 0;
    const uint64_t units = (n + kUnitRows - 1) / kUnitRows;
    const uint64_t G = std::min<uint64_t>(static_cast<uint64_t>(sm_count()) * std::min(per_sm, kFCtasPerSM), std::max<uint64_t>(units, 1));
    uint64_t umax = 0;
    for (uint64_t sl = 0; sl < G; ++sl) {
        uint64_t u0, u1;
        fused_unit_range(units, G, sl, u0, u1);
        umax = std::max(umax, u1 - u0);
    }
    if (umax * kUnitRows > static_cast<uint64_t>(kFusedMaxSteps) * kFStepRows) return 0;
    return static_cast<int>(G);
}

template <int F> struct FusedLaunch {
    static void run(const cbgx_basis& V, uint32_t cols, const double* w, double* v_out, double* slot,
                    uint32_t u_off, double eta, uint32_t max_cols, double* host_slot, bool pdl,
                    Workspace* ws, cudaStream_t st, uint32_t om_count, bool* done) {
        // geometry fixed by the solver's capacity so it never changes mid-solve
        const int grid = fused_grid<F>(V.n, max_cols);
        *done = false;
        if (grid < 1 || cols > max_cols) return;  // not eligible: caller uses the split kernels
        const size_t smem = fused_smem<F>(max_cols);
        FusedArgs a;
        a.B = view_of(V);
        a.cols = cols;
        a.out_pay = static_cast<unsigned char*>(V.d_data) + static_cast<uint64_t>(cols) * V.col_stride_bytes;
        a.out_exp = V.d_exp ? V.d_exp + static_cast<uint64_t>(cols) * V.exp_col_stride : nullptr;
        a.out_erange = V.d_erange ? V.d_erange + 2ull * cols : nullptr;
        a.fx_region = fx_at(max_cols + 2);
        a.w = w;
        a.v_out = v_out;
        a.slot = slot;
        a.om_parts = om_count ? ws->omega_parts : nullptr;
        a.om_count = om_count;
        a.u_off = u_off;
        a.eta = eta;
        a.gs = static_cast<uint32_t>((grid + 1) / 2 * 2);
        a.partials = ws->get_partials(static_cast<size_t>(kRegions) * a.gs * (cols + 1));
        // two arrival counters used by alternate launches: each launch
        // zeroes the other one (the previous launch has completed)
        unsigned* c = ws->get_counter();
        // the launch sequence advances only once the launch succeeded: each
        // launch zeroes the counter the next one uses
        const uint64_t seq = ws->fused_launches;
        a.bar = c + Workspace::kFusedBar + (seq & 1) * 32;
        a.bar_next = c + Workspace::kFusedBar + ((seq + 1) & 1) * 32;
        a.gate_hist = c + Workspace::kFusedGate;
        {
            const size_t per_set = 2 * static_cast<size_t>(a.fx_region) + 1;
            unsigned long long* fx = ws->get_fx(per_set);
            a.fx = fx + (seq & 1) * ws->fx_words;
            a.fx_next = fx + ((seq + 1) & 1) * ws->fx_words;
        }
        a.trace = fused_trace_buffer();
        a.host_slot = host_slot;
        a.rot = g_fused_rot;
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(grid);
        lc.blockDim = dim3(kFThreads);
        lc.dynamicSmemBytes = smem;
        lc.stream = st;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = 1;
        lc.attrs = at;
        lc.numAttrs = pdl ? 2 : 1;
        note_launch();
        CBGX_CUDA(cudaLaunchKernelEx(&lc, arnoldi_fused_kernel<F>, a));
        ws->fused_launches = seq + 1;
        *done = true;
    }
};

void check_basis(const cbgx_basis* V) {
    if (!V) throw Error(CBGX_EINVAL, "basis: null descriptor");
    if (V->n_pad < V->n || V->n_pad % kRowAlign) throw Error(CBGX_EINVAL, "basis: bad row padding");
    (void)fmt_of(*V);
}

}  // namespace

void launch_cgs_dot(const cbgx_basis& V, uint64_t first, uint32_t cols, const double* w, int wn,
                    int reduction, double* h, Workspace* ws, cudaStream_t st, const GateArg& gate, bool coop) {
    if (first + cols > V.capacity) throw Error(CBGX_ERANGE, "basis: column index out of range");
    dispatch_fmt<DotLaunch>(fmt_of(V), view_of(V), first, cols, w, wn, reduction, h, ws, st, gate, coop);
    CBGX_CUDA(cudaGetLastError());
}

void launch_cgs_update(const cbgx_basis& V, uint64_t first, uint32_t cols, const double* h,
                       double sign, double* w, double* norm, int reduction, Workspace* ws,
                       cudaStream_t st, const GateArg& gate) {
    if (first + cols > V.capacity) throw Error(CBGX_ERANGE, "basis: column index out of range");
    dispatch_fmt<UpdateLaunch>(fmt_of(V), view_of(V), first, cols, h, sign, w, norm, reduction, ws, st, gate);
    CBGX_CUDA(cudaGetLastError());
}

void launch_basis_write(const cbgx_basis& V, uint64_t j, const double* x, const ScaleArg& scale,
                        double* v_out, uint64_t* bad, cudaStream_t st) {
    if (j >= V.capacity) throw Error(CBGX_ERANGE, "basis: cannot write column");
    dispatch_fmt<WriteLaunch>(fmt_of(V), V, j, x, scale, v_out, bad, st);
    CBGX_CUDA(cudaGetLastError());
}

namespace {
template <int F> struct FusedProbe {
    static void run(const cbgx_basis& V, uint64_t max_cols, bool* ok) {
        *ok = fused_grid<F>(V.n, static_cast<uint32_t>(max_cols)) > 0;
    }
};
}  // namespace

bool fused_eligible(const cbgx_basis& V, uint64_t max_cols) {
    bool ok = false;
    dispatch_fmt<FusedProbe>(fmt_of(V), V, max_cols, &ok);
    return ok;
}

bool launch_arnoldi_fused(const cbgx_basis& V, uint32_t cols, const double* w, double* v_out, double* slot,
                          uint32_t u_off, double eta, uint32_t max_cols, double* host_slot, bool pdl,
                          Workspace* ws, cudaStream_t st, uint32_t om_count) {
    if (cols + 1 > V.capacity) throw Error(CBGX_ERANGE, "basis: cannot write column");
    if (om_count && (!ws->omega_parts || om_count > ws->omega_cap))
        throw Error(CBGX_EINTERNAL, "fused: omega partials missing");
    bool done = false;
    dispatch_fmt<FusedLaunch>(fmt_of(V), V, cols, w, v_out, slot, u_off, eta, max_cols, host_slot, pdl, ws, st,
                              om_count, &done);
    CBGX_CUDA(cudaGetLastError());
    return done;
}

void launch_read_sweep(const cbgx_basis& V, uint64_t col, uint64_t n, int intensity, double mul, double add,
                       double* out, Workspace* ws, cudaStream_t st) {
    dispatch_fmt<SweepLaunch>(fmt_of(V), view_of(V), col, n, intensity, mul, add, out, ws, st);
    CBGX_CUDA(cudaGetLastError());
}

void launch_basis_read(const cbgx_basis& V, uint64_t j, uint64_t first, uint64_t count, double* out,
                       cudaStream_t st) {
    if (j >= V.capacity) throw Error(CBGX_ERANGE, "basis: column index out of range");
    dispatch_fmt<ReadLaunch>(fmt_of(V), view_of(V), j, first, count, out, st);
    CBGX_CUDA(cudaGetLastError());
}

}  // namespace cbgx

using namespace cbgx;

extern "C" {

int cbgx_basis_layout(uint32_t kind, uint32_t l, uint64_t n, uint64_t capacity, cbgx_basis* out,
                      uint64_t* data_bytes, uint64_t* exp_bytes) {
    return guard([&] {
        if (!out) throw Error(CBGX_EINVAL, "basis: null descriptor");
        cbgx_basis B{};
        B.kind = kind;
        B.bit_length = kind == CBGX_FRSZ2 ? l : 0;
        B.n = n;
        B.n_pad = pad_rows(std::max<uint64_t>(n, 1));
        B.capacity = capacity;
        const int f = fmt_of(B);
        // Each column is followed by kColTail zero rows that no kernel writes:
        // the fused kernel streams whole steps, and the last range's last
        // step may run up to one step past n_pad -- it then reads zeros of
        // the same column (finite, and multiplied by w = 0) instead of the
        // next column's possibly stale data.
        const uint64_t rows = B.n_pad + kColTail;
        uint64_t col_bytes = 0, exp_words = 0;
        switch (f) {
        case kF64: col_bytes = rows * 8; break;
        case kF32: col_bytes = rows * 4; break;
        case kF16: col_bytes = rows * 2; break;
        default:
            col_bytes = rows / 32 * l * 4;
            exp_words = rows / 32;
        }
        B.col_stride_bytes = col_bytes;
        B.exp_col_stride = exp_words;
        *out = B;
        // + 64 B slack: the l=21 step loader reads up to 3 words past a
        // block's last word.
        if (data_bytes) *data_bytes = col_bytes * capacity + 64;
        if (exp_bytes) *exp_bytes = exp_words * capacity * 4;
    });
}

int cbgx_basis_write(const cbgx_basis* V, uint64_t j, const double* d_x, const double* d_scale_src,
                     int scale_mode, double* d_v_out, uint64_t* d_bad_index, void* stream) {
    return guard([&] {
        check_basis(V);
        ScaleArg sc;
        sc.src = d_scale_src;
        sc.mode = scale_mode == 1 ? 1 : 0;
        launch_basis_write(*V, j, d_x, sc, d_v_out, d_bad_index, as_stream(stream));
    });
}

int cbgx_basis_read(const cbgx_basis* V, uint64_t j, uint64_t first, uint64_t count, double* d_out,
                    void* stream) {
    return guard([&] {
        check_basis(V);
        launch_basis_read(*V, j, first, count, d_out, as_stream(stream));
    });
}

int cbgx_cgs_dot(const cbgx_basis* V, uint64_t first, uint32_t cols, const double* d_w, int with_wnorm,
                 int reduction, double* d_h, cbgx_workspace* ws, void* stream) {
    return guard([&] {
        check_basis(V);
        if (!ws) throw Error(CBGX_EINVAL, "cgs: null workspace");
        launch_cgs_dot(*V, first, cols, d_w, with_wnorm, reduction, d_h, ws_of(ws), as_stream(stream));
    });
}

int cbgx_cgs_update(const cbgx_basis* V, uint64_t first, uint32_t cols, const double* d_h, int h_sign,
                    double* d_w, double* d_wnorm2, int reduction, cbgx_workspace* ws, void* stream) {
    return guard([&] {
        check_basis(V);
        if (!ws) throw Error(CBGX_EINVAL, "cgs: null workspace");
        launch_cgs_update(*V, first, cols, d_h, h_sign < 0 ? -1.0 : 1.0, d_w, d_wnorm2, reduction,
                          ws_of(ws), as_stream(stream));
    });
}

int cbgx_arnoldi_fused_step(const cbgx_basis* V, uint32_t cols, uint32_t max_cols, const double* d_w,
                            double* d_v_out, double* d_slot, double eta, int speculate, cbgx_workspace* ws,
                            void* stream) {
    return guard([&] {
        check_basis(V);
        if (!ws) throw Error(CBGX_EINVAL, "fused: null workspace");
        if (cols < 1 || cols > max_cols || max_cols + 1 > V->capacity)
            throw Error(CBGX_ERANGE, "fused: need 1 <= cols <= max_cols < capacity");
        cudaStream_t st = as_stream(stream);
        Workspace* w = ws_of(ws);
        // the gate history the kernel reads: 0 = previous gate open (the
        // second dot pass runs speculatively), 1 = closed
        unsigned* c = w->get_counter();
        const unsigned hist = speculate ? 0u : 1u;
        CBGX_CUDA(cudaMemcpyAsync(c + Workspace::kFusedGate, &hist, sizeof(unsigned), cudaMemcpyHostToDevice, st));
        const uint32_t u_off = 3 + max_cols + 1;
        if (!launch_arnoldi_fused(*V, cols, d_w, d_v_out, d_slot, u_off, eta, max_cols, nullptr, false, w, st))
            throw Error(CBGX_EINVAL, "fused: not eligible for this basis (n, capacity, format or device)");
        CBGX_CUDA(cudaStreamSynchronize(st));  // `hist` is a host stack value
    });
}

int cbgx_debug_fused_rotation(uint32_t rot) {
    return guard([&] { g_fused_rot = rot; });
}

int cbgx_debug_fused_trace(uint64_t* out, int count) {
    return guard([&] {
        if (!g_trace) throw Error(CBGX_EINVAL, "trace: build with CBGX_NVFLAGS_EXTRA=-DCBGX_FUSED_TRACE=1 and set CBGX_TRACE_FUSED=1 before the first fused launch");
        CBGX_CUDA(cudaMemcpy(out, g_trace, std::min(count, kTraceBase + kTracePhases * 1024) * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    });
}

}  // extern "C"
