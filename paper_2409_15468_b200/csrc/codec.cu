// codec.cu -- FRSZ2 compress / decompress on sm_100a.
//
// Reference semantics: frsz2.cpp:155-266 (compress, compress_block,
// decompress*, LSB-first packing :42-71) and kernels.hpp:18-58.
//
// Fast path (block size 32, l in {16, 21, 32}): a warp step is 4 blocks,
// each lane owns 4 consecutive values of one block (see compress4_kernel).
//
// Generic path (any block size, 2 <= l <= 64): one thread per block on
// encode (blocks own disjoint words, so no atomics), one thread per value on
// decode. Not on the solver hot path; it makes the drop-in codec total over
// the reference's parameter domain.
#include <cstdint>

#include "codec.cuh"
#include "common.cuh"

namespace cbgx {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// ---- 4-values-per-lane codec (the fast path) -----------------------------
// A warp step covers 128 rows = 4 blocks; lane l owns rows 4l..4l+3 (all in
// block l/8), so every lane moves 16-32 B per global access: 2x16 B of fp64
// and 16 B (l=32) / 8 B (l=16) of codes, the block exponent reduced over 8
// lanes with 3 shuffles. l=21 codes are assembled with funnel shifts and one
// shuffle (compress) or unpacked through an 84-word per-warp shared-memory
// window (decompress) so the global side stays coalesced. kSteps warp steps
// are in flight per iteration to keep enough bytes outstanding per SM.
constexpr int kSteps = 4;

// >= 3 CTAs/SM: the l=21 packing otherwise takes 94 registers (2 CTAs/SM);
// l=21 at 2 steps x 4 CTAs/SM (64 registers, no spill): 4.0 -> 4.4 TB/s
// (scripts/ab_codec.sh; 3 steps x 3 CTAs 4.19).
#ifndef C21_STEPS
#define C21_STEPS 2
#endif
#ifndef C21_MINB
#define C21_MINB 4
#endif
template <int L, bool kScale>
__global__ void __launch_bounds__(kThreads, L == 21 ? C21_MINB : 3)
compress4_kernel(const double* __restrict__ x, uint64_t n, uint64_t nb_write,
                 uint32_t* __restrict__ exps, uint32_t* __restrict__ payload,
                 ScaleArg scale, double* __restrict__ v_out,
                 unsigned long long* __restrict__ bad, uint32_t* __restrict__ erange) {
    // erange != nullptr: the column's exponent range (erange_fold over the
    // written blocks, cbgx_basis.d_erange) folded here, one atomic pair per CTA
    uint32_t e_inv = 0, e_max = 0;
    // l=21: 2 steps in flight (4 spill at the register budget of 3 CTAs/SM)
    constexpr int kSteps = L == 21 ? C21_STEPS : ::cbgx::kSteps;
    const int lane = threadIdx.x & 31;
    const double s = kScale ? scale.value() : 1.0;
    const uint64_t nsteps = (nb_write + 3) / 4;
    const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * kWarps) + (threadIdx.x >> 5);
    const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * kWarps;
    for (uint64_t s0 = warp * kSteps; s0 < nsteps; s0 += nwarps * kSteps) {
        double v[kSteps][4];
#pragma unroll
        for (int u = 0; u < kSteps; ++u) {
            const uint64_t r = (s0 + u) * 128 + 4u * lane;
            if (s0 + u < nsteps && r + 3 < n) {
                load4_cs(x + r, v[u]);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) v[u][k] = (s0 + u < nsteps && r + k < n) ? x[r + k] : 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < kSteps; ++u) {
            if (s0 + u >= nsteps) break;  // warp-uniform
            const uint64_t r = (s0 + u) * 128 + 4u * lane;
            const uint64_t blk = r / 32;
            const bool live = blk < nb_write;  // 8-lane-uniform
            uint32_t e = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (kScale) v[u][k] = __dmul_rn(v[u][k], s);
                const uint32_t ek = exp_field(v[u][k]);
                if (ek == 0x7FFu && r + k < n) atomicMin(bad, static_cast<unsigned long long>(r + k));
                e = max(e, ek);
            }
            if (kScale && v_out) {
                if (r + 3 < n) {
                    store4(v_out + r, v[u]);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (r + k < n) v_out[r + k] = v[u][k];
                }
            }
            e = max(e, __shfl_xor_sync(0xFFFFFFFFu, e, 1));
            e = max(e, __shfl_xor_sync(0xFFFFFFFFu, e, 2));
            e = max(e, __shfl_xor_sync(0xFFFFFFFFu, e, 4));
            uint32_t c[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) c[k] = encode32<L>(v[u][k], e);
            if (live && (lane & 7) == 0) exps[blk] = e;
            if (erange && live) {  // erange_fold (basis.cuh)
                e_max = max(e_max, e);
                if (e) e_inv = max(e_inv, 2047u - e);
            }
            if constexpr (L == 32) {
                if (live) reinterpret_cast<uint4*>(payload)[r / 4] = make_uint4(c[0], c[1], c[2], c[3]);
            } else if constexpr (L == 16) {
                if (live) reinterpret_cast<uint2*>(payload)[r / 4] = make_uint2(c[0] | (c[1] << 16), c[2] | (c[3] << 16));
            } else {
                // Lane L's four codes are bits [84 L, 84 L + 84) of the step's
                // 84-word stream (block L/8 starts at 672 (L/8), value 4 (L%8)
                // + k at 21 k). The lane writes the words that START in its
                // range: at bit offsets o, o + 32 (and o + 64 when o < 20),
                // o = -84 L mod 32; a word reaching past the range takes the
                // next lane's first bits (one shuffle) -- funnel shifts of the
                // lane's 84-bit string, no shared memory.
                const uint32_t w0 = c[0] | (c[1] << 21);
                const uint32_t w1 = (c[1] >> 11) | (c[2] << 10) | (c[3] << 31);
                const uint32_t nb0 = __shfl_down_sync(0xFFFFFFFFu, w0, 1);
                const uint32_t w2 = (c[3] >> 1) | (nb0 << 20), w3 = nb0 >> 12;
                const uint32_t o = (32u - ((20u * lane) & 31u)) & 31u;
                const uint32_t i0 = (84u * lane + o) >> 5;
                const uint64_t b0 = (s0 + u) * 4;  // first block of the step
                uint32_t* dst = payload + b0 * 21 + i0;
                const uint64_t words = (min(nb_write, b0 + 4) - b0) * 21;
                if (i0 < words) dst[0] = __funnelshift_r(w0, w1, o);
                if (i0 + 1 < words) dst[1] = __funnelshift_r(w1, w2, o);
                if (o < 20u && i0 + 2 < words) dst[2] = __funnelshift_r(w2, w3, o);
            }
        }
    }
    if (erange) {  // kernel-uniform
        __shared__ uint32_t s_er[2 * kWarps];
        e_inv = __reduce_max_sync(0xFFFFFFFFu, e_inv);
        e_max = __reduce_max_sync(0xFFFFFFFFu, e_max);
        if (lane == 0) {
            s_er[threadIdx.x >> 5] = e_inv;
            s_er[kWarps + (threadIdx.x >> 5)] = e_max;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < kWarps; ++w) {
                e_inv = max(e_inv, s_er[w]);
                e_max = max(e_max, s_er[kWarps + w]);
            }
            atomicMax(erange, e_inv);
            atomicMax(erange + 1, e_max);
        }
    }
}

template <int L>
__global__ void __launch_bounds__(kThreads)
decompress4_kernel(const uint32_t* __restrict__ exps, const uint32_t* __restrict__ payload,
                   uint64_t n, double* __restrict__ out) {
    __shared__ uint32_t wbuf_all[kWarps][84 + 4];
    const int lane = threadIdx.x & 31;
    uint32_t* wbuf = wbuf_all[threadIdx.x >> 5];
    const uint64_t nb = (n + 31) / 32;
    const uint64_t nsteps = (nb + 3) / 4;
    const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * kWarps) + (threadIdx.x >> 5);
    const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * kWarps;
    for (uint64_t s0 = warp * kSteps; s0 < nsteps; s0 += nwarps * kSteps) {
        uint32_t em[kSteps];
        uint4 cw[kSteps];  // l=32: 4 codes; l=16: x,y = 4 packed codes; l=21: 3 loaded words
#pragma unroll
        for (int u = 0; u < kSteps; ++u) {
            const uint64_t r = (s0 + u) * 128 + 4u * lane;
            const uint64_t blk = min(r / 32, nb - 1);
            em[u] = __ldg(exps + blk);
            if constexpr (L == 32) {
                cw[u] = r / 32 < nb ? __ldcs(reinterpret_cast<const uint4*>(payload) + r / 4) : make_uint4(0, 0, 0, 0);
            } else if constexpr (L == 16) {
                const uint2 t = r / 32 < nb ? __ldcs(reinterpret_cast<const uint2*>(payload) + r / 4) : make_uint2(0, 0);
                cw[u] = make_uint4(t.x, t.y, 0, 0);
            } else {
                const uint64_t b0 = (s0 + u) * 4;
                const uint64_t words = b0 < nb ? (min(nb, b0 + 4) - b0) * 21 : 0;
                const uint32_t* src = payload + b0 * 21;
                cw[u].x = static_cast<uint64_t>(lane) < words ? __ldcs(src + lane) : 0u;
                cw[u].y = static_cast<uint64_t>(lane + 32) < words ? __ldcs(src + lane + 32) : 0u;
                cw[u].z = static_cast<uint64_t>(lane + 64) < words && lane + 64 < 84 ? __ldcs(src + lane + 64) : 0u;
            }
        }
#pragma unroll
        for (int u = 0; u < kSteps; ++u) {
            if (s0 + u >= nsteps) break;  // warp-uniform
            const uint64_t r = (s0 + u) * 128 + 4u * lane;
            uint32_t code[4];
            if constexpr (L == 32) {
                code[0] = cw[u].x; code[1] = cw[u].y; code[2] = cw[u].z; code[3] = cw[u].w;
            } else if constexpr (L == 16) {
                code[0] = cw[u].x & 0xFFFFu; code[1] = cw[u].x >> 16;
                code[2] = cw[u].y & 0xFFFFu; code[3] = cw[u].y >> 16;
            } else {
                wbuf[lane] = cw[u].x;
                wbuf[lane + 32] = cw[u].y;
                if (lane + 64 < 88) wbuf[lane + 64] = lane + 64 < 84 ? cw[u].z : 0u;
                __syncwarp();
                const uint32_t bit = (lane >> 3) * 672u + (lane & 7) * 84u;
                const uint32_t q = bit >> 5, sh = bit & 31u;
                const uint32_t w0 = wbuf[q], w1 = wbuf[q + 1], w2 = wbuf[q + 2], w3 = wbuf[q + 3];
                __syncwarp();
                const uint32_t o1 = sh + 21, o2 = sh + 42, o3 = sh + 63;
                code[0] = __funnelshift_r(w0, w1, sh) & 0x1FFFFFu;
                code[1] = (o1 < 32 ? __funnelshift_r(w0, w1, o1) : __funnelshift_r(w1, w2, o1 - 32)) & 0x1FFFFFu;
                code[2] = (o2 < 64 ? __funnelshift_r(w1, w2, o2 - 32) : __funnelshift_r(w2, w3, o2 - 64)) & 0x1FFFFFu;
                code[3] = (o3 < 64 ? __funnelshift_r(w1, w2, o3 - 32) : __funnelshift_r(w2, w3, o3 - 64)) & 0x1FFFFFu;
            }
            const BlockDecoder<L> dec(em[u]);
            double v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = dec(code[k]);
            if (r + 3 < n) {
                store4(out + r, v, true);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (r + k < n) out[r + k] = v[k];
            }
        }
    }
}

// ---- generic (any bs >= 1, 2 <= l <= 64) --------------------------------

__device__ __forceinline__ uint64_t stream_get(const uint32_t* w, uint64_t off, uint32_t nbits) {
    uint64_t out = 0;
    for (uint32_t got = 0; got < nbits;) {
        const uint64_t pos = off + got;
        const uint32_t sh = static_cast<uint32_t>(pos & 31);
        const uint32_t take = min(32u - sh, nbits - got);
        const uint32_t mask = take == 32 ? 0xFFFFFFFFu : ((1u << take) - 1);
        out |= static_cast<uint64_t>((w[pos >> 5] >> sh) & mask) << got;
        got += take;
    }
    return out;
}

__device__ __forceinline__ void stream_put(uint32_t* w, uint64_t off, uint64_t val, uint32_t nbits) {
    for (uint32_t put = 0; put < nbits;) {
        const uint64_t pos = off + put;
        const uint32_t sh = static_cast<uint32_t>(pos & 31);
        const uint32_t take = min(32u - sh, nbits - put);
        const uint32_t mask = take == 32 ? 0xFFFFFFFFu : ((1u << take) - 1);
        w[pos >> 5] |= (static_cast<uint32_t>(val >> put) & mask) << sh;
        put += take;
    }
}

__global__ void compress_generic_kernel(const double* __restrict__ x, uint64_t n, uint32_t bs,
                                        uint32_t l, uint64_t wpb, uint32_t* __restrict__ exps,
                                        uint32_t* __restrict__ payload,
                                        unsigned long long* __restrict__ bad) {
    const uint64_t nb = (n + bs - 1) / bs;
    for (uint64_t b = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; b < nb;
         b += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t off = b * bs;
        uint32_t e_max = 0;
        for (uint32_t j = 0; j < bs; ++j) {
            const double v = off + j < n ? x[off + j] : 0.0;
            const uint32_t e = exp_field(v);
            if (e == 0x7FFu) atomicMin(bad, static_cast<unsigned long long>(off + j));
            e_max = max(e_max, e);
        }
        exps[b] = e_max;
        uint32_t* w = payload + b * wpb;
        for (uint64_t k = 0; k < wpb; ++k) w[k] = 0;
        for (uint32_t j = 0; j < bs; ++j) {
            const double v = off + j < n ? x[off + j] : 0.0;
            stream_put(w, static_cast<uint64_t>(j) * l, encode_any(v, e_max, l), l);
        }
    }
}

__global__ void decompress_generic_kernel(const uint32_t* __restrict__ exps,
                                          const uint32_t* __restrict__ payload, uint32_t bs,
                                          uint32_t l, uint64_t wpb, uint64_t first,
                                          uint64_t count, double* __restrict__ out) {
    for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < count;
         k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t i = first + k;
        const uint64_t b = i / bs, r = i % bs;
        out[k] = decode_any(stream_get(payload + b * wpb, r * l, l), exps[b], l);
    }
}

__global__ void encode_block_kernel(const double* __restrict__ v, uint32_t count, uint32_t l,
                                    uint32_t* __restrict__ emax_out, uint64_t* __restrict__ codes,
                                    unsigned long long* __restrict__ bad) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    uint32_t e_max = 0;
    for (uint32_t j = 0; j < count; ++j) {
        const uint32_t e = exp_field(v[j]);
        if (e == 0x7FFu && *bad == ~0ull) *bad = j;
        e_max = max(e_max, e);
    }
    *emax_out = e_max;
    for (uint32_t j = 0; j < count; ++j) codes[j] = encode_any(v[j], e_max, l);
}

#ifndef CODEC_CTAS_PER_SM
#define CODEC_CTAS_PER_SM 16  // measured (scripts/ab_codec.sh): 16 > 8 ~ 32 for the 2^24 round trip
#endif
int grid_for(uint64_t units, int per_cta) {
    const uint64_t want = (units + per_cta - 1) / per_cta;
    const uint64_t cap = static_cast<uint64_t>(sm_count()) * CODEC_CTAS_PER_SM;
    return static_cast<int>(want < 1 ? 1 : (want > cap ? cap : want));
}

void validate(uint32_t bs, uint32_t l) {
    if (bs < 1) throw Error(CBGX_EINVAL, "frsz2: block_size must be >= 1");
    if (l < 2 || l > 64) throw Error(CBGX_EINVAL, "frsz2: bit_length must be in [2, 64]");
}

bool fast_path(uint32_t bs, uint32_t l) { return bs == 32 && (l == 16 || l == 21 || l == 32); }

}  // namespace

void launch_compress(const double* x, uint64_t n, uint64_t nb_write, uint32_t bs, uint32_t l,
                     uint32_t* exps, uint32_t* payload, const ScaleArg& scale, double* v_out, uint64_t* bad,
                     cudaStream_t st, uint32_t* erange) {
    validate(bs, l);
    if (nb_write == 0) return;
    auto* badp = reinterpret_cast<unsigned long long*>(bad);
    if (fast_path(bs, l)) {
        const int grid = grid_for((nb_write + 3) / 4, kWarps * kSteps);
        const bool sc = scale.src != nullptr;
#define CBGX_LAUNCH_C(LL)                                                                    \
    if (sc) CBGX_K(compress4_kernel<LL, true><<<grid, kThreads, 0, st>>>(x, n, nb_write, exps, payload, \
                                                                   scale, v_out, badp, erange)); \
    else CBGX_K(compress4_kernel<LL, false><<<grid, kThreads, 0, st>>>(x, n, nb_write, exps, payload,   \
                                                                 ScaleArg{}, nullptr, badp, erange))
        if (l == 32) { CBGX_LAUNCH_C(32); }
        else if (l == 16) { CBGX_LAUNCH_C(16); }
        else { CBGX_LAUNCH_C(21); }
#undef CBGX_LAUNCH_C
    } else {
        if (scale.src || v_out || erange)
            throw Error(CBGX_EINVAL, "frsz2: fused scale needs bs=32, l in {16,21,32}");
        const uint64_t nb = (n + bs - 1) / bs;
        if (nb_write != nb) throw Error(CBGX_EINVAL, "frsz2: generic codec writes exactly num_blocks");
        CBGX_K(compress_generic_kernel<<<grid_for(nb, 128), 128, 0, st>>>(x, n, bs, l, (static_cast<uint64_t>(bs) * l + 31) / 32,
                                                                  exps, payload, badp));
    }
    CBGX_CUDA(cudaGetLastError());
}

void launch_decompress(const uint32_t* exps, const uint32_t* payload, uint64_t n, uint32_t bs,
                       uint32_t l, uint64_t first, uint64_t count, double* out, cudaStream_t st) {
    validate(bs, l);
    if (count == 0) return;
    if (fast_path(bs, l) && first == 0 && count == n) {
        const int grid = grid_for(((n + 31) / 32 + 3) / 4, kWarps * kSteps);
        if (l == 32) CBGX_K(decompress4_kernel<32><<<grid, kThreads, 0, st>>>(exps, payload, n, out));
        else if (l == 16) CBGX_K(decompress4_kernel<16><<<grid, kThreads, 0, st>>>(exps, payload, n, out));
        else CBGX_K(decompress4_kernel<21><<<grid, kThreads, 0, st>>>(exps, payload, n, out));
    } else {
        CBGX_K(decompress_generic_kernel<<<grid_for(count, 256), 256, 0, st>>>(
            exps, payload, bs, l, (static_cast<uint64_t>(bs) * l + 31) / 32, first, count, out));
    }
    CBGX_CUDA(cudaGetLastError());
}

// Scratch u64 for synchronous non-finite checks.
uint64_t sync_bad_index(const std::function<void(uint64_t*)>& body, cudaStream_t st) {
    uint64_t* d_bad = nullptr;
    CBGX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_bad), sizeof(uint64_t), st));
    CBGX_CUDA(cudaMemsetAsync(d_bad, 0xFF, sizeof(uint64_t), st));
    uint64_t h_bad = ~0ull;
    try {
        body(d_bad);
        CBGX_CUDA(cudaMemcpyAsync(&h_bad, d_bad, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
        CBGX_CUDA(cudaFreeAsync(d_bad, st));
        CBGX_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
        cudaFreeAsync(d_bad, st);
        throw;
    }
    return h_bad;
}

[[noreturn]] void throw_non_finite(uint64_t index) {
    throw Error(CBGX_ENONFINITE, "frsz2: non-finite value at index " + std::to_string(index), index);
}

}  // namespace cbgx

using namespace cbgx;

extern "C" {

uint64_t cbgx_frsz2_num_blocks(uint64_t n, uint32_t bs) { return bs ? (n + bs - 1) / bs : 0; }
uint64_t cbgx_frsz2_words_per_block(uint32_t bs, uint32_t l) {
    return (static_cast<uint64_t>(bs) * l + 31) / 32;
}
uint64_t cbgx_frsz2_storage_bytes(uint64_t n, uint32_t bs, uint32_t l) {
    const uint64_t nb = cbgx_frsz2_num_blocks(n, bs);
    return nb * cbgx_frsz2_words_per_block(bs, l) * 4 + nb * 4;
}
double cbgx_frsz2_max_abs_error_bound(uint32_t e_max, uint32_t l) {
    return ldexp(1.0, static_cast<int>(e_max) - 1023 - (static_cast<int>(l) - 2));
}

int cbgx_frsz2_compress_async(const double* d_in, uint64_t n, uint32_t bs, uint32_t l,
                              uint32_t* d_exp, uint32_t* d_payload, uint64_t* d_bad_index,
                              void* stream) {
    return guard([&] {
        validate(bs, l);
        launch_compress(d_in, n, cbgx_frsz2_num_blocks(n, bs), bs, l, d_exp, d_payload, ScaleArg{},
                        nullptr, d_bad_index, as_stream(stream));
    });
}

int cbgx_frsz2_compress(const double* d_in, uint64_t n, uint32_t bs, uint32_t l, uint32_t* d_exp,
                        uint32_t* d_payload, void* stream) {
    return guard([&] {
        validate(bs, l);
        cudaStream_t st = as_stream(stream);
        const uint64_t bad = sync_bad_index([&](uint64_t* d_bad) {
            launch_compress(d_in, n, cbgx_frsz2_num_blocks(n, bs), bs, l, d_exp, d_payload, ScaleArg{},
                            nullptr, d_bad, st);
        }, st);
        if (bad != ~0ull) throw_non_finite(bad);
    });
}

int cbgx_frsz2_decompress(const uint32_t* d_exp, const uint32_t* d_payload, uint64_t n, uint32_t bs,
                          uint32_t l, double* d_out, void* stream) {
    return guard([&] { launch_decompress(d_exp, d_payload, n, bs, l, 0, n, d_out, as_stream(stream)); });
}

int cbgx_frsz2_decompress_range(const uint32_t* d_exp, const uint32_t* d_payload, uint64_t n,
                                uint32_t bs, uint32_t l, uint64_t first, uint64_t count,
                                double* d_out, void* stream) {
    return guard([&] {
        validate(bs, l);
        const uint64_t limit = cbgx_frsz2_num_blocks(n, bs) * bs;
        if (first > limit || count > limit - first) throw Error(CBGX_ERANGE, "frsz2: index out of range");
        launch_decompress(d_exp, d_payload, n, bs, l, first, count, d_out, as_stream(stream));
    });
}

int cbgx_frsz2_encode_block(const double* d_values, uint32_t count, uint32_t l, uint32_t* d_emax,
                            uint64_t* d_codes, void* stream) {
    return guard([&] {
        validate(count, l);
        cudaStream_t st = as_stream(stream);
        const uint64_t bad = sync_bad_index([&](uint64_t* d_bad) {
            CBGX_K(encode_block_kernel<<<1, 32, 0, st>>>(d_values, count, l, d_emax, d_codes,
                                                  reinterpret_cast<unsigned long long*>(d_bad)));
            CBGX_CUDA(cudaGetLastError());
        }, st);
        if (bad != ~0ull) throw_non_finite(bad);
    });
}

}  // extern "C"
