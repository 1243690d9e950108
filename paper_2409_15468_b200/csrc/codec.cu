// codec.cu -- FRSZ2 compress / decompress on sm_100a.
//
// Reference semantics: frsz2.cpp:155-266 (compress, compress_block,
// decompress*, LSB-first packing :42-71) and kernels.hpp:18-58.
//
// Fast path (block size 32, l in {16, 21, 32}): one warp per 32-value block,
// lane j owns value j. The block exponent is one warp max-reduction
// (__reduce_max_sync -> CREDUX), codes are produced in registers and packed
// with shuffles into coalesced stores: 128 B (l=32), 64 B (l=16) or 84 B
// (l=21: word w of the block's bit stream gathers the <= 3 codes that overlap
// it). Decompression is the mirror image. Each warp keeps kUnroll blocks in
// flight so enough loads are outstanding to saturate HBM.
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
constexpr int kUnroll = 4;

template <int L>
__device__ __forceinline__ void store_block(uint32_t code, uint32_t* __restrict__ words, int lane) {
    if constexpr (L == 32) {
        words[lane] = code;
    } else if constexpr (L == 16) {
        const uint32_t hi = __shfl_down_sync(0xFFFFFFFFu, code, 1);
        if ((lane & 1) == 0) words[lane >> 1] = code | (hi << 16);
    } else {
        static_assert(L == 21, "fast codec handles l in {16, 21, 32}");
        // Output word w covers stream bits [32w, 32w+32); codes j0..j0+2
        // with j0 = floor(32w/21) overlap it.
        const int w = lane;
        const int j0 = (32 * w) / 21;
        const uint32_t c0 = __shfl_sync(0xFFFFFFFFu, code, j0 & 31);
        const uint32_t c1 = __shfl_sync(0xFFFFFFFFu, code, (j0 + 1) & 31);
        const uint32_t c2 = __shfl_sync(0xFFFFFFFFu, code, (j0 + 2) & 31);
        const uint64_t win = static_cast<uint64_t>(c0) |
                             (static_cast<uint64_t>(j0 + 1 < 32 ? c1 : 0u) << 21) |
                             (static_cast<uint64_t>(j0 + 2 < 32 ? c2 : 0u) << 42);
        if (w < 21) words[w] = static_cast<uint32_t>(win >> (32 * w - 21 * j0));
    }
}

template <int L>
__device__ __forceinline__ uint32_t load_code(const uint32_t* __restrict__ words, int lane) {
    if constexpr (L == 32) {
        return __ldg(words + lane);
    } else if constexpr (L == 16) {
        return __ldg(reinterpret_cast<const uint16_t*>(words) + lane);
    } else {
        const uint32_t mine = lane < 21 ? __ldg(words + lane) : 0u;
        const int bit = 21 * lane;
        const int q = bit >> 5;
        const uint32_t w0 = __shfl_sync(0xFFFFFFFFu, mine, q);
        const uint32_t w1 = __shfl_sync(0xFFFFFFFFu, mine, (q + 1) & 31);
        const uint64_t win = (static_cast<uint64_t>(w1) << 32) | w0;
        return static_cast<uint32_t>(win >> (bit & 31)) & 0x1FFFFFu;
    }
}

// Encodes blocks [0, nb_write) of s*x (rows >= n read as 0.0 -- the tail
// zero padding of frsz2.cpp:187-191).
template <int L, bool kScale>
__global__ void __launch_bounds__(kThreads)
compress32_kernel(const double* __restrict__ x, uint64_t n, uint64_t nb_write,
                  uint32_t* __restrict__ exps, uint32_t* __restrict__ payload,
                  ScaleArg scale, double* __restrict__ v_out,
                  unsigned long long* __restrict__ bad) {
    const int lane = threadIdx.x & 31;
    const double s = kScale ? scale.value() : 1.0;
    const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * kWarps) + (threadIdx.x >> 5);
    const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * kWarps;
    for (uint64_t b0 = warp * kUnroll; b0 < nb_write; b0 += nwarps * kUnroll) {
        double v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint64_t row = (b0 + u) * 32 + lane;
            v[u] = (b0 + u < nb_write && row < n) ? x[row] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint64_t b = b0 + u;
            if (b >= nb_write) break;  // warp-uniform
            const uint64_t row = b * 32 + lane;
            double val = v[u];
            if (kScale) {
                val = __dmul_rn(val, s);
                if (v_out && row < n) v_out[row] = val;
            }
            const uint32_t e = exp_field(val);
            if (e == 0x7FFu) atomicMin(bad, static_cast<unsigned long long>(row));
            const uint32_t e_max = __reduce_max_sync(0xFFFFFFFFu, e);
            const uint32_t code = encode32<L>(val, e_max);
            if (lane == 0) exps[b] = e_max;
            store_block<L>(code, payload + b * L, lane);
        }
    }
}

template <int L>
__global__ void __launch_bounds__(kThreads)
decompress32_kernel(const uint32_t* __restrict__ exps, const uint32_t* __restrict__ payload,
                    uint64_t n, double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const uint64_t nb = (n + 31) / 32;
    const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * kWarps) + (threadIdx.x >> 5);
    const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * kWarps;
    for (uint64_t b0 = warp * kUnroll; b0 < nb; b0 += nwarps * kUnroll) {
        uint32_t code[kUnroll], em[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint64_t b = b0 + u < nb ? b0 + u : nb - 1;
            em[u] = __ldg(exps + b);
            code[u] = load_code<L>(payload + b * L, lane);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint64_t row = (b0 + u) * 32 + lane;
            const BlockDecoder<L> dec(em[u]);
            const double val = dec(code[u]);
            if (b0 + u < nb && row < n) out[row] = val;
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

int grid_for(uint64_t units, int per_cta) {
    const uint64_t want = (units + per_cta - 1) / per_cta;
    const uint64_t cap = static_cast<uint64_t>(sm_count()) * 8;
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
                     cudaStream_t st) {
    validate(bs, l);
    if (nb_write == 0) return;
    auto* badp = reinterpret_cast<unsigned long long*>(bad);
    if (fast_path(bs, l)) {
        const int grid = grid_for(nb_write, kWarps * kUnroll);
        const bool sc = scale.src != nullptr;
#define CBGX_LAUNCH_C(LL)                                                                    \
    if (sc) CBGX_K(compress32_kernel<LL, true><<<grid, kThreads, 0, st>>>(x, n, nb_write, exps, payload, \
                                                                   scale, v_out, badp)); \
    else CBGX_K(compress32_kernel<LL, false><<<grid, kThreads, 0, st>>>(x, n, nb_write, exps, payload,   \
                                                                 ScaleArg{}, nullptr, badp))
        if (l == 32) { CBGX_LAUNCH_C(32); }
        else if (l == 16) { CBGX_LAUNCH_C(16); }
        else { CBGX_LAUNCH_C(21); }
#undef CBGX_LAUNCH_C
    } else {
        if (scale.src || v_out) throw Error(CBGX_EINVAL, "frsz2: fused scale needs bs=32, l in {16,21,32}");
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
        const int grid = grid_for((n + 31) / 32, kWarps * kUnroll);
        if (l == 32) CBGX_K(decompress32_kernel<32><<<grid, kThreads, 0, st>>>(exps, payload, n, out));
        else if (l == 16) CBGX_K(decompress32_kernel<16><<<grid, kThreads, 0, st>>>(exps, payload, n, out));
        else CBGX_K(decompress32_kernel<21><<<grid, kThreads, 0, st>>>(exps, payload, n, out));
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
