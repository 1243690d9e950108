// basis.cuh -- Krylov basis panel access: per-format loaders/decoders shared
// by the fused CGS kernels, the basis write/read kernels and the
// reference-order (serial) kernels.
//
// Reference: basis.hpp:23-83, basis.cpp:85-205; codec kernels.hpp:18-58.
#pragma once

#include <cuda_fp16.h>

#include "cbgx.h"
#include "common.cuh"

namespace cbgx {

// Storage format tags (compile-time).
enum Fmt : int { kF64 = 0, kF32 = 1, kF16 = 2, kZ16 = 3, kZ21 = 4, kZ32 = 5 };

template <int F> struct FmtInfo;
template <> struct FmtInfo<kF64> { static constexpr int L = 0;  static constexpr bool frsz = false; };
template <> struct FmtInfo<kF32> { static constexpr int L = 0;  static constexpr bool frsz = false; };
template <> struct FmtInfo<kF16> { static constexpr int L = 0;  static constexpr bool frsz = false; };
template <> struct FmtInfo<kZ16> { static constexpr int L = 16; static constexpr bool frsz = true; };
template <> struct FmtInfo<kZ21> { static constexpr int L = 21; static constexpr bool frsz = true; };
template <> struct FmtInfo<kZ32> { static constexpr int L = 32; static constexpr bool frsz = true; };

inline int fmt_of(const cbgx_basis& B) {
    switch (B.kind) {
    case CBGX_F64: return kF64;
    case CBGX_F32: return kF32;
    case CBGX_F16: return kF16;
    case CBGX_FRSZ2:
        if (B.bit_length == 16) return kZ16;
        if (B.bit_length == 21) return kZ21;
        if (B.bit_length == 32) return kZ32;
        break;
    }
    throw Error(CBGX_EINVAL, "storage format: frsz2 bit length must be 16, 21 or 32");
}

// Plain-old-data view passed to kernels.
struct BasisView {
    const unsigned char* data;
    const uint32_t* exp;
    uint64_t col_stride_bytes;
    uint64_t exp_col_stride;
    uint64_t n;
    uint64_t n_pad;
    const uint32_t* erange;  // optional per-column exponent range (cbgx_basis.d_erange)
};

inline BasisView view_of(const cbgx_basis& B) {
    return BasisView{static_cast<const unsigned char*>(B.d_data), B.d_exp, B.col_stride_bytes,
                     B.exp_col_stride, B.n, B.n_pad, B.d_erange};
}

// ----------------------------------------- per-column fast-decode test
// erange[2j] = max over column j's nonzero blocks of (2047 - e_max) (0: all
// blocks zero), erange[2j + 1] = max e_max. A block with e_max = 0 holds
// only signed zeros (encode_one, kernels.hpp:18-37) and decodes exactly on
// the fast path with the clamped scale 2^(1-1023-...) (every product is an
// exact zero), so a column takes the vote-free fast path when its smallest
// nonzero block maximum is above L - 2 ...
template <int L>
__device__ __forceinline__ bool col_dot_fast(uint32_t inv, uint32_t) {
    return inv == 0 || 2047u - inv > static_cast<uint32_t>(L - 2);
}
// ... and, for an update with coefficient h (biased exponent h_exp), when
// h * scale stays in the range frsz_upd_ok requires for every block.
template <int L>
__device__ __forceinline__ bool col_upd_fast(uint32_t inv, uint32_t emax, double h, int h_exp) {
    if (!col_dot_fast<L>(inv, emax)) return false;
    if (h == 0.0 || inv == 0) return true;
    const int emin = 2047 - static_cast<int>(inv);
    return h_exp != 0 && h_exp + emin - 1023 - (L - 2) >= 1 && h_exp + static_cast<int>(emax) - 1023 - (L - 2) <= 1994;
}
// Column writers fold a block maximum into (inv, emax).
__device__ __forceinline__ void erange_fold(uint32_t e, uint32_t& inv, uint32_t& emax) {
    emax = max(emax, e);
    if (e) inv = max(inv, 2047u - e);
}

// ---------------------------------------------------- binary16 (half.cpp)
// half_to_double, half.cpp:62-81 (exact widening).
__device__ __forceinline__ double half_bits_to_double(uint32_t h) {
    const uint32_t e = (h >> 10) & 31u, f = h & 1023u;
    const unsigned long long s = static_cast<unsigned long long>(h >> 15) << 63;
    if (e == 0) {
        const double mag = static_cast<double>(f) * 0x1p-24;
        return (h & 0x8000u) ? -mag : mag;
    }
    if (e == 31) {
        return __longlong_as_double(static_cast<long long>(s | (0x7FFull << 52) | (f ? static_cast<unsigned long long>(f) << 42 : 0ull)));
    }
    return __longlong_as_double(static_cast<long long>(s | (static_cast<unsigned long long>(e - 15 + 1023) << 52) |
                                                       (static_cast<unsigned long long>(f) << 42)));
}

// half_from_double, half.cpp:9-60 (RNE, saturating to +-65504).
__device__ __forceinline__ uint16_t double_to_half_bits(double x) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    const uint32_t s = static_cast<uint32_t>((b >> 48) & 0x8000u);
    const int e = static_cast<int>((b >> 52) & 0x7FF);
    const unsigned long long f = b & ((1ull << 52) - 1);
    if (e == 0x7FF) return static_cast<uint16_t>(s | (f ? 0x7E00u : 0x7BFFu));
    if (e == 0) return static_cast<uint16_t>(s);
    const int ue = e - 1023;
    if (ue >= 16) return static_cast<uint16_t>(s | 0x7BFFu);
    unsigned long long sig;
    int drop;
    if (ue >= -14) {
        sig = f;
        drop = 42;
    } else {
        sig = f | (1ull << 52);
        drop = 28 - ue;
        if (drop >= 54) return static_cast<uint16_t>(s);
    }
    unsigned long long keep = sig >> drop;
    const unsigned long long rest = sig & ((1ull << drop) - 1);
    const unsigned long long halfp = 1ull << (drop - 1);
    if (rest > halfp || (rest == halfp && (keep & 1))) ++keep;
    if (ue >= -14) {
        uint32_t he = static_cast<uint32_t>(ue + 15);
        if (keep == 1024) {
            keep = 0;
            ++he;
        }
        if (he >= 31) return static_cast<uint16_t>(s | 0x7BFFu);
        return static_cast<uint16_t>(s | (he << 10) | static_cast<uint32_t>(keep));
    }
    return static_cast<uint16_t>(s | static_cast<uint32_t>(keep));
}

// ------------------------------------------------ single-element decode
template <int F>
__device__ __forceinline__ double basis_value(const BasisView& B, uint64_t col, uint64_t row) {
    const unsigned char* base = B.data + col * B.col_stride_bytes;
    if constexpr (F == kF64) {
        return reinterpret_cast<const double*>(base)[row];
    } else if constexpr (F == kF32) {
        return static_cast<double>(reinterpret_cast<const float*>(base)[row]);
    } else if constexpr (F == kF16) {
        return half_bits_to_double(reinterpret_cast<const uint16_t*>(base)[row]);
    } else {
        constexpr int L = FmtInfo<F>::L;
        const uint32_t* w = reinterpret_cast<const uint32_t*>(base);
        const uint32_t e = B.exp[col * B.exp_col_stride + row / 32];
        uint32_t code;
        if constexpr (L == 32) {
            code = w[row];
        } else if constexpr (L == 16) {
            code = reinterpret_cast<const uint16_t*>(w)[row];
        } else {
            const uint64_t bit = (row / 32) * 672 + (row % 32) * 21;
            const uint64_t q = bit >> 5;
            const unsigned long long win = (static_cast<unsigned long long>(w[q + 1]) << 32) | w[q];
            code = static_cast<uint32_t>(win >> (bit & 31)) & 0x1FFFFFu;
        }
        return BlockDecoder<L>(e)(code);
    }
}

// --------------------------------------- vectorised 4-row step (fast CGS)
// A thread's step covers 4 consecutive rows r..r+3 (r % 4 == 0), all in the
// same 32-block, of one column. The fused kernels call
//   dot(w)        -> sum_k v_k * w_k        (TREE order: any order is allowed)
//   update(h, w)  -> w_k = w_k - h * v_k    (two roundings: bit-identical)
//
// FRSZ2 fast path. With scale = 2^(e_max-1023-(L-2)) a value is
// v = +-mag * scale exactly, so
//   dot:    the step sum is (sum_k +-mag_k * w_k) * scale  (scale once/step)
//   update: h * v = +-(mag * (h * scale)) where hs = h * scale is exact
//           whenever it stays in the normal range (checked per step), hence
//           RN(h*v) = +-RN(mag*hs) bit for bit.
// Per value that is: mask, I2F.F64.U32, a sign LOP3 on the high word and one
// FP64 op. Blocks where the fast path is not exact (e_max <= L-2, where the
// reference flushes tiny values to zero, or hs outside the normal range)
// take the exact decoder (BlockDecoder) out of line.

// Sign-magnitude codes split for the fast path: magnitude and the sign moved
// to bit 31.
struct Codes4 {
    uint32_t mag[4];
    uint32_t sgn[4];
};

__device__ __forceinline__ double signed_i2f(uint32_t mag, uint32_t sgn) {
    const double d = u32_to_f64(mag);
    return __hiloint2double(__double2hiint(d) ^ static_cast<int>(sgn), __double2loint(d));
}

// 2^(e_max - 1023 - (L - 2)), the exponent clamped to the normal range:
// e_max > L - 2 leaves it unchanged; e_max = 0 (a block of signed zeros)
// gets a positive finite scale, so +-0 codes still decode to +-0.
template <int L>
__device__ __forceinline__ double frsz_scale(uint32_t e) {
    return __hiloint2double(max(static_cast<int>(e) - (L - 2), 1) << 20, 0);
}

template <int L>
__device__ __forceinline__ double fast_dot(const Codes4& c, uint32_t e, const double w[4]) {
    // two independent FMA chains (depth 3 instead of 4 dependent FP64 ops)
    const double a = fma(signed_i2f(c.mag[1], c.sgn[1]), w[1], __dmul_rn(signed_i2f(c.mag[0], c.sgn[0]), w[0]));
    const double b = fma(signed_i2f(c.mag[3], c.sgn[3]), w[3], __dmul_rn(signed_i2f(c.mag[2], c.sgn[2]), w[2]));
    return __dmul_rn(__dadd_rn(a, b), frsz_scale<L>(e));
}

// Exact per-step decode (rare path), inlined: as a real call it forces w
// out of registers (2.4x slower fused passes on B200).
template <int L>
__device__ __forceinline__ void slow_decode(const Codes4& c, uint32_t e, double v[4]) {
    const BlockDecoder<L> d(e);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t code = c.mag[k] | (c.sgn[k] >> (32 - L));
        v[k] = d(code);
    }
}

// The fast/exact split is decided per warp (all 32 lanes must be active):
// a warp-uniform branch costs no divergence bookkeeping in the hot loop.
template <int L>
__device__ __forceinline__ double frsz_dot(const Codes4& c, uint32_t e, const double w[4]) {
    if (__builtin_expect(__all_sync(0xFFFFFFFFu, e > L - 2), 1)) return fast_dot<L>(c, e, w);
    double v[4];
    slow_decode<L>(c, e, v);
    double s = __dmul_rn(v[0], w[0]);
#pragma unroll
    for (int k = 1; k < 4; ++k) s = fma(v[k], w[k], s);
    return s;
}

// Exact-decode dot / update (BlockDecoder for every value, no fast-path
// test): the path of a column whose exponent range does not prove the fast
// decode exact. Bit-identical to frsz_dot / frsz_update on every block.
template <int L>
__device__ __forceinline__ double frsz_dot_exact(const Codes4& c, uint32_t e, const double w[4]) {
    double v[4];
    slow_decode<L>(c, e, v);
    double s = __dmul_rn(v[0], w[0]);
#pragma unroll
    for (int k = 1; k < 4; ++k) s = fma(v[k], w[k], s);
    return s;
}
template <int L>
__device__ __forceinline__ void frsz_update_exact(const Codes4& c, uint32_t e, double h, double w[4]) {
    double v[4];
    slow_decode<L>(c, e, v);
#pragma unroll
    for (int k = 0; k < 4; ++k) w[k] = __dsub_rn(w[k], __dmul_rn(h, v[k]));
}

// The 4 decoded values, fast path only (caller checked e > L - 2).
template <int L>
__device__ __forceinline__ void frsz_decode_fast(const Codes4& c, uint32_t e, double v[4]) {
    const double sc = frsz_scale<L>(e);
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = __dmul_rn(signed_i2f(c.mag[k], c.sgn[k]), sc);
}

// v[k] * mul in one rounding: +-mag * RN(scale * mul), exact-equivalent to
// RN(decode(v) * mul) whenever scale * mul is itself exact (normal; the
// caller checks the block exponent range): decode(v) = +-mag * scale is
// exact and so is the scaling.
template <int L>
__device__ __forceinline__ double frsz_smul(uint32_t e, double mul) {
    return __dmul_rn(__hiloint2double(static_cast<int>((e - (L - 2)) << 20), 0), mul);
}
// The same products with one FP64 instruction per value: (2^52 + mag) *
// smul - 2^52 * smul is exactly mag * smul before the FMA's single rounding
// (c0 = -2^52 * smul, exact while smul <= 2^971: the caller's exponent
// range), then the sign -- RN is symmetric.
__device__ __forceinline__ void frsz_decode_mul_fma(const Codes4& c, double smul, double c0, double v[4]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double p = fma(__hiloint2double(0x43300000, static_cast<int>(c.mag[k])), smul, c0);
        v[k] = __hiloint2double(__double2hiint(p) ^ static_cast<int>(c.sgn[k]), __double2loint(p));
    }
}
template <int L>
__device__ __forceinline__ void frsz_decode_mul(const Codes4& c, double smul, double v[4]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = __dmul_rn(signed_i2f(c.mag[k], c.sgn[k]), smul);
}

// The 4 decoded values (warp-uniform fast/exact split like frsz_dot).
template <int L>
__device__ __forceinline__ void frsz_decode(const Codes4& c, uint32_t e, double v[4]) {
    if (__builtin_expect(__all_sync(0xFFFFFFFFu, e > L - 2), 1)) {
        frsz_decode_fast<L>(c, e, v);
        return;
    }
    slow_decode<L>(c, e, v);
}

// h_exp: biased exponent field of h (hoisted per column by the caller).
// The FMA update below is exact-equivalent when the block scale is normal and
// h * scale stays in range.
template <int L>
__device__ __forceinline__ bool frsz_upd_ok(uint32_t e, double h, int h_exp) {
    const int es = static_cast<int>(e) - (L - 2);          // scale's biased exponent
    const int hse = h_exp + es - 1023;                      // exponent of h*scale
    // hse <= 1994: 2^52 * hs stays finite, so c0 below is exact
    return es > 0 && (h == 0.0 || (h_exp != 0 && hse >= 1 && hse <= 1994));
}

template <int L>
__device__ __forceinline__ void frsz_update_fast(const Codes4& c, uint32_t e, double h, double w[4]) {
    const double hs = __dmul_rn(h, frsz_scale<L>(e));
    const double c0 = __dmul_rn(hs, -0x1p52);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        // RN(mag * hs) as one FMA on the FP64 pipe: (2^52 + mag) * hs
        // - 2^52 * hs is exactly mag * hs before the single rounding
        const double p = fma(__hiloint2double(0x43300000, static_cast<int>(c.mag[k])), hs, c0);
        w[k] = __dsub_rn(w[k], __hiloint2double(__double2hiint(p) ^ static_cast<int>(c.sgn[k]), __double2loint(p)));
    }
}

template <int L>
__device__ __forceinline__ void frsz_update(const Codes4& c, uint32_t e, double h, int h_exp, double w[4]) {
    if (__builtin_expect(__all_sync(0xFFFFFFFFu, frsz_upd_ok<L>(e, h, h_exp)), 1)) {
        frsz_update_fast<L>(c, e, h, w);
        return;
    }
    double v[4];
    slow_decode<L>(c, e, v);
#pragma unroll
    for (int k = 0; k < 4; ++k) w[k] = __dsub_rn(w[k], __dmul_rn(h, v[k]));
}

template <int F> struct Step;

template <> struct Step<kZ32> {
    uint4 c;
    uint32_t e;
    __device__ __forceinline__ void load(const BasisView& B, uint64_t col, uint64_t r) {
        c = __ldg(reinterpret_cast<const uint4*>(B.data + col * B.col_stride_bytes) + r / 4);
        e = __ldg(B.exp + col * B.exp_col_stride + r / 32);
    }
    __device__ __forceinline__ Codes4 codes() const {
        Codes4 k;
        const uint32_t w[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            k.mag[i] = w[i] & 0x7FFFFFFFu;
            k.sgn[i] = w[i] & 0x80000000u;
        }
        return k;
    }
    __device__ __forceinline__ double dot(const double w[4]) const { return frsz_dot<32>(codes(), e, w); }
    __device__ __forceinline__ void decode(double v[4]) const { frsz_decode<32>(codes(), e, v); }
    __device__ __forceinline__ void update(double h, int he, double w[4]) const { frsz_update<32>(codes(), e, h, he, w); }
    // stage-level fast path (the caller votes once over all steps of a stage)
    __device__ __forceinline__ bool fast() const { return e > 32 - 2; }
    __device__ __forceinline__ double dot_fast(const double w[4]) const { return fast_dot<32>(codes(), e, w); }
    __device__ __forceinline__ bool upd_ok(double h, int he) const { return frsz_upd_ok<32>(e, h, he); }
    __device__ __forceinline__ void update_fast(double h, int, double w[4]) const { frsz_update_fast<32>(codes(), e, h, w); }
    __device__ __forceinline__ void decode_fast(double v[4]) const { frsz_decode_fast<32>(codes(), e, v); }
    __device__ __forceinline__ double dot_exact(const double w[4]) const { return frsz_dot_exact<32>(codes(), e, w); }
    __device__ __forceinline__ void update_exact(double h, double w[4]) const { frsz_update_exact<32>(codes(), e, h, w); }
    __device__ __forceinline__ double smul(double mul) const { return frsz_smul<32>(e, mul); }
    __device__ __forceinline__ void decode_mul(double sm, double v[4]) const { frsz_decode_mul<32>(codes(), sm, v); }
    __device__ __forceinline__ void decode_mul_fma(double sm, double c0, double v[4]) const { frsz_decode_mul_fma(codes(), sm, c0, v); }
};

template <> struct Step<kZ16> {
    uint2 c;
    uint32_t e;
    __device__ __forceinline__ void load(const BasisView& B, uint64_t col, uint64_t r) {
        c = __ldg(reinterpret_cast<const uint2*>(B.data + col * B.col_stride_bytes) + r / 4);
        e = __ldg(B.exp + col * B.exp_col_stride + r / 32);
    }
    __device__ __forceinline__ Codes4 codes() const {
        Codes4 k;
        k.mag[0] = c.x & 0x7FFFu;          k.sgn[0] = (c.x << 16) & 0x80000000u;
        k.mag[1] = (c.x >> 16) & 0x7FFFu;  k.sgn[1] = c.x & 0x80000000u;
        k.mag[2] = c.y & 0x7FFFu;          k.sgn[2] = (c.y << 16) & 0x80000000u;
        k.mag[3] = (c.y >> 16) & 0x7FFFu;  k.sgn[3] = c.y & 0x80000000u;
        return k;
    }
    __device__ __forceinline__ double dot(const double w[4]) const { return frsz_dot<16>(codes(), e, w); }
    __device__ __forceinline__ void decode(double v[4]) const { frsz_decode<16>(codes(), e, v); }
    __device__ __forceinline__ void update(double h, int he, double w[4]) const { frsz_update<16>(codes(), e, h, he, w); }
    // stage-level fast path (the caller votes once over all steps of a stage)
    __device__ __forceinline__ bool fast() const { return e > 16 - 2; }
    __device__ __forceinline__ double dot_fast(const double w[4]) const { return fast_dot<16>(codes(), e, w); }
    __device__ __forceinline__ bool upd_ok(double h, int he) const { return frsz_upd_ok<16>(e, h, he); }
    __device__ __forceinline__ void update_fast(double h, int, double w[4]) const { frsz_update_fast<16>(codes(), e, h, w); }
    __device__ __forceinline__ void decode_fast(double v[4]) const { frsz_decode_fast<16>(codes(), e, v); }
    __device__ __forceinline__ double dot_exact(const double w[4]) const { return frsz_dot_exact<16>(codes(), e, w); }
    __device__ __forceinline__ void update_exact(double h, double w[4]) const { frsz_update_exact<16>(codes(), e, h, w); }
    __device__ __forceinline__ double smul(double mul) const { return frsz_smul<16>(e, mul); }
    __device__ __forceinline__ void decode_mul(double sm, double v[4]) const { frsz_decode_mul<16>(codes(), sm, v); }
    __device__ __forceinline__ void decode_mul_fma(double sm, double c0, double v[4]) const { frsz_decode_mul_fma(codes(), sm, c0, v); }
};

template <> struct Step<kZ21> {
    uint32_t w0, w1, w2, w3;
    uint32_t sh, e;
    __device__ __forceinline__ void load(const BasisView& B, uint64_t col, uint64_t r) {
        const uint32_t* p = reinterpret_cast<const uint32_t*>(B.data + col * B.col_stride_bytes);
        const uint32_t bit = (static_cast<uint32_t>(r) & 31u) * 21u;  // 0..588
        const uint64_t q = (r / 32) * 21 + (bit >> 5);
        sh = bit & 31u;
        w0 = __ldg(p + q); w1 = __ldg(p + q + 1); w2 = __ldg(p + q + 2); w3 = __ldg(p + q + 3);
        e = __ldg(B.exp + col * B.exp_col_stride + r / 32);
    }
    __device__ __forceinline__ Codes4 codes() const {
        // code k sits at bit sh + 21k of the 128-bit little-endian window
        // w0..w3 (sh + 84 <= 112): shift the window right by the thread's sh
        // once (three funnel shifts), then the codes are at the fixed bits
        // 0, 21, 42, 63 -- constant shifts, no per-code selects
        uint32_t c[4];
        const uint32_t x0 = __funnelshift_r(w0, w1, sh), x1 = __funnelshift_r(w1, w2, sh),
                       x2 = __funnelshift_r(w2, w3, sh);
        c[0] = x0;
        c[1] = __funnelshift_r(x0, x1, 21);
        c[2] = x1 >> 10;
        c[3] = __funnelshift_r(x1, x2, 31);
        Codes4 k;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            k.mag[i] = c[i] & 0xFFFFFu;
            k.sgn[i] = (c[i] << 11) & 0x80000000u;
        }
        return k;
    }
    __device__ __forceinline__ double dot(const double w[4]) const { return frsz_dot<21>(codes(), e, w); }
    __device__ __forceinline__ void decode(double v[4]) const { frsz_decode<21>(codes(), e, v); }
    __device__ __forceinline__ void update(double h, int he, double w[4]) const { frsz_update<21>(codes(), e, h, he, w); }
    // stage-level fast path (the caller votes once over all steps of a stage)
    __device__ __forceinline__ bool fast() const { return e > 21 - 2; }
    __device__ __forceinline__ double dot_fast(const double w[4]) const { return fast_dot<21>(codes(), e, w); }
    __device__ __forceinline__ bool upd_ok(double h, int he) const { return frsz_upd_ok<21>(e, h, he); }
    __device__ __forceinline__ void update_fast(double h, int, double w[4]) const { frsz_update_fast<21>(codes(), e, h, w); }
    __device__ __forceinline__ void decode_fast(double v[4]) const { frsz_decode_fast<21>(codes(), e, v); }
    __device__ __forceinline__ double dot_exact(const double w[4]) const { return frsz_dot_exact<21>(codes(), e, w); }
    __device__ __forceinline__ void update_exact(double h, double w[4]) const { frsz_update_exact<21>(codes(), e, h, w); }
    __device__ __forceinline__ double smul(double mul) const { return frsz_smul<21>(e, mul); }
    __device__ __forceinline__ void decode_mul(double sm, double v[4]) const { frsz_decode_mul<21>(codes(), sm, v); }
    __device__ __forceinline__ void decode_mul_fma(double sm, double c0, double v[4]) const { frsz_decode_mul_fma(codes(), sm, c0, v); }
};

template <> struct Step<kF64> {
    double2 a, b;
    __device__ __forceinline__ void load(const BasisView& B, uint64_t col, uint64_t r) {
        const double2* p = reinterpret_cast<const double2*>(B.data + col * B.col_stride_bytes) + r / 2;
        a = __ldg(p);
        b = __ldg(p + 1);
    }
    __device__ __forceinline__ void values(double v[4]) const { v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y; }
    __device__ __forceinline__ void decode(double v[4]) const { values(v); }
    __device__ __forceinline__ double dot(const double w[4]) const {
        double v[4];
        values(v);
        double s = __dmul_rn(v[0], w[0]);
#pragma unroll
        for (int k = 1; k < 4; ++k) s = fma(v[k], w[k], s);
        return s;
    }
    __device__ __forceinline__ void update(double h, int, double w[4]) const {
        double v[4];
        values(v);
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = __dsub_rn(w[k], __dmul_rn(h, v[k]));
    }
};

template <> struct Step<kF32> {
    float4 c;
    __device__ __forceinline__ void load(const BasisView& B, uint64_t col, uint64_t r) {
        c = __ldg(reinterpret_cast<const float4*>(B.data + col * B.col_stride_bytes) + r / 4);
    }
    __device__ __forceinline__ void values(double v[4]) const { v[0] = c.x; v[1] = c.y; v[2] = c.z; v[3] = c.w; }
    __device__ __forceinline__ void decode(double v[4]) const { values(v); }
    __device__ __forceinline__ double dot(const double w[4]) const {
        double v[4];
        values(v);
        double s = __dmul_rn(v[0], w[0]);
#pragma unroll
        for (int k = 1; k < 4; ++k) s = fma(v[k], w[k], s);
        return s;
    }
    __device__ __forceinline__ void update(double h, int, double w[4]) const {
        double v[4];
        values(v);
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = __dsub_rn(w[k], __dmul_rn(h, v[k]));
    }
};

template <> struct Step<kF16> {
    uint2 c;
    __device__ __forceinline__ void load(const BasisView& B, uint64_t col, uint64_t r) {
        c = __ldg(reinterpret_cast<const uint2*>(B.data + col * B.col_stride_bytes) + r / 4);
    }
    __device__ __forceinline__ void values(double v[4]) const {
        const uint32_t h[4] = {c.x & 0xFFFFu, c.x >> 16, c.y & 0xFFFFu, c.y >> 16};
        // warp-uniform fast path: normal halves and signed zeros widen by
        // re-biasing the exponent (exact); subnormal / inf / nan take the
        // general conversion (half.cpp:62-81)
        bool fast = true;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t e = (h[k] >> 10) & 31u;
            fast = fast && e != 31u && (e != 0u || (h[k] & 1023u) == 0u);
        }
        if (__builtin_expect(__all_sync(0xFFFFFFFFu, fast), 1)) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t e = (h[k] >> 10) & 31u;
                const uint32_t hi = ((h[k] & 0x8000u) << 16) | (e ? ((e + 1008u) << 20) | ((h[k] & 1023u) << 10) : 0u);
                v[k] = __hiloint2double(static_cast<int>(hi), 0);
            }
            return;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = half_bits_to_double(h[k]);
    }
    __device__ __forceinline__ void decode(double v[4]) const { values(v); }
    __device__ __forceinline__ double dot(const double w[4]) const {
        double v[4];
        values(v);
        double s = __dmul_rn(v[0], w[0]);
#pragma unroll
        for (int k = 1; k < 4; ++k) s = fma(v[k], w[k], s);
        return s;
    }
    __device__ __forceinline__ void update(double h, int, double w[4]) const {
        double v[4];
        values(v);
#pragma unroll
        for (int k = 0; k < 4; ++k) w[k] = __dsub_rn(w[k], __dmul_rn(h, v[k]));
    }
};

// Stored bytes per value of a format (algorithmic traffic accounting).
inline double stored_bytes_per_value(int f) {
    switch (f) {
    case kF64: return 8.0;
    case kF32: return 4.0;
    case kF16: return 2.0;
    case kZ16: return 17.0 / 8.0;
    case kZ21: return 22.0 / 8.0;
    default: return 33.0 / 8.0;
    }
}

}  // namespace cbgx
