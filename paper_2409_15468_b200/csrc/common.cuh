// common.cuh -- shared device/host helpers for the sm_100a FRSZ2 / CB-GMRES
// kernels. Everything here is bit-exact with the reference codec semantics
// (reference: proj/include/cbg/kernels.hpp:18-58).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "cbgx.h"

namespace cbgx {

// ---------------------------------------------------------------- errors
struct Error : std::runtime_error {
    int code;
    uint64_t index;
    Error(int c, const std::string& m, uint64_t i = 0) : std::runtime_error(m), code(c), index(i) {}
};

void set_error(int code, const std::string& msg, uint64_t index = 0);
void check_cuda(cudaError_t e, const char* what);
#define CBGX_CUDA(x) ::cbgx::check_cuda((x), #x)
int sm_count();
int current_device();

// Wrap a C-ABI body: exceptions -> status codes + thread-local message.
template <class F>
int guard(F&& f) {
    try {
        f();
        return CBGX_OK;
    } catch (const Error& e) {
        set_error(e.code, e.what(), e.index);
        return e.code;
    } catch (const std::bad_alloc&) {
        set_error(CBGX_ENOMEM, "out of memory");
        return CBGX_ENOMEM;
    } catch (const std::exception& e) {
        set_error(CBGX_EINTERNAL, e.what());
        return CBGX_EINTERNAL;
    }
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Rows of a basis column are padded to a multiple of this, so the fused
// CGS kernels stream whole tiles without tail predication on the basis.
constexpr uint64_t kRowAlign = 8192;
// Zero rows after each basis column's n_pad rows (see cbgx_basis_layout).
constexpr uint64_t kColTail = 2048;
inline uint64_t pad_rows(uint64_t n) { return (n + kRowAlign - 1) / kRowAlign * kRowAlign; }

// --------------------------------------------------------- device codec
// Biased 11-bit exponent field of the high word.
__device__ __forceinline__ uint32_t exp_field(double x) {
    return (static_cast<uint32_t>(__double2hiint(x)) >> 20) & 0x7FFu;
}

// kernels.hpp:18-37 for 2 <= L <= 32, given the block's e_max.
// The magnitude sig >> sh (sig = the 53-bit significand, sh = 54 - L +
// e_max - e >= 22) never uses sig's low 21 bits: it is t >> (sh - 21) with
// t = sig >> 21 (one funnel shift; the exponent and sign bits of the high
// word shift out) and a clamped shift (0 once sh - 21 >= 32) -- no 64-bit
// shift.
template <int L>
__device__ __forceinline__ uint32_t encode32(double x, uint32_t e_max) {
    const uint32_t hi = static_cast<uint32_t>(__double2hiint(x));
    const uint32_t lo = static_cast<uint32_t>(__double2loint(x));
    const uint32_t sgn = (hi >> 31) << (L - 1);
    const uint32_t e = (hi >> 20) & 0x7FFu;
    const uint32_t t = __funnelshift_l(lo, hi | 0x100000u, 11);
    const uint32_t mag = __funnelshift_rc(t, 0u, 33u - L + e_max - e);  // e <= e_max: shift >= 1
    return e == 0 ? sgn : (sgn | mag);
}

// Generic kernels.hpp:18-37 (any 2 <= l <= 64).
__device__ __forceinline__ uint64_t encode_any(double x, uint32_t e_max, uint32_t l) {
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
    const uint64_t sgn = (b >> 63) << (l - 1);
    const int e = static_cast<int>((b >> 52) & 0x7FF);
    if (e == 0) return sgn;
    const uint64_t sig = (b & ((1ull << 52) - 1)) | (1ull << 52);
    const int sh = 54 - static_cast<int>(l) + static_cast<int>(e_max) - e;
    uint64_t mag;
    if (sh >= 64) mag = 0;
    else if (sh >= 0) mag = sig >> sh;
    else mag = sig << (-sh);
    return sgn | mag;
}

// Generic kernels.hpp:42-58.
__device__ __forceinline__ double decode_any(uint64_t code, uint32_t e_max, uint32_t l) {
    const uint64_t neg = (code >> (l - 1)) & 1;
    const uint64_t mag = code & ((1ull << (l - 1)) - 1);
    if (mag == 0) return __longlong_as_double(static_cast<long long>(neg << 63));
    const int p = 63 - __clzll(static_cast<long long>(mag));
    const int e = static_cast<int>(e_max) - (static_cast<int>(l) - 2 - p);
    if (e <= 0) return __longlong_as_double(static_cast<long long>(neg << 63));
    const uint64_t rest = mag ^ (1ull << p);
    const uint64_t f52 = p <= 52 ? rest << (52 - p) : rest >> (p - 52);
    return __longlong_as_double(static_cast<long long>((neg << 63) | (static_cast<uint64_t>(e) << 52) | f52));
}

// 256-bit global accesses (sm_100: LDG/STG.E.ENL2.256): four doubles per
// lane per instruction halve the LSU instructions of the streaming kernels.
// The address must be 32-B aligned.
__device__ __forceinline__ void ld4_cs(const double* p, double v[4]) {
    asm volatile("ld.global.cs.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}
__device__ __forceinline__ void ld4_nc(const double* p, double v[4]) {
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
}
__device__ __forceinline__ void st4(double* p, const double v[4]) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
                 : "memory");
}
__device__ __forceinline__ void st4_cs(double* p, const double v[4]) {
    asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
                 : "memory");
}
__device__ __forceinline__ bool aligned32(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31u) == 0; }
__device__ __forceinline__ bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Four consecutive doubles at an 8-B aligned address: one 256-bit access,
// two 128-bit accesses or four scalar ones, by the address's alignment.
__device__ __forceinline__ void load4(const double* p, double v[4]) {
    if (aligned32(p)) {
        ld4_nc(p, v);
    } else if (aligned16(p)) {
        const double2 a = __ldg(reinterpret_cast<const double2*>(p));
        const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = __ldg(p + k);
    }
}
__device__ __forceinline__ void load4_cs(const double* p, double v[4]) {
    if (aligned32(p)) {
        ld4_cs(p, v);
    } else if (aligned16(p)) {
        const double2 a = __ldcs(reinterpret_cast<const double2*>(p));
        const double2 b = __ldcs(reinterpret_cast<const double2*>(p) + 1);
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = __ldcs(p + k);
    }
}
__device__ __forceinline__ void store4(double* p, const double v[4], bool streaming = false) {
    if (aligned32(p)) {
        if (streaming) st4_cs(p, v);
        else st4(p, v);
    } else if (aligned16(p)) {
        reinterpret_cast<double2*>(p)[0] = make_double2(v[0], v[1]);
        reinterpret_cast<double2*>(p)[1] = make_double2(v[2], v[3]);
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) p[k] = v[k];
    }
}

// Exact u32 -> double on the FP64 pipe: (2^52 + m) - 2^52. The conversion
// instruction (I2F.F64.U32) issues on the XU pipe, 16 lanes/clk/SM, which
// the FRSZ2 decode saturated (ncu: XU pipe 74% in the fused CGS kernel);
// DADD runs at the FP64 rate.
__device__ __forceinline__ double u32_to_f64(uint32_t m) {
    return __dsub_rn(__hiloint2double(0x43300000, static_cast<int>(m)), 0x1p52);
}

// Per-block decode context for the fixed-rate formats (L <= 32).
// Fast path (e_max > L-2, i.e. no decoded value can fall below 2^-1022):
//   value = (double)mag * 2^(e_max-1023-(L-2)), exact (power-of-two scale of
//   an integer < 2^31), sign folded into the scale -> DADD + LOP3 + DMUL.
// Slow path (e_max <= L-2): the integer exponent-add with the reference's
// flush of e <= 0 to a signed zero (kernels_avx2.cpp:83-118 formulation,
// bit-identical to decode_one).
template <int L>
struct BlockDecoder {
    uint32_t scale_hi;  // high word of 2^(e_max-1023-(L-2)) (fast path)
    int adj;            // e_max - 1023 - (L-2)
    bool fast;
    __device__ __forceinline__ explicit BlockDecoder(uint32_t e_max) {
        adj = static_cast<int>(e_max) - 1023 - (L - 2);
        fast = static_cast<int>(e_max) > L - 2;
        scale_hi = static_cast<uint32_t>(static_cast<int>(e_max) - (L - 2)) << 20;
    }
    // code: L-bit code in the low bits of a u32 (sign at bit L-1).
    __device__ __forceinline__ double operator()(uint32_t code) const {
        constexpr uint32_t kMagMask = (L == 32) ? 0x7FFFFFFFu : ((1u << (L - 1)) - 1u);
        const uint32_t mag = code & kMagMask;
        const uint32_t sbit = (code >> (L - 1)) << 31;
        const double dm = u32_to_f64(mag);
        if (fast) {
            return __dmul_rn(dm, __hiloint2double(static_cast<int>(scale_hi | sbit), 0));
        }
        const int hi = __double2hiint(dm);
        const int lo = __double2loint(dm);
        const int field = (hi >> 20) + adj;
        const bool keep = (mag != 0u) && (field > 0);
        const int hi2 = keep ? (hi + static_cast<int>(static_cast<uint32_t>(adj) << 20)) : 0;
        return __hiloint2double(hi2 | static_cast<int>(sbit), keep ? lo : 0);
    }
};

// -------------------------------------------- device-side solver decisions
// The re-orthogonalisation test of arnoldi_orthogonalize (gmres.cpp:51):
// h_next < eta * omega with h_next = sqrt(hn1), omega = sqrt(omega2). IEEE
// sqrt and multiply on the device give the same bits as the host's test, so
// kernels gated on it run exactly when the reference would run the pass.
struct GateArg {
    const double* hn1 = nullptr;     // ||w||^2 after the first CGS pass
    const double* omega2 = nullptr;  // ||w||^2 before orthogonalisation
    double eta = 0.0;
    __device__ __forceinline__ bool open() const {
        return hn1 == nullptr || sqrt(*hn1) < eta * sqrt(*omega2);
    }
};

// Scale applied by the basis writer: none (src == nullptr), *src (mode 0),
// 1/sqrt(*src) (mode 1: scale(1.0 / h_next, w) with h_next = sqrt(||w||^2)),
// or 1/sqrt(gate.open() ? src[1] : src[0]) (mode 2: h_next of whichever CGS
// pass ran last).
struct ScaleArg {
    const double* src = nullptr;
    int mode = 0;
    GateArg gate;
    __device__ __forceinline__ double value() const {
        if (src == nullptr) return 1.0;
        if (mode == 0) return *src;
        if (mode == 1) return 1.0 / sqrt(*src);
        return 1.0 / sqrt(gate.open() ? src[1] : src[0]);
    }
};

// ------------------------------------------------------ warp reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
    return v;
}

}  // namespace cbgx

namespace cbgx {
// Process-wide count of kernels this library launched (cbgx_launch_count).
void note_launch();
}  // namespace cbgx
#define CBGX_K(...) (::cbgx::note_launch(), __VA_ARGS__)
