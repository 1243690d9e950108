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

#include "basis.cuh"
#include "codec.cuh"
#include "common.cuh"
#include "reduce.cuh"
#include "runtime.h"

namespace cbgx {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kSteps = 4;                          // 4-row steps per thread per tile
constexpr uint64_t kTileRows = 4ull * kThreads * kSteps;  // 4096
static_assert(kRowAlign % kTileRows == 0, "tiles must divide the basis row padding");

__device__ __forceinline__ void load_w(const double* __restrict__ w, uint64_t n, uint64_t r,
                                       double out[4]) {
    if (r + 3 < n) {
        const double2 a = __ldg(reinterpret_cast<const double2*>(w + r));
        const double2 b = __ldg(reinterpret_cast<const double2*>(w + r + 2));
        out[0] = a.x; out[1] = a.y; out[2] = b.x; out[3] = b.y;
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) out[k] = r + k < n ? w[r + k] : 0.0;
    }
}

// ------------------------------------------------------------------ dot
template <int F>
__global__ void __launch_bounds__(kThreads, 2)
cgs_dot_kernel(BasisView B, uint64_t first, uint32_t cols, const double* __restrict__ w,
               int with_wnorm, double* __restrict__ partials, unsigned* __restrict__ ticket,
               double* __restrict__ h_out) {
    extern __shared__ double red[];  // [kWarps][cols + 1]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t ncol = cols + (with_wnorm ? 1 : 0);
    for (uint32_t k = threadIdx.x; k < kWarps * ncol; k += kThreads) red[k] = 0.0;
    __syncthreads();

    const uint64_t ntiles = (B.n + kTileRows - 1) / kTileRows;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t r0 = tile * kTileRows + 4ull * threadIdx.x;
        double wv[kSteps][4];
#pragma unroll
        for (int s = 0; s < kSteps; ++s) load_w(w, B.n, r0 + s * 4ull * kThreads, wv[s]);
        if (with_wnorm) {
            double acc = 0.0;
#pragma unroll
            for (int s = 0; s < kSteps; ++s)
#pragma unroll
                for (int k = 0; k < 4; ++k) acc = __dadd_rn(acc, __dmul_rn(wv[s][k], wv[s][k]));
            acc = warp_sum(acc);
            if (lane == 0) red[warp * ncol + cols] += acc;
        }
        Step<F> buf[2][kSteps];
        if (cols > 0) {
#pragma unroll
            for (int s = 0; s < kSteps; ++s) buf[0][s].load(B, first, r0 + s * 4ull * kThreads);
        }
        for (uint32_t j = 0; j < cols; j += 2) {
            // even column in buf[0]; prefetch odd column into buf[1]
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const uint32_t jj = j + half;
                if (jj >= cols) break;
                if (jj + 1 < cols) {
#pragma unroll
                    for (int s = 0; s < kSteps; ++s)
                        buf[half ^ 1][s].load(B, first + jj + 1, r0 + s * 4ull * kThreads);
                }
                double acc = buf[half][0].dot(wv[0]);
#pragma unroll
                for (int s = 1; s < kSteps; ++s) acc = __dadd_rn(acc, buf[half][s].dot(wv[s]));
                acc = warp_sum(acc);
                if (lane == 0) red[warp * ncol + jj] += acc;
            }
        }
    }
    __syncthreads();
    block_finalize(red, kWarps, ncol, partials, ticket, h_out);
}

// --------------------------------------------------------------- update
template <int F>
__global__ void __launch_bounds__(kThreads, 2)
cgs_update_kernel(BasisView B, uint64_t first, uint32_t cols, const double* __restrict__ h,
                  double h_sign, double* __restrict__ w, int with_norm,
                  double* __restrict__ partials, unsigned* __restrict__ ticket,
                  double* __restrict__ norm_out) {
    extern __shared__ double sh[];  // [cols] coefficients, then [kWarps] norm partials
    double* hs = sh;
    double* red = sh + cols;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (uint32_t k = threadIdx.x; k < cols; k += kThreads) hs[k] = h_sign * h[k];
    if (threadIdx.x < kWarps) red[threadIdx.x] = 0.0;
    __syncthreads();

    const uint64_t ntiles = (B.n + kTileRows - 1) / kTileRows;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t r0 = tile * kTileRows + 4ull * threadIdx.x;
        double wv[kSteps][4];
#pragma unroll
        for (int s = 0; s < kSteps; ++s) load_w(w, B.n, r0 + s * 4ull * kThreads, wv[s]);
        Step<F> buf[2][kSteps];
        if (cols > 0) {
#pragma unroll
            for (int s = 0; s < kSteps; ++s) buf[0][s].load(B, first, r0 + s * 4ull * kThreads);
        }
        for (uint32_t j = 0; j < cols; j += 2) {
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const uint32_t jj = j + half;
                if (jj >= cols) break;
                if (jj + 1 < cols) {
#pragma unroll
                    for (int s = 0; s < kSteps; ++s)
                        buf[half ^ 1][s].load(B, first + jj + 1, r0 + s * 4ull * kThreads);
                }
                const double hj = hs[jj];
                const int he = static_cast<int>(exp_field(hj));
#pragma unroll
                for (int s = 0; s < kSteps; ++s) buf[half][s].update(hj, he, wv[s]);
            }
        }
        double acc = 0.0;
#pragma unroll
        for (int s = 0; s < kSteps; ++s) {
            const uint64_t r = r0 + s * 4ull * kThreads;
            if (r + 3 < B.n) {
                reinterpret_cast<double2*>(w + r)[0] = make_double2(wv[s][0], wv[s][1]);
                reinterpret_cast<double2*>(w + r)[1] = make_double2(wv[s][2], wv[s][3]);
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (r + k < B.n) w[r + k] = wv[s][k];
            }
            if (with_norm) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (r + k < B.n) acc = __dadd_rn(acc, __dmul_rn(wv[s][k], wv[s][k]));
            }
        }
        if (with_norm) {
            acc = warp_sum(acc);
            if (lane == 0) red[warp] += acc;
        }
    }
    __syncthreads();
    if (with_norm) block_finalize(red, kWarps, 1, partials, ticket, norm_out);
}

// ------------------------------------------------- reference-order dot
// One thread per column, the exact order of KrylovBasis::dot: per 32-block
// partial from +0.0 left to right, then a running total over blocks
// (basis.cpp:176-186). Thread `cols` (if with_wnorm) does norm2's
// sequential <w,w> (sparse.cpp:62-66).
template <int F>
__global__ void serial_dot_kernel(BasisView B, uint64_t first, uint32_t cols,
                                  const double* __restrict__ w, int with_wnorm,
                                  double* __restrict__ h_out) {
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
                                   uint64_t n, uint64_t n_pad, const double* __restrict__ scale_src,
                                   int scale_mode, double* __restrict__ v_out) {
    double s = 1.0;
    if (scale_src) {
        const double p = *scale_src;
        s = scale_mode == 1 ? 1.0 / sqrt(p) : p;
    }
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n_pad;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        double v = 0.0;
        if (i < n) {
            v = x[i];
            if (scale_src) v = __dmul_rn(v, s);
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

int persistent_grid(uint64_t tiles) {
    const uint64_t cap = static_cast<uint64_t>(sm_count()) * 2;
    return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(tiles, cap)));
}

template <int F> struct DotLaunch {
    static void run(const BasisView& B, uint64_t first, uint32_t cols, const double* w, int wn,
                    int reduction, double* h, Workspace* ws, cudaStream_t st) {
        const uint32_t ncol = cols + (wn ? 1 : 0);
        if (ncol == 0) return;
        if (reduction == CBGX_REDUCE_REFERENCE) {
            const uint32_t threads = ncol;
            serial_dot_kernel<F><<<(threads + 63) / 64, 64, 0, st>>>(B, first, cols, w, wn, h);
            return;
        }
        const int grid = persistent_grid((B.n + kTileRows - 1) / kTileRows);
        const size_t smem = sizeof(double) * kWarps * ncol;
        if (smem > 48 * 1024) {
            CBGX_CUDA(cudaFuncSetAttribute(cgs_dot_kernel<F>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(smem)));
        }
        double* partials = ws->get_partials(static_cast<size_t>(grid) * ncol);
        cgs_dot_kernel<F><<<grid, kThreads, smem, st>>>(B, first, cols, w, wn, partials,
                                                        ws->get_counter(), h);
    }
};

template <int F> struct UpdateLaunch {
    static void run(const BasisView& B, uint64_t first, uint32_t cols, const double* h, double sign,
                    double* w, double* norm, int reduction, Workspace* ws, cudaStream_t st) {
        const int grid = persistent_grid((B.n + kTileRows - 1) / kTileRows);
        const bool fused_norm = norm && reduction == CBGX_REDUCE_TREE;
        if (cols > 0 || fused_norm) {
            const size_t smem = sizeof(double) * (cols + kWarps);
            if (smem > 48 * 1024) {
                CBGX_CUDA(cudaFuncSetAttribute(cgs_update_kernel<F>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem)));
            }
            double* partials = fused_norm ? ws->get_partials(grid) : nullptr;
            cgs_update_kernel<F><<<grid, kThreads, smem, st>>>(B, first, cols, h, sign, w, fused_norm,
                                                               partials, ws->get_counter(), norm);
        }
        if (norm && !fused_norm) launch_dot(w, w, B.n, CBGX_REDUCE_REFERENCE, norm, ws, st);
    }
};

template <int F> struct WriteLaunch {
    static void run(const cbgx_basis& V, uint64_t j, const double* x, const double* scale_src,
                    int scale_mode, double* v_out, uint64_t* bad, cudaStream_t st) {
        unsigned char* col = static_cast<unsigned char*>(V.d_data) + j * V.col_stride_bytes;
        if constexpr (FmtInfo<F>::frsz) {
            launch_compress(x, V.n, V.n_pad / 32, 32, FmtInfo<F>::L,
                            V.d_exp + j * V.exp_col_stride, reinterpret_cast<uint32_t*>(col),
                            scale_src, scale_mode, v_out, bad, st);
        } else {
            const uint64_t blocks = std::min<uint64_t>((V.n_pad + 255) / 256, static_cast<uint64_t>(sm_count()) * 16);
            write_plain_kernel<F><<<static_cast<int>(std::max<uint64_t>(blocks, 1)), 256, 0, st>>>(
                col, x, V.n, V.n_pad, scale_src, scale_mode, v_out);
        }
    }
};

template <int F> struct ReadLaunch {
    static void run(const BasisView& B, uint64_t j, uint64_t first, uint64_t count, double* out,
                    cudaStream_t st) {
        const uint64_t blocks = std::min<uint64_t>((count + 255) / 256, static_cast<uint64_t>(sm_count()) * 16);
        read_kernel<F><<<static_cast<int>(std::max<uint64_t>(blocks, 1)), 256, 0, st>>>(B, j, first, count, out);
    }
};

void check_basis(const cbgx_basis* V) {
    if (!V) throw Error(CBGX_EINVAL, "basis: null descriptor");
    if (V->n_pad < V->n || V->n_pad % kRowAlign) throw Error(CBGX_EINVAL, "basis: bad row padding");
    (void)fmt_of(*V);
}

}  // namespace

void launch_cgs_dot(const cbgx_basis& V, uint64_t first, uint32_t cols, const double* w, int wn,
                    int reduction, double* h, Workspace* ws, cudaStream_t st) {
    if (first + cols > V.capacity) throw Error(CBGX_ERANGE, "basis: column index out of range");
    dispatch_fmt<DotLaunch>(fmt_of(V), view_of(V), first, cols, w, wn, reduction, h, ws, st);
    CBGX_CUDA(cudaGetLastError());
}

void launch_cgs_update(const cbgx_basis& V, uint64_t first, uint32_t cols, const double* h,
                       double sign, double* w, double* norm, int reduction, Workspace* ws,
                       cudaStream_t st) {
    if (first + cols > V.capacity) throw Error(CBGX_ERANGE, "basis: column index out of range");
    dispatch_fmt<UpdateLaunch>(fmt_of(V), view_of(V), first, cols, h, sign, w, norm, reduction, ws, st);
    CBGX_CUDA(cudaGetLastError());
}

void launch_basis_write(const cbgx_basis& V, uint64_t j, const double* x, const double* scale_src,
                        int scale_mode, double* v_out, uint64_t* bad, cudaStream_t st) {
    if (j >= V.capacity) throw Error(CBGX_ERANGE, "basis: cannot write column");
    dispatch_fmt<WriteLaunch>(fmt_of(V), V, j, x, scale_src, scale_mode, v_out, bad, st);
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
        uint64_t col_bytes = 0, exp_words = 0;
        switch (f) {
        case kF64: col_bytes = B.n_pad * 8; break;
        case kF32: col_bytes = B.n_pad * 4; break;
        case kF16: col_bytes = B.n_pad * 2; break;
        default:
            col_bytes = B.n_pad / 32 * l * 4;
            exp_words = B.n_pad / 32;
        }
        B.col_stride_bytes = col_bytes;
        B.exp_col_stride = exp_words;
        *out = B;
        // +64 B slack: the l=21 step loader reads up to 3 words past a
        // block's last word.
        if (data_bytes) *data_bytes = col_bytes * capacity + 64;
        if (exp_bytes) *exp_bytes = exp_words * capacity * 4;
    });
}

int cbgx_basis_write(const cbgx_basis* V, uint64_t j, const double* d_x, const double* d_scale_src,
                     int scale_mode, double* d_v_out, uint64_t* d_bad_index, void* stream) {
    return guard([&] {
        check_basis(V);
        launch_basis_write(*V, j, d_x, d_scale_src, scale_mode, d_v_out, d_bad_index, as_stream(stream));
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

}  // extern "C"
