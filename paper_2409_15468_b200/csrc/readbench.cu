// readbench.cu -- streaming read benchmark of a stored (compressed) vector:
// the device analogue of the reference's run_read_benchmark (bench.cpp:
// 55-152, the paper's Fig. 3). Each value of one basis column is decoded to
// binary64 in registers (the same Step<F> loaders the CGS kernels use),
// `intensity` multiply-adds are applied (buf = buf * mul + add, two
// roundings as the reference's -ffp-contract=off build), and everything is
// folded into a checksum (deterministic fixed-shape tree instead of the
// reference's sequential block order). Stored bytes over time is the
// roofline number: at intensity 1 every format should stream at the HBM
// peak unless its decode is the bottleneck.
#include <algorithm>

#include "basis.cuh"
#include "common.cuh"
#include "reduce.cuh"
#include "runtime.h"

namespace cbgx {

namespace {

constexpr int kRThreads = 256;
constexpr uint32_t kRStep = 4 * kRThreads;  // rows per block step
constexpr int kU = 4;                        // steps in flight per thread

template <int F>
__global__ void __launch_bounds__(kRThreads)
read_sweep_kernel(BasisView B, uint64_t col, uint64_t n, int intensity, double mul, double add,
                  double* __restrict__ partials, unsigned* __restrict__ ticket, double* __restrict__ out) {
    __shared__ double red[kRThreads / 32];
    const uint64_t steps = (n + kRStep - 1) / kRStep;
    double acc = 0.0;
    for (uint64_t s = blockIdx.x; s < steps; s += static_cast<uint64_t>(kU) * gridDim.x) {
        // kU steps in flight per thread
        Step<F> st[kU];
        bool live[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint64_t ss = s + static_cast<uint64_t>(u) * gridDim.x;
            live[u] = ss < steps;  // block-uniform
            if (live[u]) st[u].load(B, col, ss * kRStep + 4u * threadIdx.x);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            if (!live[u]) continue;
            const uint64_t r = (s + static_cast<uint64_t>(u) * gridDim.x) * kRStep + 4u * threadIdx.x;
            double v[4];
            st[u].decode(v);  // all lanes: rows past n are padding (decoded, not counted)
            for (int t = 0; t < intensity; ++t)
#pragma unroll
                for (int k = 0; k < 4; ++k) v[k] = __dadd_rn(__dmul_rn(v[k], mul), add);
            if (r < n) acc = __dadd_rn(acc, __dadd_rn(__dadd_rn(v[0], v[1]), __dadd_rn(v[2], v[3])));
        }
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    block_finalize(red, kRThreads / 32, 1, partials, ticket, out);
}

template <int F> struct SweepLaunch {
    static void run(const BasisView& B, uint64_t col, uint64_t n, int intensity, double mul, double add,
                    double* out, Workspace* ws, cudaStream_t st) {
        const uint64_t steps = (n + kRStep - 1) / kRStep;
        const int grid = static_cast<int>(std::max<uint64_t>(
            1, std::min<uint64_t>((steps + kU - 1) / kU, static_cast<uint64_t>(sm_count()) * 8)));
        CBGX_K(read_sweep_kernel<F><<<grid, kRThreads, 0, st>>>(B, col, n, intensity, mul, add,
                                                              ws->get_partials(grid), ws->get_counter(), out));
    }
};

}  // namespace

}  // namespace cbgx

using namespace cbgx;

extern "C" {

int cbgx_read_sweep(const cbgx_basis* V, uint64_t col, uint64_t n, int intensity, double mul, double add,
                    double* d_checksum, cbgx_workspace* ws, void* stream) {
    return guard([&] {
        if (!V || !ws || !d_checksum) throw Error(CBGX_EINVAL, "bench: null argument");
        if (col >= V->capacity) throw Error(CBGX_ERANGE, "bench: column index out of range");
        if (n > V->n || n % 32) throw Error(CBGX_EINVAL, "bench: n must be a multiple of 32 within the column");
        if (intensity < 1) throw Error(CBGX_EINVAL, "bench: intensity must be >= 1");
        const BasisView B = view_of(*V);
        cudaStream_t st = as_stream(stream);
        switch (fmt_of(*V)) {
        case kF64: SweepLaunch<kF64>::run(B, col, n, intensity, mul, add, d_checksum, ws_of(ws), st); break;
        case kF32: SweepLaunch<kF32>::run(B, col, n, intensity, mul, add, d_checksum, ws_of(ws), st); break;
        case kF16: SweepLaunch<kF16>::run(B, col, n, intensity, mul, add, d_checksum, ws_of(ws), st); break;
        case kZ16: SweepLaunch<kZ16>::run(B, col, n, intensity, mul, add, d_checksum, ws_of(ws), st); break;
        case kZ21: SweepLaunch<kZ21>::run(B, col, n, intensity, mul, add, d_checksum, ws_of(ws), st); break;
        default: SweepLaunch<kZ32>::run(B, col, n, intensity, mul, add, d_checksum, ws_of(ws), st); break;
        }
        CBGX_CUDA(cudaGetLastError());
    });
}

int cbgx_read_sweep_timed(const cbgx_basis* V, uint64_t col, uint64_t n, int intensity, double mul, double add,
                          int trials, double* best_seconds, double* checksum) {
    return guard([&] {
        if (!best_seconds || trials < 1) throw Error(CBGX_EINVAL, "bench: trials must be >= 1");
        cudaStream_t st = nullptr;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        Workspace ws;
        double* d_sum = nullptr;
        auto cleanup = [&] {
            if (d_sum) cudaFree(d_sum);
            if (e0) cudaEventDestroy(e0);
            if (e1) cudaEventDestroy(e1);
            if (st) cudaStreamDestroy(st);
        };
        try {
            CBGX_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            CBGX_CUDA(cudaEventCreate(&e0));
            CBGX_CUDA(cudaEventCreate(&e1));
            CBGX_CUDA(cudaMalloc(&d_sum, sizeof(double)));
            auto* wsh = reinterpret_cast<cbgx_workspace*>(&ws);
            const int w = cbgx_read_sweep(V, col, n, intensity, mul, add, d_sum, wsh, st);  // warm-up
            if (w != CBGX_OK) throw Error(w, cbgx_last_error());
            float best = 0.0f;
            for (int t = 0; t < trials; ++t) {
                CBGX_CUDA(cudaEventRecord(e0, st));
                const int r = cbgx_read_sweep(V, col, n, intensity, mul, add, d_sum, wsh, st);
                if (r != CBGX_OK) throw Error(r, cbgx_last_error());
                CBGX_CUDA(cudaEventRecord(e1, st));
                CBGX_CUDA(cudaEventSynchronize(e1));
                float ms = 0.0f;
                CBGX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
                best = t == 0 ? ms : std::min(best, ms);
            }
            double h = 0.0;
            CBGX_CUDA(cudaMemcpyAsync(&h, d_sum, sizeof(double), cudaMemcpyDeviceToHost, st));
            CBGX_CUDA(cudaStreamSynchronize(st));
            *best_seconds = best * 1e-3;
            if (checksum) *checksum = h;
        } catch (...) {
            cleanup();
            throw;
        }
        cleanup();
    });
}

}  // extern "C"
