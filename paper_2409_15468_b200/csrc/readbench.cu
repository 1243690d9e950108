// readbench.cu -- C-ABI of the streaming read benchmark of a stored
// (compressed) vector: the device analogue of the reference's
// run_read_benchmark (bench.cpp:55-152, the paper's Fig. 3). The kernel
// (read_sweep_kernel, cgs.cu) streams the column through the CGS kernels'
// bulk-copy ring and decode path; each value is decoded to binary64,
// `intensity` multiply-adds are applied (buf = buf * mul + add, two
// roundings as the reference's -ffp-contract=off build) and everything is
// folded into a checksum (deterministic fixed-shape tree instead of the
// reference's sequential block order). Stored bytes over time is the
// roofline number.
#include <algorithm>

#include "basis.cuh"
#include "common.cuh"
#include "reduce.cuh"
#include "runtime.h"

using namespace cbgx;

extern "C" {

int cbgx_read_sweep(const cbgx_basis* V, uint64_t col, uint64_t n, int intensity, double mul, double add,
                    double* d_checksum, cbgx_workspace* ws, void* stream) {
    return guard([&] {
        if (!V || !ws || !d_checksum) throw Error(CBGX_EINVAL, "bench: null argument");
        if (col >= V->capacity) throw Error(CBGX_ERANGE, "bench: column index out of range");
        if (n > V->n || n % 32) throw Error(CBGX_EINVAL, "bench: n must be a multiple of 32 within the column");
        if (intensity < 1) throw Error(CBGX_EINVAL, "bench: intensity must be >= 1");
        launch_read_sweep(*V, col, n, intensity, mul, add, d_checksum, ws_of(ws), as_stream(stream));
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
