// runtime.cu -- error state, device queries and reduction workspaces for the
// C-ABI (include/cbgx.h).
#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"
#include "runtime.h"

namespace cbgx {

namespace {
std::atomic<uint64_t> g_launches{0};
thread_local std::string t_msg;
thread_local uint64_t t_index = 0;
}  // namespace

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(int code, const std::string& msg, uint64_t index) {
    (void)code;
    t_msg = msg;
    t_index = index;
}

void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        throw Error(CBGX_ECUDA, std::string("cuda: ") + cudaGetErrorString(e) + " (" + what + ")");
    }
}

int current_device() {
    int d = 0;
    CBGX_CUDA(cudaGetDevice(&d));
    return d;
}

int sm_count() {
    static int cache[64] = {0};
    const int d = current_device();
    if (d < 64 && cache[d]) return cache[d];
    int v = 0;
    CBGX_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d));
    if (d < 64) cache[d] = v;
    return v;
}

Workspace::~Workspace() {
    if (partials) cudaFree(partials);
    if (counters) cudaFree(counters);
    if (fx) cudaFree(fx);
    if (omega_parts) cudaFree(omega_parts);
}

unsigned long long* Workspace::get_fx(size_t words_per_set) {
    if (words_per_set > fx_words) {
        // a grown buffer starts zeroed (both sets): the launch sequence's
        // invariant (the set a launch uses is zero) holds from here on
        if (fx) CBGX_CUDA(cudaFree(fx));
        fx = nullptr;
        CBGX_CUDA(cudaMalloc(&fx, 2 * words_per_set * sizeof(unsigned long long)));
        CBGX_CUDA(cudaMemset(fx, 0, 2 * words_per_set * sizeof(unsigned long long)));
        CBGX_CUDA(cudaStreamSynchronize(nullptr));
        fx_words = words_per_set;
    }
    return fx;
}

double* Workspace::get_partials(size_t doubles) {
    if (doubles > partial_cap) {
        if (partials) CBGX_CUDA(cudaFree(partials));
        partials = nullptr;
        size_t cap = partial_cap ? partial_cap : 1024;
        while (cap < doubles) cap *= 2;
        CBGX_CUDA(cudaMalloc(&partials, cap * sizeof(double)));
        partial_cap = cap;
    }
    return partials;
}

double* Workspace::get_omega_parts(size_t doubles) {
    if (doubles > omega_cap) {
        if (omega_parts) CBGX_CUDA(cudaFree(omega_parts));
        omega_parts = nullptr;
        CBGX_CUDA(cudaMalloc(&omega_parts, doubles * sizeof(double)));
        omega_cap = doubles;
    }
    return omega_parts;
}

unsigned* Workspace::get_counter() {
    if (!counters) {
        CBGX_CUDA(cudaMalloc(&counters, kCounters * sizeof(unsigned)));
        CBGX_CUDA(cudaMemset(counters, 0, kCounters * sizeof(unsigned)));
        CBGX_CUDA(cudaStreamSynchronize(nullptr));  // users may launch on non-blocking streams
    }
    return counters;
}

}  // namespace cbgx

using namespace cbgx;

extern "C" {

const char* cbgx_last_error(void) { return t_msg.c_str(); }
uint64_t cbgx_last_error_index(void) { return t_index; }
int cbgx_version(void) { return 1; }
uint64_t cbgx_launch_count(void) { return g_launches.load(); }

int cbgx_set_device(int device) {
    return guard([&] { CBGX_CUDA(cudaSetDevice(device)); });
}

int cbgx_malloc(void** d_ptr, uint64_t bytes) {
    return guard([&] {
        if (!d_ptr) throw Error(CBGX_EINVAL, "malloc: null output");
        *d_ptr = nullptr;
        CBGX_CUDA(cudaMalloc(d_ptr, bytes ? bytes : 8));
    });
}

int cbgx_free(void* d_ptr) {
    return guard([&] {
        if (d_ptr) CBGX_CUDA(cudaFree(d_ptr));
    });
}

int cbgx_memcpy(void* dst, const void* src, uint64_t bytes, int kind) {
    return guard([&] {
        if (!bytes) return;
        const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice
                                 : kind == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
        CBGX_CUDA(cudaMemcpy(dst, src, bytes, k));
    });
}

int cbgx_memset(void* d_ptr, int value, uint64_t bytes) {
    return guard([&] {
        if (bytes) {
            CBGX_CUDA(cudaMemset(d_ptr, value, bytes));
            CBGX_CUDA(cudaStreamSynchronize(nullptr));  // complete before any stream uses it
        }
    });
}

int cbgx_device_info(int* device, int* sms, int64_t* l2) {
    return guard([&] {
        int d = current_device();
        if (device) *device = d;
        if (sms) *sms = sm_count();
        if (l2) {
            int v = 0;
            CBGX_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, d));
            *l2 = v;
        }
    });
}

int cbgx_workspace_create(cbgx_workspace** ws) {
    return guard([&] {
        if (!ws) throw Error(CBGX_EINVAL, "workspace: null output");
        auto* w = new Workspace();
        w->device = current_device();
        *ws = reinterpret_cast<cbgx_workspace*>(w);
    });
}

int cbgx_workspace_destroy(cbgx_workspace* ws) {
    return guard([&] { delete reinterpret_cast<Workspace*>(ws); });
}

}  // extern "C"
