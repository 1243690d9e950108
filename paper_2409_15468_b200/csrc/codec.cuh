// codec.cuh -- launchers shared between the codec and the basis/solver code.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>

#include "common.cuh"

namespace cbgx {

// Encode blocks [0, nb_write) of s*x into (exps, payload); rows >= n read as
// zero. scale_src == nullptr -> s = 1 (plain compress). Fast path only for
// bs == 32 and l in {16, 21, 32}; the generic codec requires nb_write ==
// num_blocks(n) and no scale. erange (fast path only): also fold the written
// blocks' exponent range into erange[0..1] (max of 2047 - e over nonzero
// blocks, max e; the caller zeroes it first -- cbgx_basis.d_erange).
void launch_compress(const double* x, uint64_t n, uint64_t nb_write, uint32_t bs, uint32_t l,
                     uint32_t* exps, uint32_t* payload, const ScaleArg& scale, double* v_out,
                     uint64_t* bad, cudaStream_t st, uint32_t* erange = nullptr);
void launch_decompress(const uint32_t* exps, const uint32_t* payload, uint64_t n, uint32_t bs,
                       uint32_t l, uint64_t first, uint64_t count, double* out, cudaStream_t st);
// Runs body(d_bad) with a fresh UINT64_MAX-initialised device u64, syncs and
// returns its value.
uint64_t sync_bad_index(const std::function<void(uint64_t*)>& body, cudaStream_t st);
[[noreturn]] void throw_non_finite(uint64_t index);

}  // namespace cbgx
