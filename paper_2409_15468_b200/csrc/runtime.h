// runtime.h -- host-side runtime objects shared by the kernels' launchers.
#pragma once

#include <cstddef>
#include <cstdint>

#include "cbgx.h"

namespace cbgx {

// Deterministic two-stage reductions: every reducing kernel writes one
// partial row per CTA into `partials`; the last CTA to finish (ticket from
// a device counter) sums the rows in CTA order and resets the counter.
struct Workspace {
    // [0, 16): reduction tickets; kFusedBar, kFusedBar + 32: the fused
    // kernel's alternating grid-barrier counters; kFusedGate: its last gate.
    static constexpr int kFusedBar = 32;
    static constexpr int kFusedGate = 96;
    static constexpr int kCounters = 128;
    uint64_t fused_launches = 0;
    int device = 0;
    double* partials = nullptr;
    size_t partial_cap = 0;
    unsigned* counters = nullptr;
    // fused kernel: two alternating sets of fixed-point grid accumulators
    // (zero-initialised; each launch zeroes the set the next one uses)
    unsigned long long* fx = nullptr;
    size_t fx_words = 0;  // per set
    // per-CTA omega^2 partials of the SpMV that feeds the fused kernel
    // (summed by every fused CTA; separate from `partials`, which the fused
    // kernel's grid reductions use)
    double* omega_parts = nullptr;
    size_t omega_cap = 0;
    double* get_partials(size_t doubles);
    double* get_omega_parts(size_t doubles);
    unsigned* get_counter();
    unsigned long long* get_fx(size_t words_per_set);
    ~Workspace();
};

inline Workspace* ws_of(cbgx_workspace* w) { return reinterpret_cast<Workspace*>(w); }

}  // namespace cbgx
