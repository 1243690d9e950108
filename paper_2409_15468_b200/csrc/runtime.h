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
    static constexpr int kCounters = 16;
    int device = 0;
    double* partials = nullptr;
    size_t partial_cap = 0;
    unsigned* counters = nullptr;
    double* get_partials(size_t doubles);
    unsigned* get_counter();
    ~Workspace();
};

inline Workspace* ws_of(cbgx_workspace* w) { return reinterpret_cast<Workspace*>(w); }

}  // namespace cbgx
