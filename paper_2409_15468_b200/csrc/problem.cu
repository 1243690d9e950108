// problem.cu -- host-side problem setup: the sin right-hand side of
// generate_problem (sparse.cpp:233-247). The values must come from the C
// library sin and a strictly sequential norm for bit parity with the
// reference (CUDA's device sin is a <= 2 ulp approximation), so this runs
// on the host, sin in parallel chunks and the norm in order.
#include <algorithm>
#include <cmath>
#include <thread>
#include <vector>

#include "common.cuh"

using namespace cbgx;

extern "C" int cbgx_sin_solution(uint64_t n, uint64_t first, uint64_t count, double* out, int threads) {
    return guard([&] {
        if (n < 2) throw Error(CBGX_EINVAL, "generate_problem: need at least 2 unknowns");
        if (first > n || count > n - first) throw Error(CBGX_ERANGE, "sin_solution: range out of bounds");
        int T = threads > 0 ? threads : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
        const uint64_t chunk = 1ull << 22;
        std::vector<double> buf(std::min<uint64_t>(n, chunk * static_cast<uint64_t>(T)));
        double acc = 0.0;
        auto fill = [&](uint64_t base, uint64_t len) {
            std::vector<std::thread> th;
            const uint64_t per = (len + T - 1) / T;
            for (int t = 0; t < T; ++t) {
                const uint64_t a = std::min(len, per * t), b2 = std::min(len, per * (t + 1));
                th.emplace_back([&, a, b2] {
                    for (uint64_t i = a; i < b2; ++i) buf[i] = std::sin(static_cast<double>(base + i));
                });
            }
            for (auto& x : th) x.join();
        };
        // pass 1: sequential norm (sparse.cpp:62-66 order)
        for (uint64_t base = 0; base < n; base += buf.size()) {
            const uint64_t len = std::min<uint64_t>(buf.size(), n - base);
            fill(base, len);
            for (uint64_t i = 0; i < len; ++i) acc += buf[i] * buf[i];
        }
        const double inv = 1.0 / std::sqrt(acc);
        // pass 2: the requested rows, scaled like scale(1.0 / nrm, x)
        for (uint64_t base = first; base < first + count; base += buf.size()) {
            const uint64_t len = std::min<uint64_t>(buf.size(), first + count - base);
            fill(base, len);
            for (uint64_t i = 0; i < len; ++i) out[base - first + i] = buf[i] * inv;
        }
    });
}
