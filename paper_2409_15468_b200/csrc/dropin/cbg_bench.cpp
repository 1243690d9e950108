// cbg_bench.cpp -- run_read_benchmark (bench.hpp) over the device read sweep
// (cbgx_read_sweep_timed). Input data and the runtime multiply/add constants
// come from the same std::mt19937_64 stream as the reference
// (bench.cpp:121-131), so every format stores the same values.
#include <random>
#include <stdexcept>

#include "cbg/bench.hpp"
#include "cbgx.h"

namespace cbg {

std::vector<BenchResult> run_read_benchmark(size_t elements, std::span<const StorageFormat> formats,
                                            std::span<const int> intensities, int trials, uint64_t seed) {
    constexpr size_t kBlock = KrylovBasis::kBlock;
    if (elements < kBlock) throw std::invalid_argument("bench: need at least one block");
    if (trials < 1) throw std::invalid_argument("bench: trials must be >= 1");
    for (int intensity : intensities)
        if (intensity < 1) throw std::invalid_argument("bench: intensity must be >= 1");
    const size_t n = elements / kBlock * kBlock;
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    std::vector<double> data(n);
    for (double& v : data) v = dist(rng);
    const double mul = 1.0 + dist(rng) * 1e-7;
    const double add = dist(rng) * 1e-9;
    std::vector<BenchResult> results;
    for (const StorageFormat& fmt : formats) {
        KrylovBasis basis(n, 1, fmt);
        basis.write_vector(0, data);
        const auto* desc = static_cast<const cbgx_basis*>(basis.device_descriptor());
        for (int intensity : intensities) {
            double best = 0.0, checksum = 0.0;
            if (cbgx_read_sweep_timed(desc, 0, n, intensity, mul, add, trials, &best, &checksum) != CBGX_OK)
                throw std::runtime_error(cbgx_last_error());
            BenchResult r;
            r.format = fmt.name();
            r.intensity = intensity;
            r.elements = n;
            r.stored_bytes = fmt.column_bytes(n);
            r.seconds = best;
            r.stored_gbps = static_cast<double>(r.stored_bytes) / best / 1e9;
            r.logical_gbps = static_cast<double>(n) * 8.0 / best / 1e9;
            results.push_back(std::move(r));
        }
    }
    return results;
}

}  // namespace cbg
