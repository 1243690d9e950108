// stdrng.cpp -- TEST INFRASTRUCTURE ONLY.
// Reproduces the reference tests' input generators bit-for-bit: they draw
// from libstdc++'s std::mt19937_64 + std::uniform_real_distribution /
// uniform_int_distribution (acceptance.cpp:60-68, test_kernels.cpp:26-41,
// SURVEY 8(c) golden input), whose exact algorithms are library specific.
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <random>

extern "C" {

// uniform_values(n, seed) of acceptance.cpp:60-68 with bounds [lo, hi)
void rng_uniform(uint64_t seed, double lo, double hi, double* out, size_t n) {
    std::mt19937_64 g(seed);
    std::uniform_real_distribution<double> d(lo, hi);
    for (size_t i = 0; i < n; ++i) out[i] = d(g);
}

// mixed_values(n, seed) of test_kernels.cpp:26-41
void rng_mixed(uint64_t seed, double* out, size_t n) {
    std::mt19937_64 g(seed);
    std::uniform_real_distribution<double> uni(-1.0, 1.0);
    std::uniform_int_distribution<int> ex(-1020, 1020);
    for (size_t i = 0; i < n; ++i) {
        switch (i % 7) {
        case 0: out[i] = 0.0; break;
        case 1: out[i] = -0.0; break;
        case 2: out[i] = 5e-321; break;
        case 3: out[i] = std::ldexp(uni(g), ex(g) / 4); break;
        default: out[i] = uni(g); break;
        }
    }
}

// wide-exponent vector ldexp(u, U{lo_e..hi_e})
void rng_wide(uint64_t seed, int lo_e, int hi_e, double* out, size_t n) {
    std::mt19937_64 g(seed);
    std::uniform_real_distribution<double> uni(-1.0, 1.0);
    std::uniform_int_distribution<int> ex(lo_e, hi_e);
    for (size_t i = 0; i < n; ++i) out[i] = std::ldexp(uni(g), ex(g));
}

}
