// Workload generation for the benchmark configs (host code; no device work).
//
// configs[1] (the CGEMM sweep) fills A then B from ONE generator seeded with
// seed + n, two uniform_pm1f draws per complex element, row-major
// (experiments.cpp:76-83 random_uniform_matrix, rng.hpp:13-56).  The bench has
// to run the reference's own inputs so its device decision line can be
// compared byte for byte with the reference's on the same operands; the
// reference library itself is test infrastructure, so the generator is
// restated here.  std::mt19937_64 is fully specified by the C++ standard;
// the distribution map is the reference's hand-rolled one:
//   uniform01    = (u64 >> 11) * 2^-53
//   uniform_pm1f = float(2 * uniform01 - 1)           (one rounding to f32)
//   gaussian     = Box-Muller with a cached spare      (rng.hpp:38-50)
#include <cmath>
#include <cstdint>
#include <new>
#include <random>

#include "../../include/tcec_b200.h"

struct tcec_rng_s {
    std::mt19937_64 eng;
    double spare = 0.0;
    bool have_spare = false;
    explicit tcec_rng_s(uint64_t seed) : eng(seed) {}
    double uniform01() { return double(eng() >> 11) * 0x1.0p-53; }
    double uniform01_pos() { return double((eng() >> 11) + 1) * 0x1.0p-53; }
};

extern "C" {

int tcec_rng_create(uint64_t seed, tcec_rng* out) {
    if (!out) return TCEC_ERR_INVALID_ARGUMENT;
    *out = new (std::nothrow) tcec_rng_s(seed);
    return *out ? TCEC_OK : TCEC_ERR_INVALID_ARGUMENT;
}

int tcec_rng_destroy(tcec_rng r) {
    delete r;
    return TCEC_OK;
}

uint64_t tcec_rng_next_u64(tcec_rng r) { return r->eng(); }

int tcec_rng_fill_uniform_pm1f(tcec_rng r, float* dst, int64_t n) {
    if (!r || (n > 0 && !dst)) return TCEC_ERR_INVALID_ARGUMENT;
    for (int64_t i = 0; i < n; ++i) dst[i] = float(2.0 * r->uniform01() - 1.0);
    return TCEC_OK;
}

int tcec_rng_fill_gaussian(tcec_rng r, double stddev, double* dst, int64_t n) {
    if (!r || (n > 0 && !dst)) return TCEC_ERR_INVALID_ARGUMENT;
    for (int64_t i = 0; i < n; ++i) {
        if (r->have_spare) {
            r->have_spare = false;
            dst[i] = r->spare * stddev;
            continue;
        }
        const double u1 = r->uniform01_pos();
        const double u2 = r->uniform01();
        const double rad = std::sqrt(-2.0 * std::log(u1));
        const double ang = 6.283185307179586476925286766559 * u2;
        r->spare = rad * std::sin(ang);
        r->have_spare = true;
        dst[i] = rad * std::cos(ang) * stddev;
    }
    return TCEC_OK;
}

}  // extern "C"
