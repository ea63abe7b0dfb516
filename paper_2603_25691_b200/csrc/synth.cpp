// synth.cpp — seeded host generators for test and benchmark inputs (no device work).
//
// The reference draws every random input with std::mt19937_64 and libstdc++'s
// distributions (proj/tests/test_util.hpp:10-44, observations.hpp:90-121), so these entry
// points use the same standard-library engine and distributions; tests/golden/rng_golden.json
// (made by tests/golden/make_rng_golden.cpp) pins the streams bit for bit.
#include <random>
#include <unordered_map>

#include "../../include/cphifi_b200.h"

struct cphifi_rng_s {
    std::mt19937_64 eng;
    std::normal_distribution<double> normal{0.0, 1.0};
};

namespace cphifi {
void set_last_error(const std::string& m);
}

extern "C" {

int cphifi_rng_create(uint64_t seed, cphifi_rng* out) {
    if (!out) {
        cphifi::set_last_error("cphifi_rng_create: null argument");
        return CPHIFI_INVALID_ARGUMENT;
    }
    *out = new cphifi_rng_s{std::mt19937_64(seed)};
    return CPHIFI_OK;
}

int cphifi_rng_destroy(cphifi_rng rng) {
    delete rng;
    return CPHIFI_OK;
}

int cphifi_rng_next_u64(cphifi_rng rng, uint64_t* out, int64_t count) {
    if (!rng || (count > 0 && !out)) return CPHIFI_INVALID_ARGUMENT;
    for (int64_t i = 0; i < count; ++i) out[i] = rng->eng();
    return CPHIFI_OK;
}

int cphifi_rng_uniform_real(cphifi_rng rng, double lo, double hi, double* out, int64_t count) {
    if (!rng || (count > 0 && !out)) return CPHIFI_INVALID_ARGUMENT;
    std::uniform_real_distribution<double> dist(lo, hi);
    for (int64_t i = 0; i < count; ++i) out[i] = dist(rng->eng);
    return CPHIFI_OK;
}

int cphifi_rng_uniform_int(cphifi_rng rng, int64_t lo, int64_t hi, int64_t* out, int64_t count) {
    if (!rng || (count > 0 && !out) || lo > hi) return CPHIFI_INVALID_ARGUMENT;
    for (int64_t i = 0; i < count; ++i) {
        std::uniform_int_distribution<long long> dist(lo, hi);
        out[i] = dist(rng->eng);
    }
    return CPHIFI_OK;
}

int cphifi_rng_normal(cphifi_rng rng, double mean, double stddev, double* out, int64_t count) {
    if (!rng || (count > 0 && !out)) return CPHIFI_INVALID_ARGUMENT;
    const std::normal_distribution<double>::param_type p(mean, stddev);
    for (int64_t i = 0; i < count; ++i) out[i] = rng->normal(rng->eng, p);
    return CPHIFI_OK;
}

int cphifi_rng_normal_reset(cphifi_rng rng) {
    if (!rng) return CPHIFI_INVALID_ARGUMENT;
    rng->normal.reset();
    return CPHIFI_OK;
}

// observations.hpp:90-107: partial Fisher-Yates over [0, N) with a sparse remap.
int cphifi_sample_uniform_linear(int64_t n_total, int64_t q, uint64_t seed, int64_t* picked) {
    if (q > n_total) {
        cphifi::set_last_error("sample_uniform: q exceeds tensor size");
        return CPHIFI_INVALID_ARGUMENT;
    }
    if (q > 0 && !picked) return CPHIFI_INVALID_ARGUMENT;
    std::mt19937_64 rng(seed);
    std::unordered_map<int64_t, int64_t> remap;
    remap.reserve((size_t)(2 * q));
    for (int64_t i = 0; i < q; ++i) {
        std::uniform_int_distribution<long long> dist(i, n_total - 1);
        const int64_t j = dist(rng);
        const auto fj = remap.find(j);
        const int64_t vj = fj == remap.end() ? j : fj->second;
        const auto fi = remap.find(i);
        const int64_t vi = fi == remap.end() ? i : fi->second;
        remap[j] = vi;
        picked[i] = vj;
    }
    return CPHIFI_OK;
}

}  // extern "C"
