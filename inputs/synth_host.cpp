// synth_host.cpp — seeded host generators for test and benchmark inputs (libcphifi_inputs.so).
//
// Used by the product tests, the oracle tests, bench.py's two arms and the fixture scripts, so
// that the reference arm and the oracle never load the product library.  Nothing here is part of
// the solver path.
//  - std::mt19937_64 with libstdc++'s uniform_real / uniform_int / normal distributions: the
//    reference draws every random input with them (proj/tests/test_util.hpp:10-44); pinned bit for
//    bit by tests/golden/rng_golden.json (made by tests/golden/make_rng_golden.cpp with the real
//    libstdc++).
//  - sample_uniform's index draw (observations.hpp:90-121): partial Fisher-Yates over [0, N) with
//    a sparse remap (the reference's algorithm, restated).
//  - the counter-based observation generator of configs 3 and 4 (synth_math.h), for any range of
//    draw counters [l0, l1), on all host threads — bit-identical to the device generator.
// Built with -ffp-contract=off (inputs/Makefile): synth_math.h relies on uncontracted arithmetic.
#include <cmath>
#include <random>
#include <unordered_map>
#include <vector>

#include "synth_math.h"

struct inp_rng_s {
    std::mt19937_64 eng;
    std::normal_distribution<double> normal{0.0, 1.0};
};

extern "C" {

int inp_rng_create(uint64_t seed, inp_rng_s** out) {
    if (!out) return 1;
    *out = new inp_rng_s{std::mt19937_64(seed)};
    return 0;
}

void inp_rng_destroy(inp_rng_s* rng) { delete rng; }

int inp_rng_next_u64(inp_rng_s* rng, uint64_t* out, int64_t count) {
    if (!rng || (count > 0 && !out)) return 1;
    for (int64_t i = 0; i < count; ++i) out[i] = rng->eng();
    return 0;
}

int inp_rng_uniform_real(inp_rng_s* rng, double lo, double hi, double* out, int64_t count) {
    if (!rng || (count > 0 && !out)) return 1;
    std::uniform_real_distribution<double> dist(lo, hi);
    for (int64_t i = 0; i < count; ++i) out[i] = dist(rng->eng);
    return 0;
}

int inp_rng_uniform_int(inp_rng_s* rng, int64_t lo, int64_t hi, int64_t* out, int64_t count) {
    if (!rng || (count > 0 && !out) || lo > hi) return 1;
    for (int64_t i = 0; i < count; ++i) {
        std::uniform_int_distribution<long long> dist(lo, hi);  // one distribution per draw, as the tests do
        out[i] = dist(rng->eng);
    }
    return 0;
}

int inp_rng_normal(inp_rng_s* rng, double mean, double stddev, double* out, int64_t count) {
    if (!rng || (count > 0 && !out)) return 1;
    const std::normal_distribution<double>::param_type p(mean, stddev);
    for (int64_t i = 0; i < count; ++i) out[i] = rng->normal(rng->eng, p);
    return 0;
}

int inp_rng_normal_reset(inp_rng_s* rng) {
    if (!rng) return 1;
    rng->normal.reset();
    return 0;
}

// observations.hpp:90-107 (index part): q distinct linear indices of [0, n_total).
int inp_sample_uniform_linear(int64_t n_total, int64_t q, uint64_t seed, int64_t* picked) {
    if (q > n_total || q < 0) return 1;  // "sample_uniform: q exceeds tensor size"
    if (q > 0 && !picked) return 1;
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
    return 0;
}

// Zipf CDF of mode size n, P(i) ~ (i+1)^-s; last entry forced to 1.  The device generator
// uploads exactly this table (k_synth.cu includes synth_math.h and calls inp-equivalent code).
void inp_zipf_cdf(int64_t n, double s, double* cdf) {
    double tot = 0.0;
    for (int64_t i = 0; i < n; ++i) tot += std::pow((double)(i + 1), -s);
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        acc += std::pow((double)(i + 1), -s);
        cdf[i] = acc / tot;
    }
    cdf[n - 1] = 1.0;
}

// Draws [l0, l1) of the counter-based generator.  idx_out: d columns of (l1 - l0) int32 (column m
// at idx_out + m * (l1 - l0)); vals_out: l1 - l0 doubles (NULL: indices only).  factors[m] is
// n_m x r column-major.  zipf_mode < 0: every mode uniform.
int inp_synth_observations(int d, const int64_t* shape, int64_t l0, int64_t l1, uint64_t seed, int zipf_mode,
                           double zipf_s, int64_t r, const double* const* factors, double noise_std,
                           int32_t* idx_out, double* vals_out, int threads) {
    if (d < 1 || d > 8 || l1 < l0 || !shape || !idx_out) return 1;
    if (vals_out && !factors) return 1;
    std::vector<double> cdf;
    if (zipf_mode >= 0) {
        cdf.resize((size_t)shape[zipf_mode]);
        inp_zipf_cdf(shape[zipf_mode], zipf_s, cdf.data());
    }
    const int64_t cnt = l1 - l0;
    if (threads < 1) threads = 1;
#pragma omp parallel for schedule(static) num_threads(threads)
    for (int64_t t = 0; t < cnt; ++t) {
        const uint64_t l = (uint64_t)(l0 + t);
        int64_t ix[8];
        for (int m = 0; m < d; ++m) {
            const uint64_t u = syn_draw(seed, l, (uint64_t)m);
            ix[m] = m == zipf_mode ? syn_zipf_index(u, cdf.data(), shape[m]) : syn_uniform_index(u, shape[m]);
            idx_out[(int64_t)m * cnt + t] = (int32_t)ix[m];
        }
        if (vals_out) {
            double v = 0.0;
            for (int64_t j = 0; j < r; ++j) {
                double p = factors[0][ix[0] + shape[0] * j];
                for (int m = 1; m < d; ++m) p = SYN_MUL(p, factors[m][ix[m] + shape[m] * j]);
                v = SYN_ADD(v, p);
            }
            vals_out[t] = SYN_ADD(v, SYN_MUL(noise_std, syn_normal(seed, l)));
        }
    }
    return 0;
}

// Test hooks for the deterministic transcendental pieces.
double inp_syn_log(double x) { return syn_log(x); }
double inp_syn_cos2pi(double f) { return syn_cos2pi(f); }

}  // extern "C"
