// Golden vectors for the reference's random-number stack, produced by the real libstdc++
// (the library the reference is built against: std::mt19937_64 with
// uniform_real_distribution / uniform_int_distribution<Eigen::Index> / normal_distribution,
// used by proj/tests/test_util.hpp:10-44 and observations.hpp:90-121).
// Build and run:  g++ -O2 -std=c++20 make_rng_golden.cpp -o /tmp/g && /tmp/g > rng_golden.json
#include <cstdint>
#include <cstdio>
#include <random>
#include <unordered_map>
#include <vector>

static void emit_u64(const char* name, const std::vector<uint64_t>& v, bool last = false) {
    std::printf("  \"%s\": [", name);
    for (size_t i = 0; i < v.size(); ++i) std::printf("%s\"%llu\"", i ? ", " : "", (unsigned long long)v[i]);
    std::printf("]%s\n", last ? "" : ",");
}
static void emit_i64(const char* name, const std::vector<long long>& v, bool last = false) {
    std::printf("  \"%s\": [", name);
    for (size_t i = 0; i < v.size(); ++i) std::printf("%s%lld", i ? ", " : "", v[i]);
    std::printf("]%s\n", last ? "" : ",");
}
static void emit_f64(const char* name, const std::vector<double>& v, bool last = false) {
    std::printf("  \"%s\": [", name);
    for (size_t i = 0; i < v.size(); ++i) std::printf("%s%.17g", i ? ", " : "", v[i]);
    std::printf("]%s\n", last ? "" : ",");
}

// Same partial Fisher-Yates contract as sample_uniform's index draw (restated, not copied).
static std::vector<long long> picked_indices(long long n_total, long long q, uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::unordered_map<long long, long long> remap;
    std::vector<long long> picked(q);
    for (long long i = 0; i < q; ++i) {
        std::uniform_int_distribution<long long> dist(i, n_total - 1);
        long long j = dist(rng);
        auto fj = remap.find(j);
        long long vj = fj == remap.end() ? j : fj->second;
        auto fi = remap.find(i);
        long long vi = fi == remap.end() ? i : fi->second;
        remap[j] = vi;
        picked[i] = vj;
    }
    return picked;
}

int main() {
    std::printf("{\n");
    {
        std::mt19937_64 g(0);
        std::vector<uint64_t> v;
        for (int i = 0; i < 8; ++i) v.push_back(g());
        emit_u64("mt19937_64_seed0", v);
        std::mt19937_64 g2(5489u);
        g2.discard(9999);
        emit_u64("mt19937_64_default_10000th", {g2()});
    }
    {
        std::mt19937_64 g(7);
        std::uniform_real_distribution<double> d(-1.0, 1.0);
        std::vector<double> v;
        for (int i = 0; i < 64; ++i) v.push_back(d(g));
        emit_f64("uniform_real_m1_1_seed7", v);
    }
    {
        std::mt19937_64 g(11);
        std::vector<long long> v;
        const long long ranges[][2] = {{0, 0}, {0, 1}, {3, 10}, {1, 60}, {0, 1999999}, {5, 1LL << 40},
                                       {-7, 7}, {0, (1LL << 62) + 12345}, {100, 100}};
        for (int rep = 0; rep < 4; ++rep)
            for (auto& rg : ranges) {
                std::uniform_int_distribution<long long> d(rg[0], rg[1]);
                v.push_back(d(g));
            }
        emit_i64("uniform_int_mixed_seed11", v);
    }
    {
        std::mt19937_64 g(3);
        std::normal_distribution<double> d(0.0, 1.0);
        std::vector<double> v;
        for (int i = 0; i < 65; ++i) v.push_back(d(g));
        emit_f64("normal_0_1_seed3", v);
        std::normal_distribution<double> d2(2.0, 0.1);
        std::vector<double> w;
        for (int i = 0; i < 9; ++i) w.push_back(d2(g));
        emit_f64("normal_2_01_seed3_continued", w);
    }
    emit_i64("sample_uniform_N64_q20_seed2", picked_indices(64, 20, 2));
    emit_i64("sample_uniform_N2000000_q50_seed1", picked_indices(2000000, 50, 1));
    {
        auto p = picked_indices(2000000, 200000, 1);
        unsigned long long h = 1469598103934665603ULL;  // FNV-1a over the picked sequence
        for (long long x : p) { h ^= (unsigned long long)x; h *= 1099511628211ULL; }
        emit_u64("sample_uniform_N2000000_q200000_seed1_fnv1a", {h}, true);
    }
    std::printf("}\n");
    return 0;
}
