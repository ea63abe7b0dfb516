// k_synth.cu — seeded synthetic observations generated on the device (configs 3 and 4).
//
// BASELINE configs 3/4 hold 2e8 / 1e9 observations (4.8 / 20 GB): they are drawn on the GPU
// with a counter-based generator so that every draw is a pure function of (seed, l, stream)
// and the stream is bit-identical run to run (tests/test_synth.py re-derives draws on the host
// with the same integer arithmetic).  Not part of the solver path.
//   u64(l, s) = splitmix64(seed ^ splitmix64(l * 0x9E3779B97F4A7C15 + s))
//   uniform index in [0, n): (u64 >> 32) * n >> 32;  uniform double: (u64 >> 11) * 2^-53
//   Zipf mode: smallest i with cdf[i] > u (host-built CDF of (i+1)^-s)
//   value = sum_j prod_m A_m(i_m, j) + noise_std * N(0,1)  (Box-Muller on two uniforms)
#include <cmath>

#include "kernels.cuh"

namespace cphifi {
namespace {

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__device__ __forceinline__ uint64_t draw(uint64_t seed, uint64_t l, uint64_t s) {
    return splitmix64(seed ^ splitmix64(l * 0x9E3779B97F4A7C15ull + s));
}

struct SynthArgs {
    int d = 0;
    int64_t shape[8] = {0};
    int64_t q = 0;
    uint64_t seed = 0;
    int zipf_mode = -1;
    const double* zipf_cdf = nullptr;
    int64_t r = 0;
    const double* fac[8] = {nullptr};  // device column-major n_m x r
    double noise_std = 0.0;
    int32_t* idx = nullptr;            // d x q
    double* vals = nullptr;            // q
};

__global__ void synth_kernel(const SynthArgs a) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < a.q; l += (int64_t)gridDim.x * blockDim.x) {
        int64_t ix[8];
        for (int m = 0; m < a.d; ++m) {
            const uint64_t u = draw(a.seed, (uint64_t)l, (uint64_t)m);
            const uint64_t n = (uint64_t)a.shape[m];
            if (m == a.zipf_mode) {
                const double v = (double)(u >> 11) * 0x1.0p-53;
                int64_t lo = 0, hi = a.shape[m] - 1;  // smallest i with cdf[i] > v
                while (lo < hi) {
                    const int64_t mid = (lo + hi) >> 1;
                    if (a.zipf_cdf[mid] > v) hi = mid; else lo = mid + 1;
                }
                ix[m] = lo;
            } else {
                ix[m] = (int64_t)(((u >> 32) * n) >> 32);
            }
            a.idx[(int64_t)m * a.q + l] = (int32_t)ix[m];
        }
        double v = 0.0;
        for (int64_t j = 0; j < a.r; ++j) {
            double p = a.fac[0][ix[0] + a.shape[0] * j];
            for (int m = 1; m < a.d; ++m) p *= a.fac[m][ix[m] + a.shape[m] * j];
            v += p;
        }
        const uint64_t u1 = draw(a.seed, (uint64_t)l, 64), u2 = draw(a.seed, (uint64_t)l, 65);
        const double f1 = ((double)(u1 >> 11) + 1.0) * 0x1.0p-53;  // (0, 1]
        const double f2 = (double)(u2 >> 11) * 0x1.0p-53;
        a.vals[l] = v + a.noise_std * (sqrt(-2.0 * log(f1)) * cos(6.283185307179586 * f2));
    }
}

}  // namespace

void synth_observations(int d, const int64_t* shape, int64_t q, uint64_t seed, int zipf_mode, double zipf_s, int64_t r,
                        const double* const* fac_dev, double noise_std, int32_t* idx, double* vals, int num_sms,
                        cudaStream_t s) {
    SynthArgs a;
    a.d = d;
    for (int m = 0; m < d; ++m) {
        a.shape[m] = shape[m];
        a.fac[m] = fac_dev[m];
    }
    a.q = q;
    a.seed = seed;
    a.r = r;
    a.noise_std = noise_std;
    a.idx = idx;
    a.vals = vals;
    DevBuf<double> cdf;
    if (zipf_mode >= 0) {
        const int64_t n = shape[zipf_mode];
        std::vector<double> h(n);
        double tot = 0.0;
        for (int64_t i = 0; i < n; ++i) tot += std::pow((double)(i + 1), -zipf_s);
        double acc = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            acc += std::pow((double)(i + 1), -zipf_s);
            h[i] = acc / tot;
        }
        h[n - 1] = 1.0;
        cdf.alloc(n);
        CPHIFI_CUDA(cudaMemcpyAsync(cdf.get(), h.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
        a.zipf_mode = zipf_mode;
        a.zipf_cdf = cdf.get();
        CPHIFI_CUDA(cudaStreamSynchronize(s));
    }
    synth_kernel<<<num_sms * 8, 256, 0, s>>>(a);
    CPHIFI_CHECK_LAUNCH();
    CPHIFI_CUDA(cudaStreamSynchronize(s));
}

}  // namespace cphifi
