// k_synth.cu — seeded synthetic observations generated on the device (configs 3 and 4).
//
// BASELINE configs 3/4 hold 2e8 / 1e9 observations (4.8 / 20 GB): they are drawn on the GPU with
// the counter-based generator of inputs/synth_math.h, so every draw is a pure function of (seed, l,
// stream) and bit-identical to the host generator inputs/synth_host.cpp (the oracle's inputs;
// tests/test_gpu_synth.py compares the two).  Not part of the solver path.
#include <cmath>

#include "../../inputs/synth_math.h"
#include "kernels.cuh"

namespace cphifi {
namespace {

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
            const uint64_t u = syn_draw(a.seed, (uint64_t)l, (uint64_t)m);
            ix[m] = m == a.zipf_mode ? syn_zipf_index(u, a.zipf_cdf, a.shape[m]) : syn_uniform_index(u, a.shape[m]);
            a.idx[(int64_t)m * a.q + l] = (int32_t)ix[m];
        }
        double v = 0.0;
        for (int64_t j = 0; j < a.r; ++j) {
            double p = a.fac[0][ix[0] + a.shape[0] * j];
            for (int m = 1; m < a.d; ++m) p = SYN_MUL(p, a.fac[m][ix[m] + a.shape[m] * j]);
            v = SYN_ADD(v, p);
        }
        a.vals[l] = SYN_ADD(v, SYN_MUL(a.noise_std, syn_normal(a.seed, (uint64_t)l)));
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
    if (zipf_mode >= 0) {  // the host table of inputs/synth_host.cpp inp_zipf_cdf, same arithmetic
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
