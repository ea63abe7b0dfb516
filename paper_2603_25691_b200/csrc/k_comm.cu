// k_comm.cu — the reduction of the virtual communicator (one-GPU stand-in for the NCCL all-reduce
// of the n x rp partial Yhat and of the aligned B): out = sum over ranks in rank order.
#include <algorithm>

#include "kernels.cuh"

namespace cphifi {
namespace {

struct Srcs {
    const double* p[8];
};

__global__ void rank_order_sum_kernel(const Srcs a, int nsrc, double* __restrict__ out, size_t count) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
        double s = a.p[0][i];
        for (int k = 1; k < nsrc; ++k) s += a.p[k][i];
        out[i] = s;
    }
}

}  // namespace

void rank_order_sum(const double* const* src, int nsrc, double* out, size_t count, int num_sms, cudaStream_t s) {
    if (nsrc < 1 || nsrc > 8) throw_invalid("virtual communicator: 1..8 ranks");
    if (!count) return;
    Srcs a;
    for (int k = 0; k < 8; ++k) a.p[k] = k < nsrc ? src[k] : nullptr;
    const int grid = (int)std::min<size_t>((count + 255) / 256, (size_t)num_sms * 8);
    rank_order_sum_kernel<<<grid, 256, 0, s>>>(a, nsrc, out, count);
    CPHIFI_CHECK_LAUNCH();
}

}  // namespace cphifi
