// k_als.cu — the ALS infinite-mode update's error terms on device.
//
//   AlsState::relative_error (als.hpp:221-237)
//     unaligned: sqrt(sum_l (v_l - <A_k(i_k(l),:) , z_l>)^2) / ||v||  over the observed entries,
//                z_l = prod_{m != k} A_m(i_m(l), :) (build_zhat + gather_rows with A_k in place of
//                Xhat, observations.hpp:142-198)
//     aligned:   ||T - [[A]]|| / ||T||  — the reference materialises kruskal_full (an N-sized
//                tensor); here ||T - M||^2 = ||T||^2 - 2 <A_k, B> + 1'(A_k'A_k o V)1 with the
//                MTTKRP B and Gram V the solve already computed (same other-mode factors), so
//                no N-sized pass beyond the one ||T||^2 per tensor.  Cancellation bounds the
//                absolute error of the squared error by ~1e-15 ||T||^2 (tests state the tolerance).
//
// sq_residual_kernel: blocks take equal-count contiguous ranges of the i_k-sorted plan (robust to
// Zipf rows); each block finds its row range once, every entry its row by a binary search inside
// it; rows of A_k and of the other factors are read through L1 (packed row-major, rank padded).
// Block sums are written in block order and summed in that order: deterministic.
#include "kernels.cuh"

namespace cphifi {
namespace {

constexpr int AT = 256;  // threads per block
constexpr int AE = 8;    // entries per thread

__device__ __forceinline__ double block_reduce(double v) {
    __shared__ double sh[AT / 32];
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x < 32) {
        t = threadIdx.x < AT / 32 ? sh[threadIdx.x] : 0.0;
        for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    }
    __syncthreads();
    return t;  // thread 0
}

__global__ void sq_residual_kernel(const SqResidualArgs a, double* __restrict__ partial) {
    __shared__ int64_t s_r0, s_r1;
    const int64_t per = (int64_t)AT * AE;
    const int64_t b0 = (int64_t)blockIdx.x * per, b1 = min(a.q, b0 + per);
    if (threadIdx.x == 0) {  // rows of the first and last entry of the block: largest i with rp[i] <= pos
        auto row_of = [&](int64_t pos) {
            int64_t lo = 0, hi = a.n;  // rp[lo] <= pos < rp[hi]
            while (hi - lo > 1) {
                const int64_t mid = (lo + hi) >> 1;
                if (a.row_ptr[mid] <= pos) lo = mid;
                else hi = mid;
            }
            return lo;
        };
        s_r0 = b0 < b1 ? row_of(b0) : 0;
        s_r1 = b0 < b1 ? row_of(b1 - 1) : 0;
    }
    __syncthreads();
    const int64_t r0 = s_r0, r1 = s_r1;
    double acc = 0.0;
#pragma unroll 1
    for (int e = 0; e < AE; ++e) {
        const int64_t l = b0 + threadIdx.x + (int64_t)AT * e;
        if (l >= b1) break;
        int64_t lo = r0, hi = r1 + 1;
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (a.row_ptr[mid] <= l) lo = mid;
            else hi = mid;
        }
        const double* ar = a.ak + lo * a.rp;
        const double* f[8];
        for (int m = 0; m < a.dother; ++m) f[m] = a.fac + a.fac_off[m] + (int64_t)a.idx[(int64_t)m * a.ldq + l] * a.rp;
        double fit = 0.0;
        for (int j = 0; j < a.r; ++j) {
            double z = __ldg(f[0] + j);  // modes ascending (observations.hpp:150-156)
            for (int m = 1; m < a.dother; ++m) z *= __ldg(f[m] + j);
            fit = fma(__ldg(ar + j), z, fit);
        }
        const double res = a.values[l] - fit;
        acc = fma(res, res, acc);
    }
    const double t = block_reduce(acc);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

__global__ void sum_partials_kernel(const double* __restrict__ partial, int64_t nb, double* out) {
    // one warp, lanes stride the partials, fixed tree
    double t = 0.0;
    for (int64_t b = threadIdx.x; b < nb; b += 32) t += partial[b];
    for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    if (threadIdx.x == 0) *out = t;
}

__global__ void sq_norm_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ partial) {
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)AT + threadIdx.x; i < n; i += (int64_t)gridDim.x * AT) acc = fma(x[i], x[i], acc);
    const double t = block_reduce(acc);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

}  // namespace

int64_t sq_residual_blocks(int64_t q) { return std::max<int64_t>(1, (q + (int64_t)AT * AE - 1) / ((int64_t)AT * AE)); }

void sq_residual(const SqResidualArgs& a, double* partial, double* out, cudaStream_t s) {
    if (a.dother < 1 || a.dother > 8) throw_invalid("relative_error: tensor order out of range");
    const int64_t nb = sq_residual_blocks(a.q);
    if (a.q > 0) {
        sq_residual_kernel<<<(unsigned)nb, AT, 0, s>>>(a, partial);
        CPHIFI_CHECK_LAUNCH();
        sum_partials_kernel<<<1, 32, 0, s>>>(partial, nb, out);
    } else {
        CPHIFI_CUDA(cudaMemsetAsync(out, 0, sizeof(double), s));
    }
    CPHIFI_CHECK_LAUNCH();
}

void sq_norm(const double* x, int64_t n, double* partial, int64_t nb, double* out, cudaStream_t s) {
    sq_norm_kernel<<<(unsigned)nb, AT, 0, s>>>(x, n, partial);
    CPHIFI_CHECK_LAUNCH();
    sum_partials_kernel<<<1, 32, 0, s>>>(partial, nb, out);
    CPHIFI_CHECK_LAUNCH();
}

}  // namespace cphifi
