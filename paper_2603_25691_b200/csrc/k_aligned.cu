// k_aligned.cu — the aligned subproblem's iterative and direct baselines on device (SURVEY §8f
// row 4), sm_100a.  The decoupled eigen solve (k_sandwich.cu / k_dense.cu) is the product path;
// these are the reference's comparison solvers, kept on the GPU so they can serve as device-side
// oracles at sizes the CPU restatement cannot reach:
//   * aligned_matvec (aligned.hpp:58-67): y = vec(diag(d_K) X V + lambda X), X = n x r
//   * the PCG preconditioner of solve_aligned_pcg (aligned.hpp:83-89): 1 / (V(j,j) d_K(i) + lambda)
//   * the materialised Kronecker system of solve_aligned_direct (aligned.hpp:28-37, kronecker
//     matrix_ops.hpp:13-19): sys(i + n j, k + n l) = V(j, l) K(i, k) + lambda [i + n j == k + n l]
#include "kernels.cuh"

namespace cphifi {
namespace {

// y(i, j) = d_K(i) * sum_m X(i, m) V(m, j) + lambda X(i, j); thread per (i, j), consecutive threads
// on consecutive i (column-major X, y: coalesced), V(m, j) a broadcast through L1
__global__ void aligned_matvec_kernel(const double* __restrict__ x, const double* __restrict__ dk,
                                      const double* __restrict__ v, int64_t n, int64_t r, double lambda,
                                      double* __restrict__ y) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * r; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % n, j = e / n;
        double s = 0.0;
        for (int64_t m = 0; m < r; ++m) s = fma(x[i + n * m], __ldg(v + m + r * j), s);
        y[e] = dk[i] * s + lambda * x[e];
    }
}

__global__ void aligned_dinv_kernel(const double* __restrict__ dk, const double* __restrict__ v, int64_t n, int64_t r,
                                    double lambda, double* __restrict__ dinv) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * r; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % n, j = e / n;
        dinv[e] = 1.0 / (v[j + r * j] * dk[i] + lambda);
    }
}

__global__ void hadamard_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t cnt,
                                double* __restrict__ out) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < cnt; e += (int64_t)gridDim.x * blockDim.x)
        out[e] = a[e] * b[e];
}

__global__ void kron_system_kernel(const double* __restrict__ v, const double* __restrict__ kmat, int64_t n, int64_t r,
                                   double lambda, double* __restrict__ sys) {
    const int64_t rn = n * r;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rn * rn; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = e % rn, col = e / rn;
        const int64_t i = row % n, j = row / n, k = col % n, l = col / n;
        sys[e] = v[j + r * l] * kmat[i + n * k] + (row == col ? lambda : 0.0);
    }
}

inline unsigned blocks_for(int64_t cnt) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((cnt + 255) / 256, 8192));
}

}  // namespace

void aligned_matvec_dev(const double* x, const double* dk, const double* v, int64_t n, int64_t r, double lambda,
                        double* y, cudaStream_t s) {
    if (n * r == 0) return;
    aligned_matvec_kernel<<<blocks_for(n * r), 256, 0, s>>>(x, dk, v, n, r, lambda, y);
    CPHIFI_CHECK_LAUNCH();
}

void aligned_dinv(const double* dk, const double* v, int64_t n, int64_t r, double lambda, double* dinv,
                  cudaStream_t s) {
    if (n * r == 0) return;
    aligned_dinv_kernel<<<blocks_for(n * r), 256, 0, s>>>(dk, v, n, r, lambda, dinv);
    CPHIFI_CHECK_LAUNCH();
}

void hadamard(const double* a, const double* b, int64_t cnt, double* out, cudaStream_t s) {
    if (cnt == 0) return;
    hadamard_kernel<<<blocks_for(cnt), 256, 0, s>>>(a, b, cnt, out);
    CPHIFI_CHECK_LAUNCH();
}

void kron_system(const double* v, const double* kmat, int64_t n, int64_t r, double lambda, double* sys,
                 cudaStream_t s) {
    const int64_t rn = n * r;
    if (rn == 0) return;
    kron_system_kernel<<<blocks_for(rn * rn), 256, 0, s>>>(v, kmat, n, r, lambda, sys);
    CPHIFI_CHECK_LAUNCH();
}

}  // namespace cphifi

// ---- unaligned direct / dense baselines (unaligned.hpp:52-96, 164-174) -----------------------
// Both systems are assembled from the row Grams G_i = sum_{l in row i} z_l z_l' (n x rp x rp,
// k_gram.cu) instead of the materialised q x rn factors F and G:
//   (G'F)[(j,i), (j',i')] = G_i(j,j') K(i,i')                         (nonsymmetric baseline)
//   (F'F)[(j,i), (j',i')] = sum_i'' K(i'',i) G_i''(j,j') K(i'',i')    (symmetric dense oracle)
// — the same sums, regrouped by row.
namespace cphifi {
namespace {

__global__ void nonsym_system_kernel(const double* __restrict__ g, const double* __restrict__ kmat, int64_t n,
                                     int64_t r, int64_t rp, double lambda, double* __restrict__ sys) {
    const int64_t rn = n * r;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rn * rn; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = e % rn, col = e / rn;
        const int64_t i = row % n, j = row / n, i2 = col % n, j2 = col / n;
        sys[e] = g[(i * rp + j) * rp + j2] * kmat[i + n * i2] + (row == col ? lambda : 0.0);
    }
}

// S(i'', (j r + j') n + i') = G_i''(j, j') K(i'', i')   (n x r^2 n, column-major)
__global__ void gram_scaled_kernel(const double* __restrict__ g, const double* __restrict__ kmat, int64_t n,
                                   int64_t r, int64_t rp, double* __restrict__ sm) {
    const int64_t cols = r * r * n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * cols; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i3 = e % n, col = e / n;
        const int64_t i2 = col % n, jj = col / n, j = jj / r, j2 = jj % r;
        sm[e] = g[(i3 * rp + j) * rp + j2] * kmat[i3 + n * i2];
    }
}

// sys[(j n + i), (j' n + i')] = C(i, (j r + j') n + i') + lambda [j == j'] K(i,i') + rho [same]
__global__ void sym_place_kernel(const double* __restrict__ cm, const double* __restrict__ kmat, int64_t n, int64_t r,
                                 double lambda, double rho, double* __restrict__ sys) {
    const int64_t rn = n * r;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < rn * rn; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = e % rn, col = e / rn;
        const int64_t i = row % n, j = row / n, i2 = col % n, j2 = col / n;
        double v = cm[i + n * ((j * r + j2) * n + i2)];
        if (j == j2) v += lambda * kmat[i + n * i2];
        if (row == col) v += rho;
        sys[e] = v;
    }
}

inline unsigned blocks_for2(int64_t cnt) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((cnt + 255) / 256, 16384));
}

}  // namespace

void nonsym_system(const double* g, const double* kmat, int64_t n, int64_t r, int64_t rp, double lambda, double* sys,
                   cudaStream_t s) {
    if (n * r == 0) return;
    nonsym_system_kernel<<<blocks_for2(n * r * n * r), 256, 0, s>>>(g, kmat, n, r, rp, lambda, sys);
    CPHIFI_CHECK_LAUNCH();
}

void gram_scaled(const double* g, const double* kmat, int64_t n, int64_t r, int64_t rp, double* sm, cudaStream_t s) {
    if (n * r == 0) return;
    gram_scaled_kernel<<<blocks_for2(n * r * r * n), 256, 0, s>>>(g, kmat, n, r, rp, sm);
    CPHIFI_CHECK_LAUNCH();
}

void sym_place(const double* cm, const double* kmat, int64_t n, int64_t r, double lambda, double rho, double* sys,
               cudaStream_t s) {
    if (n * r == 0) return;
    sym_place_kernel<<<blocks_for2(n * r * n * r), 256, 0, s>>>(cm, kmat, n, r, lambda, rho, sys);
    CPHIFI_CHECK_LAUNCH();
}

}  // namespace cphifi
