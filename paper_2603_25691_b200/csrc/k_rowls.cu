// k_rowls.cu — per-row minimum-norm least squares of the unaligned finite-mode update
// (AlsState::update_finite_mode, als.hpp:144-162).
//
// The reference solves, for every row i of a finite mode k with observations,
//     a_i = argmin ||Z_i a - t_i||  (minimum norm)   via CompleteOrthogonalDecomposition(Z_i),
// Z_i = the Zhat rows of the row's observations, t_i their values; rows without observations
// stay zero.  Here a_i = G_i^+ b_i with G_i = Z_i'Z_i (the row-Gram matrices of k_gram.cu, one
// pass over the observations) and b_i = Z_i' t_i (the subproblem's B): the same minimiser; the
// pseudo-inverse drops eigenvalues of G_i below r eps lambda_max(G_i) (COD's rank decision acts on
// singular values of Z_i; the two agree while cond(Z_i) < ~1e7, documented in DESIGN.md).
//
// One CTA per row: cyclic parallel Jacobi on the r x r matrix in shared memory (round-robin
// tournament, r/2 disjoint rotations per step: rows, then columns, then V), sweeps until the
// off-diagonal mass is below eps^2 of the diagonal, then a_i = V diag(1/lambda) V' b_i.
// Deterministic (fixed schedule, fixed reduction order).
#include "kernels.cuh"

namespace cphifi {
namespace {

constexpr int LT = 256;
constexpr int MAX_SWEEPS = 30;

template <int RP>
__global__ void __launch_bounds__(LT) rowls_kernel(const double* __restrict__ g, const double* __restrict__ b, int64_t n,
                                                   int r, double* __restrict__ a_out) {
    constexpr int P = RP + 1;
    extern __shared__ double rls_smem[];  // A, V: RP x P each (66.5 KB at RP = 64)
    double(*A)[P] = reinterpret_cast<double(*)[P]>(rls_smem);
    double(*V)[P] = reinterpret_cast<double(*)[P]>(rls_smem + RP * P);
    __shared__ double cs[RP / 2 > 0 ? RP / 2 : 1][2];
    __shared__ double red[LT / 32];
    __shared__ double bv[RP], tv[RP];
    __shared__ int s_done;
    const int64_t i = blockIdx.x;
    const int tid = threadIdx.x;
    const double* gi = g + i * RP * RP;
    for (int e = tid; e < RP * RP; e += LT) {
        const int p = e / RP, q = e % RP;
        A[p][q] = (p < r && q < r) ? gi[e] : 0.0;
        V[p][q] = p == q ? 1.0 : 0.0;
    }
    for (int j = tid; j < RP; j += LT) bv[j] = j < r ? b[i + n * j] : 0.0;
    __syncthreads();
    const int m = (r + 1) & ~1;  // players (a dummy one when r is odd)
    auto block_sum = [&](double v) {
        for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
        if ((tid & 31) == 0) red[tid >> 5] = v;
        __syncthreads();
        double t = 0.0;
        for (int w = 0; w < LT / 32; ++w) t += red[w];
        __syncthreads();
        return t;
    };
    for (int sweep = 0; sweep < MAX_SWEEPS && m >= 2; ++sweep) {
        // convergence: off-diagonal mass vs diagonal mass
        double off = 0.0, dia = 0.0;
        for (int e = tid; e < r * r; e += LT) {
            const int p = e / r, q = e % r;
            const double v = A[p][q] * A[p][q];
            if (p == q) dia += v;
            else off += v;
        }
        off = block_sum(off);
        dia = block_sum(dia);
        if (tid == 0) s_done = !(off > 1e-32 * dia);
        __syncthreads();
        if (s_done) break;
        for (int step = 0; step < m - 1; ++step) {
            if (tid < m / 2) {  // rotation of pair tid (circle method)
                int p = tid == 0 ? m - 1 : (step + tid) % (m - 1);
                int q = tid == 0 ? step : (step - tid + m - 1) % (m - 1);
                if (p > q) {
                    const int t = p;
                    p = q;
                    q = t;
                }
                double c = 1.0, s = 0.0;
                if (q < r && A[p][q] != 0.0) {
                    const double theta = (A[q][q] - A[p][p]) / (2.0 * A[p][q]);
                    const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(fma(theta, theta, 1.0)));
                    c = 1.0 / sqrt(fma(t, t, 1.0));
                    s = t * c;
                }
                cs[tid][0] = c;
                cs[tid][1] = s;
            }
            __syncthreads();
            // rows: A <- J' A (pairs are disjoint)
            for (int e = tid; e < (m / 2) * r; e += LT) {
                const int k = e / r, j = e % r;
                int p = k == 0 ? m - 1 : (step + k) % (m - 1);
                int q = k == 0 ? step : (step - k + m - 1) % (m - 1);
                if (p > q) {
                    const int t = p;
                    p = q;
                    q = t;
                }
                if (q >= r) continue;
                const double c = cs[k][0], s = cs[k][1];
                const double ap = A[p][j], aq = A[q][j];
                A[p][j] = c * ap - s * aq;
                A[q][j] = s * ap + c * aq;
            }
            __syncthreads();
            // columns: A <- A J, V <- V J
            for (int e = tid; e < (m / 2) * r; e += LT) {
                const int k = e / r, j = e % r;
                int p = k == 0 ? m - 1 : (step + k) % (m - 1);
                int q = k == 0 ? step : (step - k + m - 1) % (m - 1);
                if (p > q) {
                    const int t = p;
                    p = q;
                    q = t;
                }
                if (q >= r) continue;
                const double c = cs[k][0], s = cs[k][1];
                const double ap = A[j][p], aq = A[j][q];
                A[j][p] = c * ap - s * aq;
                A[j][q] = s * ap + c * aq;
                const double vp = V[j][p], vq = V[j][q];
                V[j][p] = c * vp - s * vq;
                V[j][q] = s * vp + c * vq;
            }
            __syncthreads();
        }
    }
    // pseudo-inverse solve: t_j = (V(:,j)' b) / lambda_j for lambda_j > tau, a = V t
    double lmax = 0.0;
    for (int j = 0; j < r; ++j) lmax = fmax(lmax, A[j][j]);
    const double tau = lmax * (double)r * 2.220446049250313e-16;
    for (int j = tid; j < r; j += LT) {
        double s = 0.0;
        for (int p = 0; p < r; ++p) s = fma(V[p][j], bv[p], s);
        const double lam = A[j][j];
        tv[j] = (lam > tau && lmax > 0.0) ? s / lam : 0.0;
    }
    __syncthreads();
    for (int p = tid; p < r; p += LT) {
        double s = 0.0;
        for (int j = 0; j < r; ++j) s = fma(V[p][j], tv[j], s);
        a_out[i + n * p] = s;
    }
}

}  // namespace

template <int RP>
void rowls_t(const double* g, const double* b, int64_t n, int64_t r, double* a_out, cudaStream_t s) {
    const size_t smem = sizeof(double) * 2 * RP * (RP + 1);
    func_attr_once((const void*)rowls_kernel<RP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    rowls_kernel<RP><<<(unsigned)n, LT, smem, s>>>(g, b, n, (int)r, a_out);
}

void rowls_solve(const double* g, const double* b, int64_t n, int64_t r, int64_t rp, double* a_out, cudaStream_t s) {
    if (n <= 0) return;
    switch (rp) {
        case 4: rowls_t<4>(g, b, n, r, a_out, s); break;
        case 8: rowls_t<8>(g, b, n, r, a_out, s); break;
        case 16: rowls_t<16>(g, b, n, r, a_out, s); break;
        case 32: rowls_t<32>(g, b, n, r, a_out, s); break;
        case 64: rowls_t<64>(g, b, n, r, a_out, s); break;
        default: throw_invalid("finite-mode update: padded rank above 64 is not supported");
    }
    CPHIFI_CHECK_LAUNCH();
}

}  // namespace cphifi
