// k_sandwich.cu — the eigenbasis "sandwich"  Y = U ((U' X U_V) op E) U_V'  in two launches.
//
// Both hot-path consumers of the Kronecker eigenbasis have this shape:
//   * build_preconditioner's apply (unaligned.hpp:135-139): M^-1 x = U_K ((U_K' X U_V) .* D) U_V'
//   * solve_aligned_decoupled (aligned.hpp:44-53):  W = U_K ((U_K' B U_V) ./ (sigma_j mu_i + lambda)) U_V'
// Evaluated left to right like the reference (Eigen's (A*B)*C), each phase is a ROW-LOCAL
// contraction once the n x n factor is read column-wise:
//   phase 1  core(i,:) = op( (U(:,i)' X) U_V )          (U column i contiguous)
//   phase 2  Y(i,:)    = (U'(:,i)' core) U_V'            (U' column i = U row i, contiguous)
// so a CTA owns RB rows, streams its RB columns of U (or U') together with the matching k-chunk
// of X (or core) through a 4-stage cp.async ring (64 k per stage), and finishes the r x r product and the
// element-wise op in its epilogue.  Two launches replace four DMMA GEMM launches plus an
// epilogue pass; the n x n factor is read once per phase (HBM/L2 bound: 8 n^2 bytes per phase),
// the r x n chunks come from L2.  Every sum has a fixed order: bit-reproducible.
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"
#include "tma.cuh"

namespace cphifi {
namespace {

constexpr int SW_T = 256;   // threads per CTA
constexpr int SW_KC = 64;   // k per stage
constexpr int SW_ST = 4;    // stages

__device__ __forceinline__ void cpa8(void* smem, const void* gmem, bool pred) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(pred ? 8 : 0));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int RP, int RB>
struct SwSmem {
    static constexpr int MP = RP + 1;  // pitch of the k x j chunk: conflict-free transposed fills
    double m[SW_ST][SW_KC][MP];        // X (phase 1) or core (phase 2) rows k0 .. k0 + KC
    double u[SW_ST][SW_KC][RB];        // u[kk][row] = F(k0 + kk, i0 + row), F = U or U'
    double tt[RB][MP];                 // reduced (F' M) rows of this CTA
    double red[SW_T * RB];             // k-slice partials (S x RB x RP)
};

// PH = 1: core(i, j) = op((U' X U_V)(i, j)) row-major [i * RP + j] (zero pad j >= r)
// PH = 2: y(i + n j) = (U core U_V')(i, j)
template <int RP, int RB, int PH>
__global__ void __launch_bounds__(SW_T) sandwich_kernel(const SandArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SwSmem<RP, RB>& sm = *reinterpret_cast<SwSmem<RP, RB>*>(smem_raw);
    constexpr int S = SW_T / RP;  // k-slices
    const int64_t n = a.n;
    const int r = (int)a.r;
    const int64_t i0 = (int64_t)blockIdx.x * RB;
    const int rb = (int)min((int64_t)RB, n - i0);
    const int j = threadIdx.x % RP, s = threadIdx.x / RP;
    const double* F = PH == 1 ? a.u : a.ut;  // column i of F = the row's coefficients
    const int nchunks = (int)((n + SW_KC - 1) / SW_KC);

    auto load = [&](int st, int c) {
        const int64_t k0 = (int64_t)c * SW_KC;
        const int kc = (int)min((int64_t)SW_KC, n - k0);
        for (int e = threadIdx.x; e < SW_KC * RB; e += SW_T) {
            const int kk = e % SW_KC, row = e / SW_KC;
            const bool p = kk < kc && row < rb;
            cpa8(&sm.u[st][kk][row], p ? F + (k0 + kk) + n * (i0 + row) : F, p);
        }
        if constexpr (PH == 1) {  // X column-major: consecutive threads walk k (coalesced)
            for (int e = threadIdx.x; e < SW_KC * RP; e += SW_T) {
                const int kk = e % SW_KC, jj = e / SW_KC;
                const bool p = kk < kc && jj < r;
                cpa8(&sm.m[st][kk][jj], p ? a.x + (k0 + kk) + a.ldx * jj : a.x, p);
            }
        } else {  // core row-major (pad columns are zero)
            for (int e = threadIdx.x; e < SW_KC * RP; e += SW_T) {
                const int kk = e / RP, jj = e % RP;
                const bool p = kk < kc;
                cpa8(&sm.m[st][kk][jj], p ? a.core + (k0 + kk) * RP + jj : a.core, p);
            }
        }
    };

    double acc[RB];
#pragma unroll
    for (int q = 0; q < RB; ++q) acc[q] = 0.0;
#pragma unroll
    for (int st = 0; st < SW_ST - 1; ++st) {
        if (st < nchunks) load(st, st);
        cpa_commit();
    }
    for (int c = 0; c < nchunks; ++c) {
        const int st = c % SW_ST;
        cpa_wait<SW_ST - 2>();
        __syncthreads();
        if (c + SW_ST - 1 < nchunks) load((c + SW_ST - 1) % SW_ST, c + SW_ST - 1);
        cpa_commit();
#pragma unroll
        for (int kk = s; kk < SW_KC; kk += S) {
            const double xv = sm.m[st][kk][j];
#pragma unroll
            for (int q = 0; q < RB; ++q) acc[q] = fma(sm.u[st][kk][q], xv, acc[q]);
        }
    }
    cpa_wait<0>();
    __syncthreads();
    // reduce the S k-slices in slice order
    double* red = sm.red;
#pragma unroll
    for (int q = 0; q < RB; ++q) red[(s * RB + q) * RP + j] = acc[q];
    __syncthreads();
    for (int e = threadIdx.x; e < RB * RP; e += SW_T) {
        const int q = e / RP, jj = e % RP;
        double t = 0.0;
        for (int z = 0; z < S; ++z) t += red[(z * RB + q) * RP + jj];
        sm.tt[q][jj] = t;
    }
    __syncthreads();
    // epilogue: (row of F' M) times U_V (phase 1) or U_V' (phase 2), then the element-wise op
    for (int e = threadIdx.x; e < RB * RP; e += SW_T) {
        const int q = e / RP, jj = e % RP;
        if (q >= rb) continue;
        const int64_t i = i0 + q;
        if (jj >= r) {
            if constexpr (PH == 1) a.core_out[i * RP + jj] = 0.0;
            continue;
        }
        double c = 0.0;
        for (int m = 0; m < r; ++m) c = fma(sm.tt[q][m], PH == 1 ? a.uv[m + (int64_t)r * jj] : a.uv[jj + (int64_t)r * m], c);
        if constexpr (PH == 1) {
            double out;
            if (a.op == SW_MUL) {
                out = c * a.dmat[i + n * jj];
            } else {
                const double den = a.e_col[jj] * a.e_row[i] + a.beta;
                if (den == 0.0) *a.flag = 1;
                out = c / den;
            }
            a.core_out[i * RP + jj] = out;
        } else {
            a.y[i + a.ldy * jj] = c;
        }
    }
}

// uv[m][j] = U_V(m, j) (phase 1) or U_V(j, m) (phase 2), zero beyond r: one 8-byte cp.async per
// element (completion awaited by stage_uv_wait before the epilogue), plain stores for the padding
template <int RP, int NT, int PH>
__device__ __forceinline__ void stage_uv(double (*uv)[RP + 1], const double* src, int r) {
    for (int e = threadIdx.x; e < RP * RP; e += NT) {
        const int m = e / RP, j = e % RP;
        if (m < r && j < r) {
            const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(&uv[m][j]));
            const double* g = src + (PH == 1 ? m + (int64_t)r * j : j + (int64_t)r * m);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(g) : "memory");
        } else {
            uv[m][j] = 0.0;
        }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void stage_uv_wait() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// ---- v2 (even n, 16-byte aligned columns): bulk-copy ring, k across lanes -----------------
// Each stage brings KC consecutive k of the CTA's RB columns of F (U or U') and of every column of
// M (X, or the phase-1 core, both column-major with leading dimension ld) with one bulk copy per
// column: smem rows contiguous in k, so lanes walk k (conflict-free) and warps split the columns
// j.  The per-(j, row) partial sums are reduced over the 32 lanes through shared memory in lane
// order.  Phase 1 writes core column-major (n x r); phase 2 reads it.  (v1 above: one 8-byte
// cp.async per element, 28-31 us per phase at n = 1024, r = 32 — latency-bound by the request
// count, like the per-column MTTKRP copies.)
constexpr int SW2_T = 256, SW2_W = SW2_T / 32, SW2_ST = 4;
template <int RP>
struct Sw2 {
    static constexpr int KC = RP >= 64 ? 64 : (RP >= 32 ? 128 : 256);  // k per stage
    static constexpr int JPW = RP / SW2_W;                              // columns per warp
};
template <int RP, int RB>
struct Sw2Smem {
    static constexpr int KC = Sw2<RP>::KC;
    double m[SW2_ST][RP][KC];
    double u[SW2_ST][RB][KC];
    double tt[RB][RP + 1];
    double uv[RP][RP + 1];  // as in v3 below
    uint64_t full[SW2_ST];
};
template <int RP, int RB, int PH>
__global__ void __launch_bounds__(SW2_T) sandwich2_kernel(const SandArgs a, const __grid_constant__ CUtensorMap tm_f,
                                                          const __grid_constant__ CUtensorMap tm_m) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    using SM = Sw2Smem<RP, RB>;
    SM& sm = *reinterpret_cast<SM*>(smem_raw);
    constexpr int KC = Sw2<RP>::KC, JPW = Sw2<RP>::JPW;
    const int64_t n = a.n;
    const int r = (int)a.r;
    const int64_t i0 = (int64_t)blockIdx.x * RB;
    const int rb = (int)min((int64_t)RB, n - i0);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nch = (int)((n + KC - 1) / KC);
    if (threadIdx.x == 0) {
        for (int st = 0; st < SW2_ST; ++st) tma::mbar_init(&sm.full[st], 1);
        tma::fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int c) {  // thread 0: two 2-D tensor copies per stage (out-of-range reads as 0)
        const int st = c % SW2_ST;
        const int k0 = c * KC;
        tma::mbar_expect_tx(&sm.full[st], (unsigned)(sizeof(double) * KC * (RB + RP)));
        tma::tensor_g2s_2d(&sm.u[st][0][0], &tm_f, k0, (int)i0, &sm.full[st]);
        tma::tensor_g2s_2d(&sm.m[st][0][0], &tm_m, k0, 0, &sm.full[st]);
    };
    if (threadIdx.x == 0)
        for (int c = 0; c < min(nch, SW2_ST); ++c) issue(c);
    stage_uv<RP, SW2_T, PH>(sm.uv, a.uv, r);
    double acc[JPW][RB];
#pragma unroll
    for (int jj = 0; jj < JPW; ++jj)
#pragma unroll
        for (int q = 0; q < RB; ++q) acc[jj][q] = 0.0;
    for (int c = 0; c < nch; ++c) {
        const int st = c % SW2_ST;
        const int kc = (int)min((int64_t)KC, n - (int64_t)c * KC);
        tma::mbar_wait(&sm.full[st], (unsigned)((c / SW2_ST) & 1));
        for (int kk = lane; kk < kc; kk += 32) {
            double uq[RB];
#pragma unroll
            for (int q = 0; q < RB; ++q) uq[q] = q < rb ? sm.u[st][q][kk] : 0.0;
#pragma unroll
            for (int jj = 0; jj < JPW; ++jj) {
                const int j = warp + SW2_W * jj;
                const double xv = j < r ? sm.m[st][j][kk] : 0.0;
#pragma unroll
                for (int q = 0; q < RB; ++q) acc[jj][q] = fma(uq[q], xv, acc[jj][q]);
            }
        }
        __syncthreads();  // every warp is done with slot st
        if (threadIdx.x == 0 && c + SW2_ST < nch) {
            tma::fence_proxy_async();
            issue(c + SW2_ST);
        }
    }
    // lane partials -> shared memory (the ring is idle now), summed over lanes in lane order
    double* red = &sm.m[0][0][0];  // W x 32 x (JPW * RB)
    static_assert(SW2_T * JPW * RB <= SW2_ST * RP * KC, "reduction fits the ring");
#pragma unroll
    for (int jj = 0; jj < JPW; ++jj)
#pragma unroll
        for (int q = 0; q < RB; ++q) red[(warp * 32 + lane) * (JPW * RB) + jj * RB + q] = acc[jj][q];
    __syncthreads();
    for (int e = threadIdx.x; e < SW2_W * JPW * RB; e += SW2_T) {
        const int w = e / (JPW * RB), rem = e % (JPW * RB), jj = rem / RB, q = rem % RB;
        double t = 0.0;
        for (int l = 0; l < 32; ++l) t += red[(w * 32 + l) * (JPW * RB) + rem];
        sm.tt[q][w + SW2_W * jj] = t;
    }
    stage_uv_wait();
    __syncthreads();
    for (int e = threadIdx.x; e < RB * RP; e += SW2_T) {
        const int q = e / RP, jj = e % RP;
        if (q >= rb || jj >= r) continue;
        const int64_t i = i0 + q;
        double c0 = 0.0, c1 = 0.0;  // two chains, summed once: a fixed order
#pragma unroll
        for (int m = 0; m < RP; m += 2) {
            c0 = fma(sm.tt[q][m], sm.uv[m][jj], c0);
            c1 = fma(sm.tt[q][m + 1], sm.uv[m + 1][jj], c1);
        }
        const double c = c0 + c1;
        if constexpr (PH == 1) {
            double out;
            if (a.op == SW_MUL) {
                out = c * a.dmat[i + n * jj];
            } else {
                const double den = a.e_col[jj] * a.e_row[i] + a.beta;
                if (den == 0.0) *a.flag = 1;
                out = c / den;
            }
            a.core_out[i + n * jj] = out;
        } else {
            a.y[i + a.ldy * jj] = c;
        }
    }
}

// ---- v3: the n x n x r products on the FP64 tensor cores (DMMA m8n8k4) ------------------------
// Phase PH computes, for the CTA's RB = 8 rows i, C(i, :) = sum_k F(i, k) M(k, :) with
//   phase 1: F = U' (so C = U' X), M = X row-major padded (a transposed copy, `xrm`);
//   phase 2: F = U,                M = the phase-1 core, written row-major padded by phase 1,
// then the same r x r epilogue as v2.  A stage brings KC k-values of the F rows (tensor-map box
// RB x KC over F(i, k) = f[i + n k]: shared memory [KC][RB], so an A fragment — 8 rows i x 4 k —
// is 32 consecutive doubles) and of M (box RPP x KC over the row-major M: [KC][RPP], the pitch
// RPP = RP + 8 spreads a B fragment's 4 k-rows over all 32 banks).  The 8 warps split every
// stage's k-steps (warp w: k-steps w, w + 8, ...), each holding RP / 8 accumulator tiles; the
// warp partials are summed in warp order at the end: deterministic.
constexpr int SW3_T = 256, SW3_W = 8, SW3_RB = 8;
template <int RP>
struct Sw3 {
    static constexpr int RPP = RP + 8;                  // B-tile pitch
    static constexpr int KC = RP >= 64 ? 64 : 128;     // k per stage
    static constexpr int NTL = RP / 8;                  // 8 x 8 output tiles per CTA
    static constexpr int ST = RP >= 64 ? 3 : 4;        // ring stages (U_V staged beside them)
};
template <int RP>
struct Sw3Smem {
    static constexpr int KC = Sw3<RP>::KC, RPP = Sw3<RP>::RPP, ST = Sw3<RP>::ST;
    double a[ST][KC][SW3_RB];
    double b[ST][KC][RPP];
    double red[SW3_W][SW3_RB][RP];
    double tt[SW3_RB][RP + 1];
    double uv[RP][RP + 1];  // U_V (phase 1) or U_V' (phase 2), zero-padded: uv[m][j] multiplies tt[q][m]
    uint64_t full[ST];
};
__device__ __forceinline__ void dmma_sw(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}
template <int RP, int PH>
__global__ void __launch_bounds__(SW3_T) sandwich3_kernel(const SandArgs a, const __grid_constant__ CUtensorMap tm_f,
                                                          const __grid_constant__ CUtensorMap tm_m, double* core_rm) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    using SM = Sw3Smem<RP>;
    SM& sm = *reinterpret_cast<SM*>(smem_raw);
    constexpr int KC = Sw3<RP>::KC, RPP = Sw3<RP>::RPP, NTL = Sw3<RP>::NTL, RB = SW3_RB, SW3_ST = Sw3<RP>::ST;
    const int64_t n = a.n;
    const int r = (int)a.r;
    const int64_t i0 = (int64_t)blockIdx.x * RB;
    const int rb = (int)min((int64_t)RB, n - i0);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nch = (int)((n + KC - 1) / KC);
    if (threadIdx.x == 0) {
        for (int st = 0; st < SW3_ST; ++st) tma::mbar_init(&sm.full[st], 1);
        tma::fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int c) {  // thread 0: two 2-D tensor copies per stage (out-of-range reads as 0)
        const int st = c % SW3_ST;
        tma::mbar_expect_tx(&sm.full[st], (unsigned)(sizeof(double) * KC * (RB + RPP)));
        tma::tensor_g2s_2d(&sm.a[st][0][0], &tm_f, (int)i0, c * KC, &sm.full[st]);
        tma::tensor_g2s_2d(&sm.b[st][0][0], &tm_m, 0, c * KC, &sm.full[st]);
    };
    if (threadIdx.x == 0)
        for (int c = 0; c < min(nch, SW3_ST); ++c) issue(c);
    // the epilogue's r x r factor, staged by asynchronous copies while the ring fills (its reads
    // were a dependent chain of global loads per output element)
    stage_uv<RP, SW3_T, PH>(sm.uv, a.uv, r);
    double acc[NTL][2];
#pragma unroll
    for (int t = 0; t < NTL; ++t) acc[t][0] = acc[t][1] = 0.0;
    const int fi = lane >> 2, fk = lane & 3;
    for (int c = 0; c < nch; ++c) {
        const int st = c % SW3_ST;
        tma::mbar_wait(&sm.full[st], (unsigned)((c / SW3_ST) & 1));
        // (k beyond n reads as zero in both operands: the padded k-steps add nothing)
#pragma unroll
        for (int ks = warp; ks < KC / 4; ks += SW3_W) {
            const int k = 4 * ks + fk;
            const double av = sm.a[st][k][fi];
#pragma unroll
            for (int t = 0; t < NTL; ++t) dmma_sw(acc[t], av, sm.b[st][k][8 * t + fi]);
        }
        __syncthreads();  // every warp is done with slot st
        if (threadIdx.x == 0 && c + SW3_ST < nch) {
            tma::fence_proxy_async();
            issue(c + SW3_ST);
        }
    }
    // warp partials (C fragment: row fi, columns 8 t + 2 fk + {0, 1}) summed in warp order
#pragma unroll
    for (int t = 0; t < NTL; ++t) {
        sm.red[warp][fi][8 * t + 2 * fk] = acc[t][0];
        sm.red[warp][fi][8 * t + 2 * fk + 1] = acc[t][1];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < RB * RP; e += SW3_T) {
        const int q = e / RP, jj = e % RP;
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < SW3_W; ++w) t += sm.red[w][q][jj];
        sm.tt[q][jj] = t;
    }
    stage_uv_wait();
    __syncthreads();
    for (int e = threadIdx.x; e < RB * RPP; e += SW3_T) {
        const int q = e / RPP, jj = e % RPP;
        if (q >= rb) continue;
        const int64_t i = i0 + q;
        if (jj >= r) {  // zero pad of the row-major core (phase 2's B operand)
            if constexpr (PH == 1) core_rm[i * RPP + jj] = 0.0;
            continue;
        }
        double c0 = 0.0, c1 = 0.0;  // two chains, summed once: a fixed order
#pragma unroll
        for (int m = 0; m < RP; m += 2) {
            c0 = fma(sm.tt[q][m], sm.uv[m][jj], c0);
            c1 = fma(sm.tt[q][m + 1], sm.uv[m + 1][jj], c1);
        }
        const double c = c0 + c1;
        if constexpr (PH == 1) {
            double out;
            if (a.op == SW_MUL) {
                out = c * a.dmat[i + n * jj];
            } else {
                const double den = a.e_col[jj] * a.e_row[i] + a.beta;
                if (den == 0.0) *a.flag = 1;
                out = c / den;
            }
            core_rm[i * RPP + jj] = out;
        } else {
            a.y[i + a.ldy * jj] = c;
        }
    }
}

// x (n x r, column stride ldx) -> xrm (n x RPP row-major, zero pad)
__global__ void to_rows_padded_kernel(const double* __restrict__ x, int64_t ldx, int64_t n, int r, int rpp,
                                      double* __restrict__ xrm) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * rpp; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = e / rpp;
        const int j = (int)(e % rpp);
        xrm[e] = j < r ? x[k + ldx * j] : 0.0;
    }
}

template <int RP>
void launch3_rp(const SandArgs& a, cudaStream_t s) {
    constexpr int KC = Sw3<RP>::KC, RPP = Sw3<RP>::RPP;
    const uint64_t n = (uint64_t)a.n;
    double* core_rm = a.core_out;               // n x RPP
    double* xrm = a.core_out + (size_t)n * RPP;  // n x RPP
    const size_t smem = sizeof(Sw3Smem<RP>);
    to_rows_padded_kernel<<<(unsigned)std::min<int64_t>(((int64_t)n * RPP + 255) / 256, 4096), 256, 0, s>>>(
        a.x, a.ldx, (int64_t)n, (int)a.r, RPP, xrm);
    CPHIFI_CHECK_LAUNCH();
    CUtensorMap tf1, tf2, tm1, tm2;
    const bool ok = encode_tmap_2d_f64(&tf1, a.ut, n, n, n, SW3_RB, KC) && encode_tmap_2d_f64(&tf2, a.u, n, n, n, SW3_RB, KC) &&
                    encode_tmap_2d_f64(&tm1, xrm, RPP, n, RPP, RPP, KC) &&
                    encode_tmap_2d_f64(&tm2, core_rm, RPP, n, RPP, RPP, KC);
    if (!ok) throw Error(CPHIFI_CUDA_ERROR, "sandwich: tensor map encoding failed");
    const unsigned grid = (unsigned)((a.n + SW3_RB - 1) / SW3_RB);
    func_attr_once((const void*)sandwich3_kernel<RP, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    func_attr_once((const void*)sandwich3_kernel<RP, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    sandwich3_kernel<RP, 1><<<grid, SW3_T, smem, s>>>(a, tf1, tm1, core_rm);
    CPHIFI_CHECK_LAUNCH();
    sandwich3_kernel<RP, 2><<<grid, SW3_T, smem, s>>>(a, tf2, tm2, core_rm);
    CPHIFI_CHECK_LAUNCH();
}

// ---- v5: v3 with the M operand multicast across a thread-block cluster ------------------------
// v3's CTAs (128 at config 2) each stream ALL of M (X or the core: n x (r + 8) doubles) next to
// their 8 rows of F: ~49 MB of L2 -> SM traffic per phase against 8 MB of F, and the phase waits
// on it (ncu: 11 us per phase, tensor pipe 27 %, L2 11 %).  Here the CL CTAs of a cluster share
// every M chunk: CTA q copies k-rows [q KC / CL, (q + 1) KC / CL) of the chunk and multicasts them
// into the same slot of every CTA of the cluster (its F box stays CTA-local), so a CTA pulls 1/CL
// of M from L2.  A slot is refilled only once every CTA of the cluster is done with it: each CTA
// arrives on the `empty` barrier of every peer (remote mbarrier arrive) and waits on its own
// (CL arrivals) before issuing into the slot.  Same fragments, warp split and summation order as
// v3: bit-identical to it.
template <int RP>
struct Sw5Smem {
    Sw3Smem<RP> s3;
    uint64_t empty[Sw3<RP>::ST];
};
__device__ __forceinline__ unsigned cluster_ctarank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n"
                 "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// arrive on the mbarrier at the same shared-memory offset in CTA `cta` of the cluster
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, unsigned cta) {
    unsigned remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(tma::smem_u32(bar)), "r"(cta));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(tma::smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 2-D tensor-map copy multicast to the CTAs of `mask` (same smem offsets, complete_tx on each
// CTA's barrier at the offset of `bar`)
__device__ __forceinline__ void tensor_g2s_2d_mc(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                                 uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(tma::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(tma::smem_u32(bar)), "h"(mask)
        : "memory");
}
template <int RP, int PH, int CL>
__global__ void __launch_bounds__(SW3_T) sandwich5_kernel(const SandArgs a, const __grid_constant__ CUtensorMap tm_f,
                                                          const __grid_constant__ CUtensorMap tm_m, double* core_rm) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Sw5Smem<RP>& sm5 = *reinterpret_cast<Sw5Smem<RP>*>(smem_raw);
    Sw3Smem<RP>& sm = sm5.s3;
    constexpr int KC = Sw3<RP>::KC, RPP = Sw3<RP>::RPP, NTL = Sw3<RP>::NTL, RB = SW3_RB, ST = Sw3<RP>::ST;
    constexpr int KS = KC / CL;  // k-rows of every M chunk this CTA copies for the cluster
    static_assert(KC % CL == 0 && (KS * RPP * 8) % 128 == 0, "multicast slices 128-byte aligned");
    const int64_t n = a.n;
    const int r = (int)a.r;
    const int64_t i0 = (int64_t)blockIdx.x * RB;
    const int rb = (int)min((int64_t)RB, n - i0);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nch = (int)((n + KC - 1) / KC);
    const unsigned q = cluster_ctarank();
    if (threadIdx.x == 0) {
        for (int st = 0; st < ST; ++st) {
            tma::mbar_init(&sm.full[st], 1);
            tma::mbar_init(&sm5.empty[st], CL);
        }
        tma::fence_mbar_init();
    }
    cluster_sync_all();  // every CTA's barriers initialised before a peer's multicast lands
    auto issue = [&](int c) {  // thread 0: own F box, this CTA's slice of the M chunk to the cluster
        const int st = c % ST;
        tma::mbar_expect_tx(&sm.full[st], (unsigned)(sizeof(double) * KC * (RB + RPP)));
        tma::tensor_g2s_2d(&sm.a[st][0][0], &tm_f, (int)i0, c * KC, &sm.full[st]);
        tensor_g2s_2d_mc(&sm.b[st][q * KS][0], &tm_m, 0, c * KC + (int)q * KS, &sm.full[st], (uint16_t)((1u << CL) - 1));
    };
    if (threadIdx.x == 0)
        for (int c = 0; c < min(nch, ST); ++c) issue(c);
    stage_uv<RP, SW3_T, PH>(sm.uv, a.uv, r);
    double acc[NTL][2];
#pragma unroll
    for (int t = 0; t < NTL; ++t) acc[t][0] = acc[t][1] = 0.0;
    const int fi = lane >> 2, fk = lane & 3;
    for (int c = 0; c < nch; ++c) {
        const int st = c % ST;
        tma::mbar_wait(&sm.full[st], (unsigned)((c / ST) & 1));
#pragma unroll
        for (int ks = warp; ks < KC / 4; ks += SW3_W) {
            const int k = 4 * ks + fk;
            const double av = sm.a[st][k][fi];
#pragma unroll
            for (int t = 0; t < NTL; ++t) dmma_sw(acc[t], av, sm.b[st][k][8 * t + fi]);
        }
        __syncthreads();  // every warp is done with slot st
        if (threadIdx.x == 0 && c + ST < nch) {
            for (unsigned p = 0; p < (unsigned)CL; ++p) mbar_arrive_cluster(&sm5.empty[st], p);
            mbar_wait_cluster(&sm5.empty[st], (unsigned)((c / ST) & 1));  // the whole cluster is done with st
            tma::fence_proxy_async();
            issue(c + ST);
        }
    }
#pragma unroll
    for (int t = 0; t < NTL; ++t) {
        sm.red[warp][fi][8 * t + 2 * fk] = acc[t][0];
        sm.red[warp][fi][8 * t + 2 * fk + 1] = acc[t][1];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < RB * RP; e += SW3_T) {
        const int qq = e / RP, jj = e % RP;
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < SW3_W; ++w) t += sm.red[w][qq][jj];
        sm.tt[qq][jj] = t;
    }
    stage_uv_wait();
    __syncthreads();
    for (int e = threadIdx.x; e < RB * RPP; e += SW3_T) {
        const int qq = e / RPP, jj = e % RPP;
        if (qq >= rb) continue;
        const int64_t i = i0 + qq;
        if (jj >= r) {
            if constexpr (PH == 1) core_rm[i * RPP + jj] = 0.0;
            continue;
        }
        double c0 = 0.0, c1 = 0.0;  // two chains, summed once: a fixed order (as v3)
#pragma unroll
        for (int m = 0; m < RP; m += 2) {
            c0 = fma(sm.tt[qq][m], sm.uv[m][jj], c0);
            c1 = fma(sm.tt[qq][m + 1], sm.uv[m + 1][jj], c1);
        }
        const double c = c0 + c1;
        if constexpr (PH == 1) {
            double out;
            if (a.op == SW_MUL) {
                out = c * a.dmat[i + n * jj];
            } else {
                const double den = a.e_col[jj] * a.e_row[i] + a.beta;
                if (den == 0.0) *a.flag = 1;
                out = c / den;
            }
            core_rm[i * RPP + jj] = out;
        } else {
            a.y[i + a.ldy * jj] = c;
        }
    }
    cluster_sync_all();  // no CTA leaves while a peer may still arrive on its barriers
}

template <int RP, int PH, int CL>
void launch5_ph(const SandArgs& a, const CUtensorMap& tf, const CUtensorMap& tm, double* core_rm, unsigned grid,
                cudaStream_t s) {
    auto kern = sandwich5_kernel<RP, PH, CL>;
    const size_t smem = sizeof(Sw5Smem<RP>);
    func_attr_once((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(SW3_T, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CPHIFI_CUDA(cudaLaunchKernelEx(&cfg, kern, a, tf, tm, core_rm));
}

// false: no cluster size divides the grid (the caller takes v3)
template <int RP>
bool launch5_rp(const SandArgs& a, int cl_max, cudaStream_t s) {
    constexpr int KC = Sw3<RP>::KC, RPP = Sw3<RP>::RPP;
    const uint64_t n = (uint64_t)a.n;
    const unsigned grid = (unsigned)((a.n + SW3_RB - 1) / SW3_RB);
    int cl = 8;
    while (cl > 1 && (cl > cl_max || grid % cl != 0 || KC % cl != 0 || ((KC / cl) * RPP * 8) % 128 != 0)) cl /= 2;
    if (cl < 2) return false;
    double* core_rm = a.core_out;
    double* xrm = a.core_out + (size_t)n * RPP;
    to_rows_padded_kernel<<<(unsigned)std::min<int64_t>(((int64_t)n * RPP + 255) / 256, 4096), 256, 0, s>>>(
        a.x, a.ldx, (int64_t)n, (int)a.r, RPP, xrm);
    CPHIFI_CHECK_LAUNCH();
    CUtensorMap tf1, tf2, tm1, tm2;
    const uint32_t ks = (uint32_t)(KC / cl);
    const bool ok = encode_tmap_2d_f64(&tf1, a.ut, n, n, n, SW3_RB, KC) && encode_tmap_2d_f64(&tf2, a.u, n, n, n, SW3_RB, KC) &&
                    encode_tmap_2d_f64(&tm1, xrm, RPP, n, RPP, RPP, ks) &&
                    encode_tmap_2d_f64(&tm2, core_rm, RPP, n, RPP, RPP, ks);
    if (!ok) throw Error(CPHIFI_CUDA_ERROR, "sandwich: tensor map encoding failed");
    switch (cl) {
        case 8:
            launch5_ph<RP, 1, 8>(a, tf1, tm1, core_rm, grid, s);
            launch5_ph<RP, 2, 8>(a, tf2, tm2, core_rm, grid, s);
            break;
        case 4:
            launch5_ph<RP, 1, 4>(a, tf1, tm1, core_rm, grid, s);
            launch5_ph<RP, 2, 4>(a, tf2, tm2, core_rm, grid, s);
            break;
        default:
            launch5_ph<RP, 1, 2>(a, tf1, tm1, core_rm, grid, s);
            launch5_ph<RP, 2, 2>(a, tf2, tm2, core_rm, grid, s);
            break;
    }
    return true;
}

template <int RP, int RB, int PH>
void launch2_t(const SandArgs& a, cudaStream_t s) {
    auto kern = sandwich2_kernel<RP, RB, PH>;
    const size_t smem = sizeof(Sw2Smem<RP, RB>);
    func_attr_once((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    constexpr int KC = Sw2<RP>::KC;
    const uint64_t n = (uint64_t)a.n;
    CUtensorMap tf, tm;  // F = U or U' (n x n), M = X (ld ldx) or core (ld n); r columns of M
    const bool ok = encode_tmap_2d_f64(&tf, PH == 1 ? a.u : a.ut, n, n, n, KC, RB) &&
                    encode_tmap_2d_f64(&tm, PH == 1 ? a.x : a.core, n, (uint64_t)a.r, PH == 1 ? (uint64_t)a.ldx : n, KC, RP);
    if (!ok) throw Error(CPHIFI_CUDA_ERROR, "sandwich: tensor map encoding failed");
    kern<<<(unsigned)((a.n + RB - 1) / RB), SW2_T, smem, s>>>(a, tf, tm);
    CPHIFI_CHECK_LAUNCH();
}
template <int RP, int PH>
void launch2_rb(const SandArgs& a, int rb, cudaStream_t s) {
    // accumulators per thread: RP / 8 columns x RB rows <= 32 (RB = 16 measured slower)
    constexpr int RBMAX = 256 / RP >= 8 ? 8 : 256 / RP;
    if (rb >= 8 && RBMAX >= 8) launch2_t<RP, (RBMAX >= 8 ? 8 : RBMAX), PH>(a, s);
    else if (rb >= 4 && RBMAX >= 4) launch2_t<RP, (RBMAX >= 4 ? 4 : RBMAX), PH>(a, s);
    else if (rb >= 2) launch2_t<RP, 2, PH>(a, s);
    else launch2_t<RP, 1, PH>(a, s);
}
template <int PH>
void launch2_ph(const SandArgs& a, int rb, cudaStream_t s) {
    switch (a.rp) {
        case 8: launch2_rb<8, PH>(a, rb, s); break;
        case 16: launch2_rb<16, PH>(a, rb, s); break;
        case 32: launch2_rb<32, PH>(a, rb, s); break;
        case 64: launch2_rb<64, PH>(a, rb, s); break;
        default: throw_invalid("sandwich: padded rank must be 8, 16, 32 or 64");
    }
}

template <int RP, int RB, int PH>
void launch_t(const SandArgs& a, cudaStream_t s) {
    auto kern = sandwich_kernel<RP, RB, PH>;
    const size_t smem = sizeof(SwSmem<RP, RB>);
    func_attr_once((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const unsigned grid = (unsigned)((a.n + RB - 1) / RB);
    kern<<<grid, SW_T, smem, s>>>(a);
    CPHIFI_CHECK_LAUNCH();
}

template <int RP, int PH>
void launch_rb(const SandArgs& a, int rb, cudaStream_t s) {
    switch (rb) {
        case 1: launch_t<RP, 1, PH>(a, s); break;
        case 2: launch_t<RP, 2, PH>(a, s); break;
        case 4: launch_t<RP, 4, PH>(a, s); break;
        default: launch_t<RP, 8, PH>(a, s); break;
    }
}

template <int PH>
void launch_ph(const SandArgs& a, int rb, cudaStream_t s) {
    switch (a.rp) {
        case 8: launch_rb<8, PH>(a, rb, s); break;
        case 16: launch_rb<16, PH>(a, rb, s); break;
        case 32: launch_rb<32, PH>(a, rb, s); break;
        case 64: launch_rb<64, PH>(a, rb, s); break;
        default: throw_invalid("sandwich: padded rank must be 8, 16, 32 or 64");
    }
}

// ---- v4: split-K DMMA, one tile per CTA, partial sums reduced by the last CTA of each row block ----
// v3's CTAs each stream ALL of M (X or the core: n x (r + 8) doubles, 327 KB at config 2) next to
// their 8 rows of F, so a phase moves ~42 MB through L2 for a 67 MFLOP product (~10 us).  Here CTA
// (ib, kb) takes the BI x BK block of F and the BK x r block of M once, as 2 x 8 TMA boxes of 16 k
// with the 128-byte swizzle, runs the BI x RP x BK product on DMMA (8 warps, output tiles split
// between them, full k per tile) and stores its partial block; the last CTA of row block ib
// (arrival counter, reset by that CTA) sums the nkb partials in kb order and runs the epilogue (x U_V
// or U_V', the element-wise op) for its BI rows.  Both operands are read k-contiguous — F(i, k) =
// G(k, i) with G = U (phase 1: F = U') or U' (phase 2: F = U), M = X or the core column-major — so a
// box row is 16 consecutive k of one i (or j) and the swizzle (chunk ^ row mod 8) spreads an
// m8n8k4 fragment's 8 rows x 2 chunks over all bank groups: 2 wavefronts per fragment, the minimum.
// X is read in place (no transposed copy); fixed summation order throughout: bit-reproducible.
constexpr int SW4_T = 256, SW4_W = 8, SW4_BI = 32, SW4_BK = 128, SW4_KB = 16, SW4_NB = SW4_BK / SW4_KB;
template <int RP>
struct Sw4Smem {
    double a[SW4_NB][SW4_BI][SW4_KB];  // box b: G(k0 + 16 b + k, i0 + i), swizzled 16-byte chunks
    double b[SW4_NB][RP][SW4_KB];      // box b: M(k0 + 16 b + k, j), swizzled
    double uv[RP][RP + 1];
    double c[SW4_BI][RP + 1];
    uint64_t full;
    unsigned last;
};
// element (row y, k) of a swizzled box of 16-double rows
__device__ __forceinline__ int swz(int y, int k) { return y * SW4_KB + ((((k >> 1) ^ (y & 7))) << 1) + (k & 1); }
// scratch (doubles): core column-major n x r | partials nkb x n x RP | row-block counters
template <int RP, int PH>
__global__ void __launch_bounds__(SW4_T, 2) sandwich4_kernel(const SandArgs a, const __grid_constant__ CUtensorMap tm_g,
                                                             const __grid_constant__ CUtensorMap tm_m) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    using SM = Sw4Smem<RP>;
    // the swizzled boxes need 1024-byte alignment (the launch adds the slack)
    // (offset arithmetic on smem_raw keeps the accesses in the shared state space: LDS, not generic)
    const unsigned mis = static_cast<unsigned>(__cvta_generic_to_shared(smem_raw)) & 1023u;
    SM& sm = *reinterpret_cast<SM*>(smem_raw + ((1024u - mis) & 1023u));
    constexpr int BI = SW4_BI, BK = SW4_BK, TJ = RP / 8, NTL = (BI / 8) * TJ, TPW = NTL / SW4_W;
    static_assert(NTL % SW4_W == 0, "output tiles split evenly over the warps");
    const int64_t n = a.n;
    const int r = (int)a.r;
    const int nkb = (int)((n + BK - 1) / BK);
    const int kb = blockIdx.x % nkb, ib = blockIdx.x / nkb;
    const int64_t i0 = (int64_t)ib * BI, k0 = (int64_t)kb * BK;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, kq = lane & 3;
    double* core = a.core_out;                                  // n x r column-major
    double* part = a.core_out + n * RP;                         // nkb x n x RP
    unsigned* cnt = reinterpret_cast<unsigned*>(part + (int64_t)nkb * n * RP);
    if (tid == 0) {
        tma::mbar_init(&sm.full, 1);
        tma::fence_mbar_init();
        tma::mbar_expect_tx(&sm.full, (unsigned)(sizeof(double) * SW4_NB * SW4_KB * (BI + RP)));
#pragma unroll
        for (int bx = 0; bx < SW4_NB; ++bx) {
            tma::tensor_g2s_2d(&sm.a[bx][0][0], &tm_g, (int)(k0 + SW4_KB * bx), (int)i0, &sm.full);
            tma::tensor_g2s_2d(&sm.b[bx][0][0], &tm_m, (int)(k0 + SW4_KB * bx), 0, &sm.full);
        }
    }
    __syncthreads();  // barrier initialised
    stage_uv<RP, SW4_T, PH>(sm.uv, a.uv, r);  // every CTA: the last one of its row block needs it at once
    tma::mbar_wait(&sm.full, 0);
    double acc[TPW][2];
#pragma unroll
    for (int t = 0; t < TPW; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll
    for (int bx = 0; bx < SW4_NB; ++bx) {
        const double* ab = &sm.a[bx][0][0];
        const double* bb = &sm.b[bx][0][0];
#pragma unroll
        for (int kk = 0; kk < SW4_KB; kk += 4) {
            const int k = kk + kq;
#pragma unroll
            for (int t = 0; t < TPW; ++t) {
                const int tile = warp + SW4_W * t, ti = tile / TJ, tj = tile % TJ;
                dmma_sw(acc[t], ab[swz(8 * ti + g, k)], bb[swz(8 * tj + g, k)]);
            }
        }
    }
#pragma unroll
    for (int t = 0; t < TPW; ++t) {
        const int tile = warp + SW4_W * t, ti = tile / TJ, tj = tile % TJ;
        const int64_t row = i0 + 8 * ti + g;
        if (row < n)
            __stcg(reinterpret_cast<double2*>(part + ((int64_t)kb * n + row) * RP + 8 * tj + 2 * kq),
                   make_double2(acc[t][0], acc[t][1]));
    }
    __syncthreads();  // the CTA's partial stores precede thread 0's release
    if (tid == 0) {
        unsigned old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt + ib) : "memory");
        sm.last = old == (unsigned)nkb - 1;
        if (sm.last) cnt[ib] = 0;
    }
    __syncthreads();
    if (!sm.last) {
        stage_uv_wait();
        return;
    }
    const int rb = (int)min((int64_t)BI, n - i0);
    constexpr int PER = BI * RP / SW4_T;  // partial sums per thread, loads all in flight
    static_assert(BI * RP % SW4_T == 0, "even split");
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int e = tid + SW4_T * u, q = e / RP, jj = e % RP;
        double v = 0.0;
        if (q < rb) {
            double pv[8];
            for (int k8 = 0; k8 < nkb; k8 += 8) {
#pragma unroll
                for (int t = 0; t < 8; ++t) pv[t] = k8 + t < nkb ? __ldcg(part + ((int64_t)(k8 + t) * n + i0 + q) * RP + jj) : 0.0;
#pragma unroll
                for (int t = 0; t < 8; ++t) v += pv[t];  // kb order
            }
        }
        sm.c[q][jj] = v;
    }
    stage_uv_wait();
    __syncthreads();
    for (int e = tid; e < BI * RP; e += SW4_T) {
        const int jj = e / BI, q = e % BI;  // consecutive threads: consecutive rows (column-major outputs)
        if (q >= rb || jj >= r) continue;
        const int64_t i = i0 + q;
        double c0 = 0.0, c1 = 0.0;  // two chains, summed once: a fixed order
#pragma unroll
        for (int m = 0; m < RP; m += 2) {
            c0 = fma(sm.c[q][m], sm.uv[m][jj], c0);
            c1 = fma(sm.c[q][m + 1], sm.uv[m + 1][jj], c1);
        }
        const double c = c0 + c1;
        if constexpr (PH == 1) {
            double out;
            if (a.op == SW_MUL) {
                out = c * a.dmat[i + n * jj];
            } else {
                const double den = a.e_col[jj] * a.e_row[i] + a.beta;
                if (den == 0.0) *a.flag = 1;
                out = c / den;
            }
            core[i + n * jj] = out;
        } else {
            a.y[i + a.ldy * jj] = c;
        }
    }
}

template <int RP>
bool launch4_rp(const SandArgs& a, cudaStream_t s) {
    const size_t smem = sizeof(Sw4Smem<RP>) + 1024;  // + alignment slack for the swizzled boxes
    const uint64_t n = (uint64_t)a.n;
    CUtensorMap tg1, tg2, tm1, tm2;
    // phase 1: F = U' -> G = U; M = X.  phase 2: F = U -> G = U'; M = the core (n x r, ld n)
    const bool ok = encode_tmap_2d_f64(&tg1, a.u, n, n, n, SW4_KB, SW4_BI, true) &&
                    encode_tmap_2d_f64(&tg2, a.ut, n, n, n, SW4_KB, SW4_BI, true) &&
                    encode_tmap_2d_f64(&tm1, a.x, n, (uint64_t)a.r, (uint64_t)a.ldx, SW4_KB, RP, true) &&
                    encode_tmap_2d_f64(&tm2, a.core_out, n, (uint64_t)a.r, n, SW4_KB, RP, true);
    if (!ok) return false;
    func_attr_once((const void*)sandwich4_kernel<RP, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    func_attr_once((const void*)sandwich4_kernel<RP, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t nkb = (a.n + SW4_BK - 1) / SW4_BK, nib = (a.n + SW4_BI - 1) / SW4_BI;
    sandwich4_kernel<RP, 1><<<(unsigned)(nkb * nib), SW4_T, smem, s>>>(a, tg1, tm1);
    CPHIFI_CHECK_LAUNCH();
    sandwich4_kernel<RP, 2><<<(unsigned)(nkb * nib), SW4_T, smem, s>>>(a, tg2, tm2);
    CPHIFI_CHECK_LAUNCH();
    return true;
}

}  // namespace

int64_t sandwich_rp(int64_t r) { return pow2_at_least(r, 8); }

bool sandwich_supported(int64_t n, int64_t r) {
    if (const char* e = std::getenv("CPHIFI_SANDWICH")) {
        if (std::atoi(e) == 0) return false;
    }
    return r >= 1 && r <= 64 && n >= 1 && n <= 2048;
}

__global__ void transpose_kernel(const double* __restrict__ a, int64_t n, double* __restrict__ at) {
    __shared__ double t[32][33];
    const int64_t bx = (int64_t)blockIdx.x * 32, by = (int64_t)blockIdx.y * 32;
    for (int yy = threadIdx.y; yy < 32; yy += 8) {
        const int64_t i = bx + threadIdx.x, j = by + yy;
        if (i < n && j < n) t[yy][threadIdx.x] = a[i + n * j];
    }
    __syncthreads();
    for (int yy = threadIdx.y; yy < 32; yy += 8) {
        const int64_t i = by + threadIdx.x, j = bx + yy;  // at(i, j) = a(j, i)
        if (i < n && j < n) at[i + n * j] = t[threadIdx.x][yy];
    }
}

__global__ void scale_cols_kernel(const double* __restrict__ a, int64_t n, const double* __restrict__ d,
                                  double* __restrict__ out) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x)
        out[e] = a[e] * d[e / n];
}

__global__ void scale_rows_kernel(const double* __restrict__ a, int64_t n, const double* __restrict__ d,
                                  double* __restrict__ out) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x)
        out[e] = a[e] * d[e % n];
}
void scale_rows(const double* a, int64_t n, const double* d, double* out, cudaStream_t s) {
    scale_rows_kernel<<<(unsigned)std::min<int64_t>((n * n + 255) / 256, 4096), 256, 0, s>>>(a, n, d, out);
    CPHIFI_CHECK_LAUNCH();
}

void scale_cols(const double* a, int64_t n, const double* d, double* out, cudaStream_t s) {
    scale_cols_kernel<<<(unsigned)std::min<int64_t>((n * n + 255) / 256, 4096), 256, 0, s>>>(a, n, d, out);
    CPHIFI_CHECK_LAUNCH();
}

// sigma_j -> 1 / sigma_j, or 0 below r eps sigma_max (a pseudo-inverse on the eigenbasis)
__global__ void invert_spectrum_kernel(double* sv, int64_t r) {
    double mx = 0.0;
    for (int64_t j = 0; j < r; ++j) mx = fmax(mx, sv[j]);
    const double tau = mx * (double)r * 2.220446049250313e-16;
    for (int64_t j = threadIdx.x; j < r; j += blockDim.x) sv[j] = (sv[j] > tau && mx > 0.0) ? 1.0 / sv[j] : 0.0;
}
void invert_spectrum(double* sv, int64_t r, cudaStream_t s) {
    invert_spectrum_kernel<<<1, 64, 0, s>>>(sv, r);
    CPHIFI_CHECK_LAUNCH();
}
__global__ void scale_columns_kernel(double* a, int64_t m, int64_t r, const double* d) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * r; e += (int64_t)gridDim.x * blockDim.x)
        a[e] *= d[e / m];
}
void scale_columns(double* a, int64_t m, int64_t r, const double* d, cudaStream_t s) {
    scale_columns_kernel<<<(unsigned)std::min<int64_t>((m * r + 255) / 256, 2048), 256, 0, s>>>(a, m, r, d);
    CPHIFI_CHECK_LAUNCH();
}

// Eigenbasis preconditioner in one launch (small r): z~(i,:) = ((r~(i,:) U_V) o D(i,:)) U_V' for a
// block of 32 rows per CTA.  Lane = row (column-major r~, D, z~: every warp access is one
// contiguous 256-byte column segment), warp w = columns [w JT, (w + 1) JT); the r~ block and the
// intermediate t are staged column-major in shared memory (lanes on consecutive rows: conflict-
// free), U_V' row-major so a thread's JT columns of U_V(m, :) are one broadcast vector load.
// Fixed summation order (m ascending), as the reference's GEMMs per row.
constexpr int PR_T = 256, PR_RB = 32, PR_W = PR_T / 32;
template <int JT>
__global__ void __launch_bounds__(PR_T) precond_rot_kernel(const double* __restrict__ rt, const double* __restrict__ uv,
                                                           const double* __restrict__ dmat, int64_t n, int r,
                                                           double* __restrict__ zt) {
    constexpr int RP = JT * PR_W;  // padded rank (columns)
    constexpr int LDU = RP + 2;    // padded row stride: the transposed staging writes spread over banks
    extern __shared__ __align__(16) double prs[];
    double* suv = prs;                  // suv[m * LDU + j] = U_V(m, j)   (0 beyond r)
    double* sr = suv + RP * LDU;        // sr[m * PR_RB + q] = r~(i0 + q, m), later t
    const int64_t i0 = (int64_t)blockIdx.x * PR_RB;
    const int q = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t i = i0 + q;
    const bool row_ok = i < n;
    // every load of the CTA issued before the first use (unrolled): U_V read coalesced (m fastest)
#pragma unroll
    for (int k = 0; k < (RP * RP + PR_T - 1) / PR_T; ++k) {
        const int e = threadIdx.x + k * PR_T;
        const int m = e % RP, j = e / RP;
        if (e < RP * RP) suv[m * LDU + j] = (m < r && j < r) ? uv[m + (int64_t)r * j] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < JT; ++k) {
        const int m = w + k * PR_W;
        sr[m * PR_RB + q] = (row_ok && m < r) ? rt[i + n * m] : 0.0;
    }
    __syncthreads();
    double acc[JT];
#pragma unroll
    for (int u = 0; u < JT; ++u) acc[u] = 0.0;
    const int j0 = w * JT;
    for (int m = 0; m < r; ++m) {
        const double a = sr[m * PR_RB + q];
        const double* um = suv + m * LDU + j0;
#pragma unroll
        for (int u = 0; u < JT; ++u) acc[u] = fma(a, um[u], acc[u]);
    }
#pragma unroll
    for (int u = 0; u < JT; ++u) {
        const int j = j0 + u;
        if (j < r && row_ok) acc[u] *= dmat[i + n * j];
    }
    __syncthreads();  // everyone is done reading r~
#pragma unroll
    for (int u = 0; u < JT; ++u) sr[(j0 + u) * PR_RB + q] = acc[u];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < JT; ++u) acc[u] = 0.0;
    for (int m = 0; m < r; ++m) {  // z~(i, j) = sum_m t(i, m) U_V(j, m)
        const double t = sr[m * PR_RB + q];
#pragma unroll
        for (int u = 0; u < JT; ++u) acc[u] = fma(t, suv[(j0 + u) * LDU + m], acc[u]);
    }
    if (row_ok) {
#pragma unroll
        for (int u = 0; u < JT; ++u)
            if (j0 + u < r) zt[i + n * (j0 + u)] = acc[u];
    }
}
template <int JT>
void launch_precond_rot(const double* rt, const double* uv, const double* dmat, int64_t n, int64_t r, double* zt,
                        cudaStream_t s) {
    constexpr int RP = JT * PR_W;
    const size_t smem = sizeof(double) * (RP * (RP + 2) + RP * PR_RB);
    func_attr_once((const void*)precond_rot_kernel<JT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    precond_rot_kernel<JT><<<(unsigned)((n + PR_RB - 1) / PR_RB), PR_T, smem, s>>>(rt, uv, dmat, n, (int)r, zt);
    CPHIFI_CHECK_LAUNCH();
}
void precond_rot_small(const double* rt, const double* uv, const double* dmat, int64_t n, int64_t r, double* zt,
                       cudaStream_t s) {
    if (r <= 8) launch_precond_rot<1>(rt, uv, dmat, n, r, zt, s);
    else if (r <= 16) launch_precond_rot<2>(rt, uv, dmat, n, r, zt, s);
    else if (r <= 32) launch_precond_rot<4>(rt, uv, dmat, n, r, zt, s);
    else if (r <= 64) launch_precond_rot<8>(rt, uv, dmat, n, r, zt, s);
    else throw_invalid("precond_rot_small: rank above 64");
}

void transpose_sq(const double* a, int64_t n, double* at, cudaStream_t s) {
    const unsigned g = (unsigned)((n + 31) / 32);
    transpose_kernel<<<dim3(g, g), dim3(32, 8), 0, s>>>(a, n, at);
    CPHIFI_CHECK_LAUNCH();
}

int64_t sandwich_scratch_doubles(int64_t n, int64_t r) {
    const int64_t rp = sandwich_rp(r);
    const int64_t nkb = (n + SW4_BK - 1) / SW4_BK, nib = (n + SW4_BI - 1) / SW4_BI;
    const int64_t v4 = n * rp + nkb * n * rp + (nib + 1) / 2 + 1;  // core, partials, counters
    return std::max<int64_t>(2 * n * (rp + 8), v4);  // v3: row-major core and X copy, pitch rp + 8
}

int64_t sandwich_counter_offset(int64_t n, int64_t r) {
    const int64_t rp = sandwich_rp(r);
    return n * rp + (n + SW4_BK - 1) / SW4_BK * n * rp;
}

void sandwich(SandArgs a, int num_sms, cudaStream_t s) {
    a.rp = sandwich_rp(a.r);
    a.core = a.core_out;
    // v3 (DMMA) from n = 512 on: config 2 (n = 1024, r = 32) decoupled 35.7 -> 31.4 us; at n = 200
    // (config 0) its 25 CTAs lose to v2 (18.7 vs 14.3 us)
    bool v3 = a.n >= 512 && a.n % 2 == 0 && reinterpret_cast<uintptr_t>(a.u) % 16 == 0 &&
              reinterpret_cast<uintptr_t>(a.ut) % 16 == 0 && reinterpret_cast<uintptr_t>(a.core_out) % 16 == 0;
    if (const char* e = std::getenv("CPHIFI_SANDWICH_V3")) v3 = v3 && std::atoi(e) != 0;
    // v4 (split-K DMMA): opt-in (CPHIFI_SANDWICH_V4=1) — measured slower than v3 at config 2
    // (15.6 + 14.2 us against 10.3 + 9.1 per phase: its CTAs sit mostly idle behind the last-arrival
    // reduction of each row block)
    bool v4 = false;
    if (const char* e = std::getenv("CPHIFI_SANDWICH_V4")) v4 = v3 && a.rp >= 16 && std::atoi(e) != 0;
    if (v4) {  // (false: a tensor map could not be encoded, e.g. X not 16-byte aligned)
        switch (a.rp) {
            case 16: if (launch4_rp<16>(a, s)) return; break;
            case 32: if (launch4_rp<32>(a, s)) return; break;
            case 64: if (launch4_rp<64>(a, s)) return; break;
            default: break;
        }
    }
    // v5 (v3 + cluster multicast of the M chunks): opt-in, CPHIFI_SANDWICH_V5=k caps the cluster
    // size at k.  Measured slower at config 2 (decoupled 26.1 us with v3; v5 with clusters of 2 / 4
    // / 8: 33.2 / 35.3 / 68.1 us — the cluster-wide slot release per chunk serialises the CTAs the
    // per-CTA rings kept independent; profiles/round2c/sandwich_v5.txt)
    int v5 = 0;
    if (const char* e = std::getenv("CPHIFI_SANDWICH_V5")) v5 = std::atoi(e);
    if (v3 && v5 >= 2) {
        bool done = false;
        switch (a.rp) {
            case 8: done = launch5_rp<8>(a, v5, s); break;
            case 16: done = launch5_rp<16>(a, v5, s); break;
            case 32: done = launch5_rp<32>(a, v5, s); break;
            case 64: done = launch5_rp<64>(a, v5, s); break;
            default: break;
        }
        if (done) return;
    }
    if (v3) {
        switch (a.rp) {
            case 8: launch3_rp<8>(a, s); return;
            case 16: launch3_rp<16>(a, s); return;
            case 32: launch3_rp<32>(a, s); return;
            case 64: launch3_rp<64>(a, s); return;
            default: break;
        }
    }
    // rows per CTA: about two CTAs per SM, at most 8
    int rb = 1;
    while (rb < 8 && (a.n + rb - 1) / rb > 2 * num_sms) rb *= 2;
    bool v2 = a.n % 2 == 0 && a.ldx % 2 == 0 && reinterpret_cast<uintptr_t>(a.u) % 16 == 0 &&
              reinterpret_cast<uintptr_t>(a.ut) % 16 == 0 && reinterpret_cast<uintptr_t>(a.x) % 16 == 0 &&
              reinterpret_cast<uintptr_t>(a.core_out) % 16 == 0;
    if (const char* e = std::getenv("CPHIFI_SANDWICH_V1")) v2 = v2 && std::atoi(e) == 0;
    if (v2) {  // core column-major n x r (v2 layout); about one CTA per SM (each CTA streams all
               // of X / core from L2, so fewer, taller CTAs cut that traffic)
        int rb2 = 1;
        while (rb2 < 8 && (a.n + rb2 - 1) / rb2 > num_sms) rb2 *= 2;
        if (const char* e = std::getenv("CPHIFI_SANDWICH_RB")) rb2 = std::atoi(e);
        launch2_ph<1>(a, rb2, s);
        launch2_ph<2>(a, rb2, s);
        return;
    }
    launch_ph<1>(a, rb, s);
    launch_ph<2>(a, rb, s);
}

}  // namespace cphifi
