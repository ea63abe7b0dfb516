// k_dense.cu — FP64 tensor-core (DMMA m8n8k4) contractions for sm_100a.
//
// tcgen05.mma has no f64 kind, so the FP64 tensor path on B200 is the warp-level
// `mma.sync.aligned.m8n8k4.row.col.f64` (SASS: DMMA.8x8x4).  These kernels cover every
// dense contraction on the hot path:
//   * K*X, K*Yhat + lambda*Xhat + rho*x   (unaligned.hpp:106,112-114)
//   * U_K' X, (.)U_V .* D, U_K(.), (.)U_V' (unaligned.hpp:137; aligned.hpp:44-53)
//   * dense MTTKRP T_(1) Z for k = 0      (tensor.hpp:174-182) with Z generated on the fly
// Split-K partial sums are reduced in a FIXED order (thread-block cluster + distributed
// shared memory for the GEMMs, an ordered second pass for the MTTKRP), so results are
// bit-reproducible run to run.
#include <cooperative_groups.h>

#include <map>

#include "kernels.cuh"
#include "tma.cuh"

namespace cg = cooperative_groups;

namespace cphifi {
namespace {

constexpr int BM = 64;       // rows per CTA tile (4 warps x 16 rows)
constexpr int BK = 32;       // K per pipeline stage
constexpr int NT = 128;      // threads per CTA
constexpr int STAGES = 3;
constexpr int APAD = BM + 4; // smem row pitch (doubles); == 4 mod 16 -> conflict-free frags

template <int BN, int BMv = BM, int ST = STAGES>
struct GemmSmem {
    double a[ST][BK][BMv + 4];  // pitch == 4 mod 16 doubles: conflict-free fragment loads
    double b[ST][BK][BN + 4];
};

// MTTKRP tile shape: 128 rows (8 warps x 16), 4 cp.async stages (one CTA per SM)
constexpr int BMM = 128;
constexpr int NTM = 256;
constexpr int STM = 4;

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    int sz = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// A tile: sm.a[st][kk][ii] = A(i0+ii, k0+kk); zero outside [m) x [k0, kend)
template <int BN>
__device__ __forceinline__ void load_a(GemmSmem<BN>& sm, int st, const double* __restrict__ a,
                                       int64_t a_rs, int64_t a_cs, int64_t m, int64_t i0,
                                       int64_t k0, int64_t kend) {
    if (a_rs == 1) {
        for (int e = threadIdx.x; e < BM * BK; e += NT) {
            const int ii = e % BM, kk = e / BM;
            const int64_t i = i0 + ii, kx = k0 + kk;
            const bool p = (i < m) && (kx < kend);
            cp_async8(&sm.a[st][kk][ii], p ? a + i + kx * a_cs : a, p);
        }
    } else {
        for (int e = threadIdx.x; e < BM * BK; e += NT) {
            const int kk = e % BK, ii = e / BK;
            const int64_t i = i0 + ii, kx = k0 + kk;
            const bool p = (i < m) && (kx < kend);
            cp_async8(&sm.a[st][kk][ii], p ? a + i * a_rs + kx * a_cs : a, p);
        }
    }
}

template <int BN>
__device__ __forceinline__ void load_b(GemmSmem<BN>& sm, int st, const double* __restrict__ b,
                                       int64_t b_rs, int64_t b_cs, int64_t n, int64_t j0,
                                       int64_t k0, int64_t kend) {
    if (b_cs == 1) {
        for (int e = threadIdx.x; e < BN * BK; e += NT) {
            const int jj = e % BN, kk = e / BN;
            const int64_t j = j0 + jj, kx = k0 + kk;
            const bool p = (j < n) && (kx < kend);
            cp_async8(&sm.b[st][kk][jj], p ? b + kx * b_rs + j : b, p);
        }
    } else {
        for (int e = threadIdx.x; e < BN * BK; e += NT) {
            const int kk = e % BK, jj = e / BK;
            const int64_t j = j0 + jj, kx = k0 + kk;
            const bool p = (j < n) && (kx < kend);
            cp_async8(&sm.b[st][kk][jj], p ? b + kx * b_rs + j * b_cs : b, p);
        }
    }
}

template <int BN, int BMv = BM, int ST = STAGES>
__device__ __forceinline__ void mma_stage(const GemmSmem<BN, BMv, ST>& sm, int st, double (&acc)[2][BN / 8][2]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int kq = lane & 3, g = lane >> 2;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
        const int kr = ks * 4 + kq;
        const double a0 = sm.a[st][kr][warp * 16 + g];
        const double a1 = sm.a[st][kr][warp * 16 + 8 + g];
#pragma unroll
        for (int nf = 0; nf < BN / 8; ++nf) {
            const double bv = sm.b[st][kr][nf * 8 + g];
            dmma(acc[0][nf], a0, bv);
            dmma(acc[1][nf], a1, bv);
        }
    }
}

__device__ __forceinline__ void epilogue_store(const GemmArgs& g, int64_t i, int64_t j, double v) {
    if (i >= g.m) return;
    if (j < g.n) {
        double out = v;
        switch (g.epi) {
            case EPI_AXPY2: {
                const int64_t e = i + g.ld_e * j;
                out = v + g.beta1 * g.e1[e];
                out = out + g.beta2 * g.e2[e];
                break;
            }
            case EPI_HADAMARD:
                out = v * g.e1[i + g.ld_e * j];
                break;
            case EPI_SCALE_DIV: {
                const double den = g.e_col[j] * g.e_row[i] + g.beta1;
                if (den == 0.0) *g.flag = 1;
                out = v / den;
                break;
            }
            case EPI_ROWSCALE: {
                const double e = g.e1 ? g.e1[i + g.ld_e * j] : 0.0;
                out = g.e_row[i] * (v + g.beta1 * e) + g.beta2 * e;
                break;
            }
            default:
                break;
        }
        if (g.c) g.c[i * g.c_rs + j * g.c_cs] = out;
        if (g.c2) g.c2[i * g.ld2 + j] = out;
    } else if (g.c2 && j < g.ld2) {
        g.c2[i * g.ld2 + j] = 0.0;
    }
}

// grid: (ceil(m/BM), S, ceil(n/BN)); cluster (1, S, 1) splits K across the S CTAs.
template <int BN>
__global__ void __launch_bounds__(NT) gemm_dmma_kernel(const GemmArgs g) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    GemmSmem<BN>& sm = *reinterpret_cast<GemmSmem<BN>*>(smem_raw);
    const int S = gridDim.y, rank = blockIdx.y;
    const int64_t i0 = (int64_t)blockIdx.x * BM, j0 = (int64_t)blockIdx.z * BN;
    int64_t kchunk = (g.k + S - 1) / S;
    kchunk = (kchunk + BK - 1) / BK * BK;
    const int64_t kbeg = (int64_t)rank * kchunk;
    const int64_t kend = min(g.k, kbeg + kchunk);
    const int ntiles = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;

    double acc[2][BN / 8][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < BN / 8; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    // prologue
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < ntiles) {
            load_a<BN>(sm, s, g.a, g.a_rs, g.a_cs, g.m, i0, kbeg + (int64_t)s * BK, kend);
            load_b<BN>(sm, s, g.b, g.b_rs, g.b_cs, g.n, j0, kbeg + (int64_t)s * BK, kend);
        }
        cp_async_commit();
    }
    for (int t = 0; t < ntiles; ++t) {
        const int nxt = t + STAGES - 1;
        if (nxt < ntiles) {
            load_a<BN>(sm, nxt % STAGES, g.a, g.a_rs, g.a_cs, g.m, i0, kbeg + (int64_t)nxt * BK, kend);
            load_b<BN>(sm, nxt % STAGES, g.b, g.b_rs, g.b_cs, g.n, j0, kbeg + (int64_t)nxt * BK, kend);
        }
        cp_async_commit();
        cp_async_wait<STAGES - 1>();
        __syncthreads();
        mma_stage<BN>(sm, t % STAGES, acc);
        __syncthreads();
    }
    cp_async_wait<0>();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gq = lane >> 2, tq = lane & 3;
    if (S == 1) {
#pragma unroll
        for (int mf = 0; mf < 2; ++mf)
#pragma unroll
            for (int nf = 0; nf < BN / 8; ++nf)
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    epilogue_store(g, i0 + warp * 16 + mf * 8 + gq, j0 + nf * 8 + tq * 2 + h, acc[mf][nf][h]);
        return;
    }
    // cluster split-K: stage the partial tile in smem, reduce over ranks in rank order
    __syncthreads();
    double* part = reinterpret_cast<double*>(smem_raw);  // BM x (BN+1)
    constexpr int PP = BN + 1;
#pragma unroll
    for (int mf = 0; mf < 2; ++mf)
#pragma unroll
        for (int nf = 0; nf < BN / 8; ++nf)
#pragma unroll
            for (int h = 0; h < 2; ++h)
                part[(warp * 16 + mf * 8 + gq) * PP + nf * 8 + tq * 2 + h] = acc[mf][nf][h];
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();
    const int rows_per = BM / S;
    for (int e = threadIdx.x; e < rows_per * BN; e += NT) {
        const int ii = rank * rows_per + e / BN, jj = e % BN;
        double s = 0.0;
        for (int src = 0; src < S; ++src) {
            const double* rp = cluster.map_shared_rank(part, src);
            s += rp[ii * PP + jj];
        }
        epilogue_store(g, i0 + ii, j0 + jj, s);
    }
    cluster.sync();
}

template <int BN>
void launch_gemm(const GemmArgs& g, int num_sms, cudaStream_t s) {
    const int mt = (int)((g.m + BM - 1) / BM);
    const int nt = (int)((g.n + BN - 1) / BN);
    int S = 1;
    // largest split (power of two <= 8) that still fits one wave of co-resident CTAs
    while (S < 8 && (int64_t)mt * nt * (2 * S) <= 2 * num_sms && g.k / (2 * S) >= 2 * BK) S *= 2;
    const size_t smem = sizeof(GemmSmem<BN>);
    func_attr_once((const void*)gemm_dmma_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    func_attr_once((const void*)gemm_dmma_kernel<BN>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(mt, S, nt);
    cfg.blockDim = dim3(NT, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = S;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CPHIFI_CUDA(cudaLaunchKernelEx(&cfg, gemm_dmma_kernel<BN>, g));
}

// ---- MTTKRP (k = 0): A = T slab (n0 x Mloc, column-major), B = Z rows generated -------
// The K dimension (unfolding columns c = i1 + n1 * outer, mode 1 fastest, tensor.hpp:70-73) is
// walked in tiles that never straddle an `outer` index (i2, ..., i_{d-1}): a tile is BK
// consecutive i1 of one outer, so its Khatri-Rao rows are A_1(i1, :) * Wout(outer, :) with
// Wout(o, :) = A_{d-1}(i_{d-1}, :) * ... * A_2(i2, :) precomputed once (the reference's
// khatri_rao multiplies left to right in descending mode order, matrix_ops.hpp:24-42; A_1 is
// the last factor, so the association — and every rounding — is the same).
__global__ void kr_outer_kernel(const MttkrpArgs a, int64_t n_outer, double* __restrict__ wout) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n_outer * a.r) return;
    const int64_t o = e / a.r, j = e % a.r;
    double* dst = wout + o * a.ldw + j;
    if (a.d == 2) {
        *dst = 1.0;
        return;
    }
    int64_t sub[8];
    int64_t rem = o;
    for (int m = 2; m < a.d; ++m) {
        sub[m] = rem % a.shape[m];
        rem /= a.shape[m];
    }
    double w = a.fac[a.d - 1][sub[a.d - 1] + a.ld[a.d - 1] * j];
    for (int m = a.d - 2; m >= 2; --m) w *= a.fac[m][sub[m] + a.ld[m] * j];
    *dst = w;
}

template <int BN>
__device__ __forceinline__ void load_tile_mttkrp(GemmSmem<BN, BMM, STM>& sm, double* ws, int st, const MttkrpArgs& a,
                                                 int64_t chunks, const double* __restrict__ wout, int64_t i0, int64_t j0,
                                                 int64_t tile) {
    const int64_t n0 = a.shape[0], n1 = a.shape[1];
    const int64_t outer = tile / chunks, c1 = (tile - outer * chunks) * BK;
    const int cnt = (int)min((int64_t)BK, n1 - c1);
    const double* tcol = a.t + (c1 + n1 * outer) * n0;  // first T column of the tile
    if ((n0 & 1) == 0) {  // 16-byte copies: column segments are 16-byte aligned
        for (int e = threadIdx.x; e < (BMM / 2) * BK; e += NTM) {
            const int ii = 2 * (e % (BMM / 2)), kk = e / (BMM / 2);
            const int64_t i = i0 + ii;
            const bool p = (i < n0) && (kk < cnt);
            const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(&sm.a[st][kk][ii]));
            const double* src = p ? tcol + i + (int64_t)kk * n0 : a.t;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(p ? 16 : 0));
        }
    } else {
        for (int e = threadIdx.x; e < BMM * BK; e += NTM) {
            const int ii = e % BMM, kk = e / BMM;
            const int64_t i = i0 + ii;
            const bool p = (i < n0) && (kk < cnt);
            cp_async8(&sm.a[st][kk][ii], p ? tcol + i + (int64_t)kk * n0 : a.t, p);
        }
    }
    // B tile staged RAW (A_1 block and the Wout row, both cp.async); the product
    // z = A_1(i1, j) * Wout(outer, j) is formed when the DMMA fragment is loaded
    const double* a1 = a.fac[1] + c1 + a.off1;
    for (int e = threadIdx.x; e < BN * BK; e += NTM) {
        const int kk = e % BK, jj = e / BK;  // consecutive threads: consecutive i1 (coalesced)
        const int64_t j = j0 + jj;
        const bool p = (j < a.r) && (kk < cnt);
        cp_async8(&sm.b[st][kk][jj], p ? a1 + kk + a.ld[1] * j : a.fac[1], p);
    }
    if (threadIdx.x < BN) {
        const int64_t j = j0 + threadIdx.x;
        cp_async8(ws + st * BN + threadIdx.x, j < a.r ? wout + outer * a.ldw + j : wout, j < a.r);
    }
}

template <int BN>
__device__ __forceinline__ void mma_stage_scaled(const GemmSmem<BN, BMM, STM>& sm, const double* ws, int st,
                                                 double (&acc)[2][BN / 8][2]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int kq = lane & 3, g = lane >> 2;
    double w[BN / 8];
#pragma unroll
    for (int nf = 0; nf < BN / 8; ++nf) w[nf] = ws[st * BN + nf * 8 + g];
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
        const int kr = ks * 4 + kq;
        const double a0 = sm.a[st][kr][warp * 16 + g];
        const double a1 = sm.a[st][kr][warp * 16 + 8 + g];
#pragma unroll
        for (int nf = 0; nf < BN / 8; ++nf) {
            const double bv = sm.b[st][kr][nf * 8 + g] * w[nf];
            dmma(acc[0][nf], a0, bv);
            dmma(acc[1][nf], a1, bv);
        }
    }
}

template <int BN>
__global__ void __launch_bounds__(NTM) mttkrp_dmma_kernel(const MttkrpArgs a, int64_t chunks, int64_t ktiles,
                                                         const double* __restrict__ wout, double* __restrict__ work) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    GemmSmem<BN, BMM, STM>& sm = *reinterpret_cast<GemmSmem<BN, BMM, STM>*>(smem_raw);
    double* ws = reinterpret_cast<double*>(smem_raw + sizeof(GemmSmem<BN, BMM, STM>));  // STM x BN
    const int P = gridDim.y, split = blockIdx.y;
    const int64_t n0 = a.shape[0];
    const int64_t i0 = (int64_t)blockIdx.x * BMM, j0 = (int64_t)blockIdx.z * BN;
    const int64_t tb = ktiles * split / P, te = ktiles * (split + 1) / P;
    const int ntiles = (int)(te - tb);

    double acc[2][BN / 8][2];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < BN / 8; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;

#pragma unroll
    for (int s = 0; s < STM - 1; ++s) {
        if (s < ntiles) load_tile_mttkrp<BN>(sm, ws, s, a, chunks, wout, i0, j0, tb + s);
        cp_async_commit();
    }
    for (int t = 0; t < ntiles; ++t) {
        const int nxt = t + STM - 1;
        if (nxt < ntiles) load_tile_mttkrp<BN>(sm, ws, nxt % STM, a, chunks, wout, i0, j0, tb + nxt);
        cp_async_commit();
        cp_async_wait<STM - 1>();
        __syncthreads();
        mma_stage_scaled<BN>(sm, ws, t % STM, acc);
        __syncthreads();
    }
    cp_async_wait<0>();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gq = lane >> 2, tq = lane & 3;
    double* out = work + (int64_t)split * n0 * a.r;
#pragma unroll
    for (int mf = 0; mf < 2; ++mf)
#pragma unroll
        for (int nf = 0; nf < BN / 8; ++nf)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t i = i0 + warp * 16 + mf * 8 + gq, j = j0 + nf * 8 + tq * 2 + h;
                if (i < n0 && j < a.r) out[i + n0 * j] = acc[mf][nf][h];
            }
}

// MTTKRP v2 (BN <= 32): 16 warps = 4 row groups (32 rows x BN each, 4 x BN/8 independent DMMA
// accumulators per k-step) x 4 k-groups (each takes 2 of the 8 k-steps of a stage; their
// partials are summed in k-group order at the end).  The B tile is scaled by Wout once per stage
// in shared memory (one DMUL per element instead of one per warp and fragment), so the DMMA
// chain has no FP64 dependency in front of it.  ncu on the v1 kernel (8 warps, per-warp B
// scaling): DMMA pipe 46 % active, stalls dominated by fixed-latency waits with 2 warps per
// scheduler.
constexpr int NTV = 512;
constexpr int KGV = 4;  // k-groups
template <int BN>
__global__ void __launch_bounds__(NTV, 1) mttkrp_v2_kernel(const MttkrpArgs a, int64_t chunks, int64_t ktiles,
                                                           const double* __restrict__ wout, double* __restrict__ work) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    GemmSmem<BN, BMM, STM>& sm = *reinterpret_cast<GemmSmem<BN, BMM, STM>*>(smem_raw);
    double* ws = reinterpret_cast<double*>(smem_raw + sizeof(GemmSmem<BN, BMM, STM>));  // STM x BN
    constexpr int NF = BN / 8;
    const int P = gridDim.y, split = blockIdx.y;
    const int64_t n0 = a.shape[0];
    const int64_t i0 = (int64_t)blockIdx.x * BMM, j0 = (int64_t)blockIdx.z * BN;
    const int64_t tb = ktiles * split / P, te = ktiles * (split + 1) / P;
    const int ntiles = (int)(te - tb);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int rg = warp & 3, kg = warp >> 2;
    const int kq = lane & 3, g = lane >> 2;

    double acc[4][NF][2];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < NF; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;

    auto load = [&](int st, int64_t tile) {  // the v1 tile loader, 512 threads
        const int64_t n1 = a.shape[1];
        const int64_t outer = tile / chunks, c1 = (tile - outer * chunks) * BK;
        const int cnt = (int)min((int64_t)BK, n1 - c1);
        const double* tcol = a.t + (c1 + n1 * outer) * n0;
        if ((n0 & 1) == 0) {
            for (int e = threadIdx.x; e < (BMM / 2) * BK; e += NTV) {
                const int ii = 2 * (e % (BMM / 2)), kk = e / (BMM / 2);
                const int64_t i = i0 + ii;
                const bool p = (i < n0) && (kk < cnt);
                const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(&sm.a[st][kk][ii]));
                const double* src = p ? tcol + i + (int64_t)kk * n0 : a.t;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(p ? 16 : 0));
            }
        } else {
            for (int e = threadIdx.x; e < BMM * BK; e += NTV) {
                const int ii = e % BMM, kk = e / BMM;
                const int64_t i = i0 + ii;
                const bool p = (i < n0) && (kk < cnt);
                cp_async8(&sm.a[st][kk][ii], p ? tcol + i + (int64_t)kk * n0 : a.t, p);
            }
        }
        const double* a1 = a.fac[1] + c1 + a.off1;
        for (int e = threadIdx.x; e < BN * BK; e += NTV) {
            const int kk = e % BK, jj = e / BK;
            const int64_t j = j0 + jj;
            const bool p = (j < a.r) && (kk < cnt);
            cp_async8(&sm.b[st][kk][jj], p ? a1 + kk + a.ld[1] * j : a.fac[1], p);
        }
        if (threadIdx.x < BN) {
            const int64_t j = j0 + threadIdx.x;
            cp_async8(ws + st * BN + threadIdx.x, j < a.r ? wout + outer * a.ldw + j : wout, j < a.r);
        }
    };

#pragma unroll
    for (int s = 0; s < STM - 1; ++s) {
        if (s < ntiles) load(s, tb + s);
        cp_async_commit();
    }
    for (int t = 0; t < ntiles; ++t) {
        const int st = t % STM;
        cp_async_wait<STM - 2>();  // stage t landed (this thread's copies)
        __syncthreads();           // ... everyone's; and every warp is done with stage t - 1
        if (t + STM - 1 < ntiles) load((t + STM - 1) % STM, tb + t + STM - 1);
        cp_async_commit();
        // z = A_1(i1, j) * Wout(outer, j): scale the B tile once, in place
        for (int e = threadIdx.x; e < BN * BK; e += NTV) {
            const int kk = e / BN, jj = e % BN;
            sm.b[st][kk][jj] *= ws[st * BN + jj];
        }
        __syncthreads();
#pragma unroll
        for (int k2 = 0; k2 < BK / 4 / KGV; ++k2) {
            const int kr = (kg * (BK / 4 / KGV) + k2) * 4 + kq;
            double af[4], bf[NF];
#pragma unroll
            for (int mf = 0; mf < 4; ++mf) af[mf] = sm.a[st][kr][rg * 32 + mf * 8 + g];
#pragma unroll
            for (int nf = 0; nf < NF; ++nf) bf[nf] = sm.b[st][kr][nf * 8 + g];
#pragma unroll
            for (int mf = 0; mf < 4; ++mf)
#pragma unroll
                for (int nf = 0; nf < NF; ++nf) dmma(acc[mf][nf], af[mf], bf[nf]);
        }
    }
    cp_async_wait<0>();
    __syncthreads();
    // k-group partials -> shared memory, summed in k-group order
    double* red = reinterpret_cast<double*>(smem_raw);  // KGV x BMM x BN
#pragma unroll
    for (int mf = 0; mf < 4; ++mf)
#pragma unroll
        for (int nf = 0; nf < NF; ++nf)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int ii = rg * 32 + mf * 8 + g, jj = nf * 8 + kq * 2 + h;
                red[(kg * BMM + ii) * BN + jj] = acc[mf][nf][h];
            }
    __syncthreads();
    double* out = work + (int64_t)split * n0 * a.r;
    for (int e = threadIdx.x; e < BMM * BN; e += NTV) {
        const int ii = e % BMM, jj = e / BMM;
        const int64_t i = i0 + ii, j = j0 + jj;
        if (i < n0 && j < a.r) {
            double s = red[ii * BN + jj];
#pragma unroll
            for (int k = 1; k < KGV; ++k) s += red[(k * BMM + ii) * BN + jj];
            out[i + n0 * j] = s;
        }
    }
}

// MTTKRP v3 (BN <= 32, tensor-map TMA): a warp-specialised 5-stage ring.  Warp 8 is the
// producer: per tile ONE 2-D tensor copy brings the T box (132 rows x 32 unfolding columns; the 4
// extra rows land in the conflict-free pitch padding, rows past n0 read as zero), ONE brings the
// A_1 box (36 i1 x BN columns, transposed layout k fastest, j past r read as zero) and one bulk
// copy the Wout row, all completing on the slot's `full` mbarrier.  (Per-column bulk copies — 65
// instructions per stage — capped the stream at ~2 TB/s: the copy engine's per-instruction
// cost, not DRAM, was the limit.)  Warps 0-7 consume (4 row groups of 32 rows x 2 k-groups; one
// warp per scheduler already saturates DMMA, profiles/micro/dmma_issue.cu) and release the slot
// on its `empty` mbarrier: no CTA-wide barrier inside the loop.  Each split takes a contiguous
// tile range; tiles of one `outer` index share the Wout row, so the DMMAs accumulate the raw
// T_tile x A_1 tile products into a per-outer accumulator that is scaled by Wout (per output
// column) and folded into the result when `outer` changes: no FP64 work besides DMMA in the loop
// (per-fragment scaling + masking cost 8 % of the DMMA throughput).  Partial k chunks (n1 not a
// multiple of 32) take a masked path.
constexpr int ST3 = 5;
// 8 consumer warps tile the 128 x BN CTA tile with WR x WC warp tiles; the rest of the 8 go to
// k-groups that split each stage's k-steps (their partials are summed in order at the end).
// 32 x 16 tiles (KG = 1) keep the per-outer accumulators at 2 x 16 doubles per lane, so the
// compiler can hold the next k-step's fragments in registers (the 32 x 32 / KG = 2 layout at 168
// registers reloaded fragments right before each DMMA: LDS latency exposed, 75 % of DMMA peak).
template <int BN, int WR, int WC>
struct V3 {
    static constexpr int RG = BMM / WR;                 // row groups
    static constexpr int CG = BN / WC;                  // column groups
    static constexpr int KG = 8 / (RG * CG);            // k-groups (8 consumer warps)
    static constexpr int NC = RG * CG * KG * 32;        // consumer threads
    static constexpr int MF = WR / 8, NF = WC / 8;      // fragments per k-step
    static_assert(RG * CG * KG == 8 && KG >= 1, "8 consumer warps");
};
constexpr int AP3 = BMM + 4;          // T box rows = smem pitch
constexpr int BKP3 = BK + 4;          // A_1 box rows = smem pitch of the transposed B tile
// B tile: [j][k] (pitch BKP3) from a column-major B (the MTTKRP's A_1, a GEMM's X), or [k][j]
// (pitch BN + 4, the 4 extra columns read past the tile or as zero) from a row-major B (BROW)
// A tile: AM = 0 [k][i] (pitch AP3) from a column-major A (the MTTKRP's unfolding for mode 0, a
// GEMM's A); AM = 1 / 2 [i][k] (pitch BK + 4) — the transposed unfoldings of the middle / last
// mode of a 3-way column-major tensor, through a 3-D / 2-D tensor map — with one stage fewer.
template <int BN, int AM = 0>
struct Mttkrp3Smem {
    static constexpr int NST = AM == 0 ? ST3 : ST3 - 1;
    static constexpr int ASZ = AM == 0 ? BK * AP3 : BMM * (BK + 4);
    static constexpr int BSZ = BN * BKP3 > BK * (BN + 4) ? BN * BKP3 : BK * (BN + 4);
    double a[NST][ASZ];
    double bt[NST][BSZ];
    double w[NST][BN];  // the tile's Wout row (its `outer` index)
    uint64_t full[NST], empty[NST];
};
template <int BN, int WR, int WC, bool BROW, int AM = 0>
__global__ void __launch_bounds__(V3<BN, WR, WC>::NC + 32, 1) mttkrp_v3_kernel(const MttkrpArgs a, const __grid_constant__ CUtensorMap tm_t,
                                                                const __grid_constant__ CUtensorMap tm_a1, int64_t chunks,
                                                                int64_t ktiles, const double* __restrict__ wout,
                                                                double* __restrict__ work) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    using SMT = Mttkrp3Smem<BN, AM>;
    constexpr int ST3 = SMT::NST;
    SMT& sm = *reinterpret_cast<SMT*>(smem_raw);
    auto aidx = [](int k, int i) { return AM == 0 ? k * AP3 + i : i * (BK + 4) + k; };
    using L = V3<BN, WR, WC>;
    constexpr int NC3 = L::NC, MF = L::MF, NF = L::NF, RG = L::RG, CG = L::CG, KG = L::KG;
    const int P = gridDim.y, split = blockIdx.y;
    const int64_t n0 = a.shape[0], n1 = a.shape[1];
    const int64_t i0 = (int64_t)blockIdx.x * BMM, j0 = (int64_t)blockIdx.z * BN;
    const int64_t tb = ktiles * split / P, te = ktiles * (split + 1) / P;
    const int ntiles = (int)(te - tb);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int rows = (int)min((int64_t)BMM, n0 - i0);
    auto bidx = [](int k, int j) { return BROW ? k * (BN + 4) + j : j * BKP3 + k; };
    const int bcols = (int)min((int64_t)BN, a.r - j0);

    if (threadIdx.x == 0) {
        for (int s = 0; s < ST3; ++s) {
            tma::mbar_init(&sm.full[s], 1);
            tma::mbar_init(&sm.empty[s], NC3 / 32);
        }
        tma::fence_mbar_init();
    }
    __syncthreads();

    // tile (outer, chunk) of this split's t-th step, advanced without 64-bit division
    struct TileIt {
        int64_t outer, cidx;
    };
    auto tile_first = [&]() { return TileIt{tb / chunks, tb % chunks}; };
    auto tile_next = [&](TileIt& it) {
        if (++it.cidx == chunks) {
            it.cidx = 0;
            ++it.outer;
        }
    };

    if (warp == NC3 / 32) {  // ---- producer warp (one lane) ----
        if (lane == 0) {
            const unsigned wb = (unsigned)((bcols * 8 + 15) & ~15);  // Wout row (2 spare doubles past the end)
            const unsigned bytes = (unsigned)(sizeof(double) * (SMT::ASZ + (BROW ? BK * (BN + 4) : BN * BKP3))) + wb;
            // L2 prefetch runs l2_ahead tiles in front of the ring: the shared-memory stages then
            // fill from L2, and the loaded-HBM latency hides behind the prefetch distance
            const int pf = a.l2_ahead;
            TileIt it = tile_first(), itp = tile_first();
            for (int t = 0; t < min(pf, ntiles); ++t) {
                tma::tensor_prefetch_l2_2d(&tm_t, (int)i0, (int)(itp.cidx * BK + n1 * itp.outer));
                tile_next(itp);
            }
            for (int t = 0; t < ntiles; ++t, tile_next(it)) {
                const int st = t % ST3;
                if (pf > 0 && t + pf < ntiles) {
                    tma::tensor_prefetch_l2_2d(&tm_t, (int)i0, (int)(itp.cidx * BK + n1 * itp.outer));
                    tile_next(itp);
                }
                if (t >= ST3) tma::mbar_wait(&sm.empty[st], (unsigned)(((t / ST3) - 1) & 1));
                const int64_t outer = it.outer, c1 = it.cidx * BK;
                if (a.probe >= 2 && t >= ST3) {  // profiling: compute only (stale stages)
                    tma::mbar_arrive(&sm.full[st]);
                    continue;
                }
                tma::mbar_expect_tx(&sm.full[st], bytes);
                if constexpr (AM == 0) tma::tensor_g2s_2d(&sm.a[st][0], &tm_t, (int)i0, (int)(c1 + n1 * outer), &sm.full[st]);
                else if constexpr (AM == 2) tma::tensor_g2s_2d(&sm.a[st][0], &tm_t, (int)(c1 + n1 * outer), (int)i0, &sm.full[st]);
                else tma::tensor_g2s_3d(&sm.a[st][0], &tm_t, (int)c1, (int)i0, (int)outer, &sm.full[st]);
                if constexpr (BROW) tma::tensor_g2s_2d(&sm.bt[st][0], &tm_a1, (int)j0, (int)(c1 + a.off1), &sm.full[st]);
                else tma::tensor_g2s_2d(&sm.bt[st][0], &tm_a1, (int)(c1 + a.off1), (int)j0, &sm.full[st]);
                tma::bulk_g2s(&sm.w[st][0], wout + outer * a.ldw + j0, wb, &sm.full[st]);
            }
        }
    } else {  // ---- consumer warps ----
        const int rg = warp % RG, cg = (warp / RG) % CG, kg = warp / (RG * CG);
        const int kq = lane & 3, g = lane >> 2;
        double acc[MF][NF][2], tmp[MF][NF][2];
#pragma unroll
        for (int x = 0; x < MF; ++x)
#pragma unroll
            for (int y = 0; y < NF; ++y) acc[x][y][0] = acc[x][y][1] = tmp[x][y][0] = tmp[x][y][1] = 0.0;
        // acc += tmp * Wout(outer, column) for the lane's C columns nf * 8 + 2 kq + h (a one-outer
        // look-ahead of the Wout loads spilled registers and measured slower)
        // acc += tmp * Wout(outer, column) for the lane's C columns nf * 8 + 2 kq + h, done after
        // the LAST tile of an outer (its slot still holds that outer's Wout row in shared memory)
        auto fold = [&](int st) {
#pragma unroll
            for (int nf = 0; nf < NF; ++nf)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int jj = cg * WC + nf * 8 + 2 * kq + h;
                    const double wv = jj < bcols ? sm.w[st][jj] : 0.0;
#pragma unroll
                    for (int mf = 0; mf < MF; ++mf) {
                        acc[mf][nf][h] = fma(tmp[mf][nf][h], wv, acc[mf][nf][h]);
                        tmp[mf][nf][h] = 0.0;
                    }
                }
        };
        TileIt it = tile_first();
        for (int t = 0; t < ntiles; ++t) {
            const int st = t % ST3;
            const int cnt = (int)min((int64_t)BK, n1 - it.cidx * BK);
            const int64_t outer = it.outer;
            tile_next(it);
            const bool last_of_outer = t + 1 == ntiles || it.outer != outer;
            tma::mbar_wait(&sm.full[st], (unsigned)((t / ST3) & 1));
            if (a.probe != 1) {
                if (cnt == BK) {  // full chunk: DMMA only
#pragma unroll
                    for (int k2 = 0; k2 < BK / 4 / KG; ++k2) {
                        const int kr = (kg * (BK / 4 / KG) + k2) * 4 + kq;
                        double af[MF], bf[NF];
#pragma unroll
                        for (int mf = 0; mf < MF; ++mf) af[mf] = sm.a[st][aidx(kr, rg * WR + mf * 8 + g)];
#pragma unroll
                        for (int nf = 0; nf < NF; ++nf) bf[nf] = sm.bt[st][bidx(kr, cg * WC + nf * 8 + g)];
#pragma unroll
                        for (int mf = 0; mf < MF; ++mf)
#pragma unroll
                            for (int nf = 0; nf < NF; ++nf) dmma(tmp[mf][nf], af[mf], bf[nf]);
                    }
                } else {  // partial chunk: k past the extent masked to zero in B
#pragma unroll
                    for (int k2 = 0; k2 < BK / 4 / KG; ++k2) {
                        const int kr = (kg * (BK / 4 / KG) + k2) * 4 + kq;
                        double af[MF], bf[NF];
#pragma unroll
                        for (int mf = 0; mf < MF; ++mf) af[mf] = sm.a[st][aidx(kr, rg * WR + mf * 8 + g)];
#pragma unroll
                        for (int nf = 0; nf < NF; ++nf) bf[nf] = kr < cnt ? sm.bt[st][bidx(kr, cg * WC + nf * 8 + g)] : 0.0;
#pragma unroll
                        for (int mf = 0; mf < MF; ++mf)
#pragma unroll
                            for (int nf = 0; nf < NF; ++nf) dmma(tmp[mf][nf], af[mf], bf[nf]);
                    }
                }
                if (last_of_outer) fold(st);
            }
            __syncwarp();
            if (lane == 0) tma::mbar_arrive(&sm.empty[st]);
        }
        __syncthreads();  // (1) the ring is drained by every consumer
        double* red = reinterpret_cast<double*>(smem_raw);  // KG x BMM x BN
#pragma unroll
        for (int mf = 0; mf < MF; ++mf)
#pragma unroll
            for (int nf = 0; nf < NF; ++nf)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int ii = rg * WR + mf * 8 + g, jj = cg * WC + nf * 8 + kq * 2 + h;
                    red[(kg * BMM + ii) * BN + jj] = acc[mf][nf][h];
                }
    }
    if (warp == NC3 / 32) __syncthreads();  // the producer's side of (1)
    __syncthreads();
    const double* red = reinterpret_cast<const double*>(smem_raw);
    double* out = work + (int64_t)split * n0 * a.r;
    for (int e = threadIdx.x; e < BMM * BN; e += blockDim.x) {
        const int ii = e % BMM, jj = e / BMM;
        const int64_t i = i0 + ii, j = j0 + jj;
        if (ii < rows && j < a.r) {
            double s = red[ii * BN + jj];
#pragma unroll
            for (int k = 1; k < KG; ++k) s += red[(k * BMM + ii) * BN + jj];
            out[i + n0 * j] = s;
        }
    }
}

// sum_p work[p * stride + e] in p order, the loads of 8 splits in flight at a time (a plain loop
// left one L2 round trip per split exposed: config 2's 18-split reduce took 7.6 us)
__device__ __forceinline__ double sum_splits(const double* __restrict__ work, int P, int64_t stride, int64_t e) {
    double s = 0.0;
    int p = 0;
    for (; p + 8 <= P; p += 8) {
        double v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = __ldcg(work + (int64_t)(p + j) * stride + e);
#pragma unroll
        for (int j = 0; j < 8; ++j) s += v[j];
    }
    for (; p < P; ++p) s += __ldcg(work + (int64_t)p * stride + e);
    return s;
}

__global__ void reduce_splits_kernel(const double* __restrict__ work, int P, int64_t cnt,
                                     double* __restrict__ out) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < cnt; e += (int64_t)gridDim.x * blockDim.x)
        out[e] = sum_splits(work, P, cnt, e);
}

template <int BN, int WR, int WC, bool BROW = false, int AM = 0>
void launch_v3(const MttkrpArgs& ap, const CUtensorMap& tm_t, const CUtensorMap& tm_a1, int mt, int64_t P, int nt,
               int64_t chunks, int64_t ktiles, const double* wout, double* work, cudaStream_t s) {
    const size_t smem3 = sizeof(Mttkrp3Smem<BN, AM>);
    func_attr_once((const void*)mttkrp_v3_kernel<BN, WR, WC, BROW, AM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3);
    mttkrp_v3_kernel<BN, WR, WC, BROW, AM><<<dim3(mt, (unsigned)P, nt), V3<BN, WR, WC>::NC + 32, smem3, s>>>(ap, tm_t, tm_a1, chunks,
                                                                                           ktiles, wout, work);
    const cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess) {
        cudaFuncAttributes fa;
        cudaFuncGetAttributes(&fa, mttkrp_v3_kernel<BN, WR, WC, BROW, AM>);
        throw Error(CPHIFI_CUDA_ERROR, std::string("mttkrp_v3 launch: ") + cudaGetErrorString(le) + " regs " +
                                           std::to_string(fa.numRegs) + " maxthreads " + std::to_string(fa.maxThreadsPerBlock));
    }
}

template <int BN>
void launch_mttkrp(const MttkrpArgs& a, int num_sms, cudaStream_t s, DevBuf<double>& work) {
    const int64_t n0 = a.shape[0];
    int64_t n_outer = 1;
    for (int m = 2; m < a.d; ++m) n_outer *= a.shape[m];
    const int64_t chunks = (a.shape[1] + BK - 1) / BK;
    const int64_t ktiles = n_outer * chunks;
    const int mt = (int)((n0 + BMM - 1) / BMM);
    const int nt = (int)((a.r + BN - 1) / BN);
    // exactly one wave (one CTA per SM): a partial second wave would double the duration
    int64_t P = std::max<int64_t>(1, (int64_t)num_sms / (mt * nt));
    P = std::max<int64_t>(1, std::min<int64_t>(P, ktiles));
    P = std::min<int64_t>(P, 1024);
    MttkrpArgs aw = a;
    aw.ldw = (a.r + 1) & ~1LL;  // 16-byte Wout rows (the v3 producer bulk-copies them)
    const size_t need = (size_t)P * n0 * a.r + (size_t)n_outer * aw.ldw + 2;
    if (work.n < need) work.alloc(need);
    double* wout = work.get() + (size_t)P * n0 * a.r;
    kr_outer_kernel<<<(unsigned)((n_outer * a.r + 255) / 256), 256, 0, s>>>(aw, n_outer, wout);
    CPHIFI_CHECK_LAUNCH();
    const size_t smem = sizeof(GemmSmem<BN, BMM, STM>) + sizeof(double) * STM * BN;
    func_attr_once((const void*)mttkrp_dmma_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    bool v2 = BN <= 32;
    if (const char* e = std::getenv("CPHIFI_MTTKRP_V1")) v2 = v2 && std::atoi(e) == 0;
    // v3 (tensor-map TMA ring) needs 16-byte aligned bases and leading dimensions (even n0 and
    // A_1 leading dimension) and int32 box coordinates
    int64_t ncols = 1;
    for (int m = 1; m < a.d; ++m) ncols *= a.shape[m];
    CUtensorMap tm_t, tm_a1;
    bool v3 = v2 && (n0 % 2 == 0) && (a.ld[1] % 2 == 0) && ncols < (1LL << 31) &&
              encode_tmap_2d_f64(&tm_t, a.t, (uint64_t)n0, (uint64_t)ncols, (uint64_t)n0, BMM + 4, BK) &&
              encode_tmap_2d_f64(&tm_a1, a.fac[1], (uint64_t)a.ld[1], (uint64_t)a.r, (uint64_t)a.ld[1], BK + 4, BN);
    if (const char* e = std::getenv("CPHIFI_MTTKRP_V3")) v3 = v3 && std::atoi(e) != 0;
    MttkrpArgs ap = aw;
    if (const char* e = std::getenv("CPHIFI_MTTKRP_PROBE")) ap.probe = std::atoi(e);
    if (const char* e = std::getenv("CPHIFI_MTTKRP_L2AHEAD")) ap.l2_ahead = std::atoi(e);
    if constexpr (BN <= 32) {
        static_assert(sizeof(double) * KGV * BMM * BN <= sizeof(GemmSmem<BN, BMM, STM>), "reduction fits");
        if (v3) {
            int wc = BN >= 16 ? 16 : BN;  // warp tile 32 x 16 (KG = 1 at BN = 32); CPHIFI_MTTKRP_WC=32 -> 32 x 32, KG = 2
            if (const char* e = std::getenv("CPHIFI_MTTKRP_WC")) wc = std::atoi(e);
            if constexpr (BN == 32) {
                if (wc == 32) launch_v3<BN, 32, 32, false>(ap, tm_t, tm_a1, mt, P, nt, chunks, ktiles, wout, work.get(), s);
                else launch_v3<BN, 32, 16, false>(ap, tm_t, tm_a1, mt, P, nt, chunks, ktiles, wout, work.get(), s);
            } else {
                launch_v3<BN, 32, BN, false>(ap, tm_t, tm_a1, mt, P, nt, chunks, ktiles, wout, work.get(), s);
            }
        } else if (v2) {
            func_attr_once((const void*)mttkrp_v2_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            mttkrp_v2_kernel<BN><<<dim3(mt, (unsigned)P, nt), NTV, smem, s>>>(aw, chunks, ktiles, wout, work.get());
        }
    }
    if (!v2)
        mttkrp_dmma_kernel<BN><<<dim3(mt, (unsigned)P, nt), NTM, smem, s>>>(aw, chunks, ktiles, wout, work.get());
    CPHIFI_CHECK_LAUNCH();
    const int64_t cnt = n0 * a.r;
    reduce_splits_kernel<<<(unsigned)std::min<int64_t>((cnt + 255) / 256, 4 * num_sms), 256, 0, s>>>(
        work.get(), (int)P, cnt, a.b);
    CPHIFI_CHECK_LAUNCH();
}

// ---- small kernels -------------------------------------------------------------------
// V(row, col) = prod_{m != k} (A_m' A_m)(row, col): one warp per entry, lanes stride the rows
// of A_m (coalesced), fixed xor-shuffle tree; V is exactly symmetric (same products, same order).
struct GramKrArgs {
    int d = 0, k = 0;
    int64_t r = 0;
    const double* fac[8] = {nullptr};
    int64_t shape[8] = {0};
};
__global__ void gram_kernel(const GramKrArgs g, double* v) {
    const int64_t e = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (e >= g.r * g.r) return;
    const int64_t row = e % g.r, col = e / g.r;
    double acc = 1.0;
    for (int m = 0; m < g.d; ++m) {
        if (m == g.k) continue;
        const double* a = g.fac[m];
        const int64_t nm = g.shape[m];
        double s = 0.0;
        for (int64_t i = lane; i < nm; i += 32) s = fma(a[i + nm * row], a[i + nm * col], s);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        acc *= s;
    }
    if (lane == 0) v[e] = acc;
}

__global__ void kernel_matrix_kernel(int kind, const double* __restrict__ pts, int64_t n, double p,
                                     double* __restrict__ kmat) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n * n) return;
    const int64_t i = e % n, j = e / n;
    double v;
    if (i == j) {
        v = 1.0;
    } else {
        // evaluate on the (max, min) ordered pair exactly as kernel.hpp:29-33 does for j < i
        const int64_t a = i > j ? i : j, b = i > j ? j : i;
        if (kind == 0) {
            const double dd = pts[a] - pts[b];
            v = exp(-dd * dd * p);  // p = 1 / (2 sigma^2)
        } else {
            const double t = p * fabs(pts[a] - pts[b]);  // p = sqrt(3) / ell
            v = (1.0 + t) * exp(-t);
        }
    }
    kmat[e] = v;
}

__global__ void clamp_kernel(double* v, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) v[i] = v[i] < 0.0 ? 0.0 : v[i];
}

// max |A(i,j) - A(j,i)| and max |A(i,j)| (sym_eig's symmetry check, kernel.hpp:40-49): 32 x 32 tile
// pairs (i-tile <= j-tile) through shared memory so both the tile and its transpose are read
// coalesced; the maxima of non-negative doubles are folded with 64-bit integer atomicMax on their
// bit patterns (order-independent: exact and deterministic).  (One 256-thread block took 8.5 ms
// at n = 4096.)
__global__ void max_asym_kernel(const double* __restrict__ a, int64_t n, unsigned long long* out2) {
    __shared__ double t0[32][33], t1[32][33];
    const int64_t bi = blockIdx.x, bj = blockIdx.y;
    if (bi > bj) return;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    double m1 = 0.0, m2 = 0.0;
    for (int yy = ty; yy < 32; yy += 8) {
        const int64_t r0 = bi * 32 + tx, c0 = bj * 32 + yy;  // tile (bi, bj): A(r0, c0)
        const int64_t r1 = bj * 32 + tx, c1 = bi * 32 + yy;  // tile (bj, bi)
        t0[yy][tx] = (r0 < n && c0 < n) ? a[r0 + n * c0] : 0.0;
        t1[yy][tx] = (r1 < n && c1 < n) ? a[r1 + n * c1] : 0.0;
    }
    __syncthreads();
    for (int yy = ty; yy < 32; yy += 8) {
        const double v = t0[yy][tx];  // A(bi*32 + tx, bj*32 + yy)
        m1 = fmax(m1, fabs(v - t1[tx][yy]));  // A(bj*32 + yy, bi*32 + tx)
        m2 = fmax(m2, fabs(v));
        m2 = fmax(m2, fabs(t1[yy][tx]));
    }
    for (int off = 16; off > 0; off >>= 1) {
        m1 = fmax(m1, __shfl_xor_sync(0xffffffffu, m1, off));
        m2 = fmax(m2, __shfl_xor_sync(0xffffffffu, m2, off));
    }
    if (tx == 0) {
        atomicMax(out2, (unsigned long long)__double_as_longlong(m1));
        atomicMax(out2 + 1, (unsigned long long)__double_as_longlong(m2));
    }
}

// D(i,j) = 1 / (gamma sigma_j mu_i^2 + lambda mu_i + rho)   (unaligned.hpp:125-133)
__global__ void precond_diag_kernel(const double* mu, const double* sv, int64_t n, int64_t r, double gamma,
                                    double lambda, double rho, double* dmat, int* flag) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n * r) return;
    const int64_t i = e % n, j = e / n;
    const double den = gamma * sv[j] * mu[i] * mu[i] + lambda * mu[i] + rho;
    if (den <= 0.0) *flag = 1;
    dmat[e] = 1.0 / den;
}

__global__ void pack_rows_kernel(const double* src, int64_t rows, int64_t ld, int64_t r, int64_t rp,
                                 double* dst) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= rows * rp) return;
    const int64_t i = e / rp, j = e % rp;
    dst[e] = j < r ? src[i + ld * j] : 0.0;
}

__global__ void rm_to_cm_kernel(const double* src, int64_t rows, int64_t rp, int64_t r, double* dst) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= rows * r) return;
    const int64_t i = e % rows, j = e / rows;
    dst[e] = src[i * rp + j];
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

// FP64 peak probes (the roofline denominators MEASURED_PEAKS.json lacks): 8 independent
// dependency chains per thread (DFMA) / per warp (DMMA m8n8k4 = 256 FMA per instruction).
__global__ void peak_dfma_kernel(int iters, double seed, double* out) {
    double a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = seed + u * 1e-3 + threadIdx.x * 1e-9;
    const double b = 0.999999, c = 1e-7;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] = fma(a[u], b, c);
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) s += a[u];
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

__global__ void peak_dmma_kernel(int iters, double seed, double* out) {
    double acc[8][2];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u][0] = acc[u][1] = 0.0;
    const double av = seed + threadIdx.x * 1e-9, bv = 1.0 - threadIdx.x * 1e-9;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int u = 0; u < 8; ++u) dmma(acc[u], av, bv);
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) s += acc[u][0] + acc[u][1];
    if (s == 12345.678) out[0] = s;
}

}  // namespace

bool encode_tmap_2d_f64(CUtensorMap* map, const double* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box0,
                        uint32_t box1, bool swizzle128) {
    using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Fn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<Fn>(p);
    }();
    if (!fn || reinterpret_cast<uintptr_t>(base) % 16 != 0 || (ld * sizeof(double)) % 16 != 0) return false;
    const cuuint64_t dims[2] = {rows, cols};
    const cuuint64_t strides[1] = {ld * sizeof(double)};
    const cuuint32_t box[2] = {box0, box1};
    const cuuint32_t es[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool encode_tmap_3d_f64(CUtensorMap* map, const double* base, uint64_t n0, uint64_t n1, uint64_t n2, uint32_t b0,
                        uint32_t b1, uint32_t b2) {
    using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Fn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<Fn>(p);
    }();
    if (!fn || reinterpret_cast<uintptr_t>(base) % 16 != 0 || (n0 * sizeof(double)) % 16 != 0) return false;
    const cuuint64_t dims[3] = {n0, n1, n2};
    const cuuint64_t strides[2] = {n0 * sizeof(double), n0 * n1 * sizeof(double)};
    const cuuint32_t box[3] = {b0, b1, b2};
    const cuuint32_t es[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void fp64_peaks(int num_sms, cudaStream_t s, double* dfma_tflops, double* dmma_tflops) {
    DevBuf<double> sink(1);
    cudaEvent_t e0, e1;
    CPHIFI_CUDA(cudaEventCreate(&e0));
    CPHIFI_CUDA(cudaEventCreate(&e1));
    const int blocks = num_sms * 8, threads = 256, iters = 4096;
    float ms = 0.0f;
    peak_dfma_kernel<<<blocks, threads, 0, s>>>(iters, 1.0, sink.get());  // warm-up
    CPHIFI_CUDA(cudaEventRecord(e0, s));
    peak_dfma_kernel<<<blocks, threads, 0, s>>>(iters, 1.0, sink.get());
    CPHIFI_CUDA(cudaEventRecord(e1, s));
    CPHIFI_CUDA(cudaEventSynchronize(e1));
    CPHIFI_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *dfma_tflops = 2.0 * 8.0 * iters * (double)blocks * threads / (ms * 1e-3) / 1e12;
    peak_dmma_kernel<<<blocks, threads, 0, s>>>(iters / 4, 1.0, sink.get());
    CPHIFI_CUDA(cudaEventRecord(e0, s));
    peak_dmma_kernel<<<blocks, threads, 0, s>>>(iters / 4, 1.0, sink.get());
    CPHIFI_CUDA(cudaEventRecord(e1, s));
    CPHIFI_CUDA(cudaEventSynchronize(e1));
    CPHIFI_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *dmma_tflops = 2.0 * 256.0 * 8.0 * (iters / 4) * (double)blocks * (threads / 32) / (ms * 1e-3) / 1e12;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    CPHIFI_CHECK_LAUNCH();
}

// ---- large dense GEMMs through the MTTKRP v3 machinery (tensor-map TMA ring, DMMA) ---------
// C = A B with A column-major (M x K, the n x n kernel / eigenbasis) and B column- or row-major
// (K x N, N <= 64): a 2-mode "MTTKRP" with Wout = 1 (exact), split-K partials summed in split
// order by reduce_epi_kernel, which applies the GEMM epilogue.  (The cluster split-K DMMA GEMM
// above ran the config-4 contractions at ~49 % of the DMMA peak.)
__global__ void reduce_epi_kernel(const double* __restrict__ work, int P, int64_t m, int64_t ncols, const GemmArgs g) {
    const int64_t nn = g.c2 ? max(ncols, g.ld2) : ncols;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m * nn; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % m, j = e / m;
        const double acc = j < ncols ? sum_splits(work, P, m * ncols, e) : 0.0;
        epilogue_store(g, i, j, acc);
    }
}

// Split-K scratch of the plain GEMM, per host thread: grow-only, and a buffer it outgrows is
// retired, never freed — instantiated CUDA graphs (the PCG loop, the host-buffer matvec) hold its
// address for their lifetime, so freeing it would leave them writing into released memory.
struct GrowScratch {
    double* p = nullptr;
    size_t n = 0;
    int dev = -1;
    void ensure(int device, size_t need) {
        if (dev == device && n >= need) return;
        static std::mutex mu;
        static std::vector<double*> retired;  // alive until process exit
        std::lock_guard<std::mutex> lk(mu);
        if (p) retired.push_back(p);
        const size_t cnt = std::max(need + need / 2, (size_t)1 << 16);
        p = nullptr;
        CPHIFI_CUDA(cudaMalloc(&p, cnt * sizeof(double)));
        n = cnt;
        dev = device;
    }
    double* get() const { return p; }
};

// Split-K partials: one grow-only buffer per CUDA stream (each context owns its stream, and all
// work on a stream — direct launches and the graphs captured from it — runs in stream order, so
// the buffer is never used by two GEMMs at once; graphs keep the address they captured, which
// stays valid because outgrown buffers are retired, not freed).
GrowScratch& stream_scratch(cudaStream_t s) {
    static std::mutex mu;
    static std::map<cudaStream_t, GrowScratch> per_stream;
    std::lock_guard<std::mutex> lk(mu);
    return per_stream[s];
}

// The plain GEMM runs the MTTKRP ring with a single Khatri-Rao outer row Wout = 1: one constant
// buffer per device, filled once outside any graph capture (inside a capture the fill is a
// captured node in front of the GEMM, and the buffer is filled again on the next uncaptured call).
constexpr int ONES_N = 256;
__global__ void fill_ones_kernel(double* p) {
    if (threadIdx.x < ONES_N) p[threadIdx.x] = 1.0;
}
const double* gemm_ones(int dev, cudaStream_t s) {
    static std::mutex mu;
    static double* buf[64] = {nullptr};
    static bool filled[64] = {false};
    if (dev < 0 || dev >= 64) throw_runtime("gemm: device index out of range");
    std::lock_guard<std::mutex> lk(mu);
    if (!buf[dev]) CPHIFI_CUDA(cudaMalloc(&buf[dev], sizeof(double) * ONES_N));
    if (!filled[dev]) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        CPHIFI_CUDA(cudaStreamIsCapturing(s, &cs));
        fill_ones_kernel<<<1, ONES_N, 0, s>>>(buf[dev]);
        CPHIFI_CHECK_LAUNCH();
        if (cs == cudaStreamCaptureStatusNone) filled[dev] = true;
    }
    return buf[dev];
}

bool gemm_tma_ok(const GemmArgs& g) {
    if (const char* e = std::getenv("CPHIFI_GEMM_TMA"))
        if (std::atoi(e) == 0) return false;
    const bool bcol = g.b_rs == 1, brow = g.b_cs == 1 && !bcol;
    const int64_t ldb = bcol ? g.b_cs : g.b_rs;
    return g.m >= 512 && g.k >= 512 && g.n >= 1 && g.n <= 64 && g.a_rs == 1 && g.a_cs % 2 == 0 && (bcol || brow) &&
           ldb % 2 == 0 && reinterpret_cast<uintptr_t>(g.a) % 16 == 0 && reinterpret_cast<uintptr_t>(g.b) % 16 == 0 &&
           g.k < (1LL << 31) && g.m < (1LL << 31);
}

// EPI_GRAM: split-K reduction of Xhat rows (partials summed in p order, as reduce_epi_kernel) fused
// with the row-Gram apply Yhat(i, a) = sum_b G_i(b, a) Xhat(i, b) (b ascending, as gram_apply):
// bit-identical to the two launches it replaces.  GR rows per CTA, RP threads per row.
template <int RP>
__global__ void __launch_bounds__(RP * 2) reduce_gram_kernel(const double* __restrict__ work, int P, int64_t m,
                                                             int64_t ncols, const GemmArgs g) {
    constexpr int GR = 2;
    __shared__ double xs[GR][RP];
    const int rr = threadIdx.x / RP, a = threadIdx.x % RP;
    const int64_t i = (int64_t)blockIdx.x * GR + rr;
    const double x = (i < m && a < ncols) ? sum_splits(work, P, m * ncols, i + m * a) : 0.0;
    xs[rr][a] = x;
    __syncthreads();
    if (i >= m || g.row_ptr[i + 1] == g.row_ptr[i]) return;  // rows without observations stay zero
    const double* gi = g.gram + i * RP * RP + a;
    constexpr int U = RP < 16 ? RP : 16;
    double s = 0.0;
#pragma unroll
    for (int b0 = 0; b0 < RP; b0 += U) {
        double gv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) gv[u] = __ldcs(gi + (b0 + u) * RP);
#pragma unroll
        for (int u = 0; u < U; ++u) s = fma(gv[u], xs[rr][b0 + u], s);
    }
    g.yhat[i * RP + a] = s;
}

void launch_reduce_gram(const double* work, int P, int64_t m, int64_t ncols, const GemmArgs& g, cudaStream_t s) {
    const unsigned grid = (unsigned)((m + 1) / 2);
    switch (g.rp) {
        case 4: reduce_gram_kernel<4><<<grid, 8, 0, s>>>(work, P, m, ncols, g); break;
        case 8: reduce_gram_kernel<8><<<grid, 16, 0, s>>>(work, P, m, ncols, g); break;
        case 16: reduce_gram_kernel<16><<<grid, 32, 0, s>>>(work, P, m, ncols, g); break;
        case 32: reduce_gram_kernel<32><<<grid, 64, 0, s>>>(work, P, m, ncols, g); break;
        case 64: reduce_gram_kernel<64><<<grid, 128, 0, s>>>(work, P, m, ncols, g); break;
        default: throw_invalid("gemm: EPI_GRAM needs a padded rank in [4, 64]");
    }
    CPHIFI_CHECK_LAUNCH();
}

template <int BN>
int64_t splitk_depth_t(const GemmArgs& g, int num_sms) {  // as gemm_tma_t below
    const int mt = (int)((g.m + BMM - 1) / BMM), nt = (int)((g.n + BN - 1) / BN);
    const int64_t chunks = (g.k + BK - 1) / BK;
    return std::max<int64_t>(1, std::min<int64_t>((int64_t)num_sms / (mt * nt), chunks));
}

template <int BN>
void gemm_tma_t(const GemmArgs& g, int num_sms, cudaStream_t s) {
    GrowScratch& work = stream_scratch(s);
    int dev = 0;
    CPHIFI_CUDA(cudaGetDevice(&dev));
    const bool brow = !(g.b_rs == 1);
    const int mt = (int)((g.m + BMM - 1) / BMM), nt = (int)((g.n + BN - 1) / BN);
    const int64_t chunks = (g.k + BK - 1) / BK;
    int64_t P = std::max<int64_t>(1, std::min<int64_t>((int64_t)num_sms / (mt * nt), chunks));
    const size_t need = (size_t)P * g.m * g.n + 2;
    work.ensure(dev, need);
    const double* wout = gemm_ones(dev, s);
    MttkrpArgs a;
    a.d = 2;
    a.shape[0] = g.m;
    a.shape[1] = g.k;
    a.r = g.n;
    a.t = g.a;
    a.fac[1] = g.b;
    a.ld[1] = brow ? g.b_rs : g.b_cs;
    a.off1 = 0;
    a.ldw = (g.n + 1) & ~1LL;
    CUtensorMap tm_a, tm_b;
    const bool ok = encode_tmap_2d_f64(&tm_a, g.a, (uint64_t)g.m, (uint64_t)g.k, (uint64_t)g.a_cs, BMM + 4, BK) &&
                    (brow ? encode_tmap_2d_f64(&tm_b, g.b, (uint64_t)g.n, (uint64_t)g.k, (uint64_t)g.b_rs, BN + 4, BK)
                          : encode_tmap_2d_f64(&tm_b, g.b, (uint64_t)g.k, (uint64_t)g.n, (uint64_t)g.b_cs, BK + 4, BN));
    if (!ok) throw Error(CPHIFI_CUDA_ERROR, "gemm: tensor map encoding failed");
    constexpr int WC = BN >= 16 ? 16 : BN;
    if (brow) launch_v3<BN, 32, WC, true>(a, tm_a, tm_b, mt, P, nt, chunks, chunks, wout, work.get(), s);
    else launch_v3<BN, 32, WC, false>(a, tm_a, tm_b, mt, P, nt, chunks, chunks, wout, work.get(), s);
    if (g.epi == EPI_GRAM) {
        launch_reduce_gram(work.get(), (int)P, g.m, g.n, g, s);
        return;
    }
    if (g.epi == EPI_PARTIALS) {
        *g.parts_out = work.get();
        *g.p_out = (int)P;
        return;
    }
    const int64_t cnt = g.m * (g.c2 ? std::max(g.n, g.ld2) : g.n);
    reduce_epi_kernel<<<(unsigned)std::min<int64_t>((cnt + 255) / 256, 4 * num_sms), 256, 0, s>>>(work.get(), (int)P, g.m,
                                                                                                  g.n, g);
    CPHIFI_CHECK_LAUNCH();
}

int gemm_splitk_depth(const GemmArgs& g, int num_sms) {
    if (g.n <= 8) return (int)splitk_depth_t<8>(g, num_sms);
    if (g.n <= 16) return (int)splitk_depth_t<16>(g, num_sms);
    return (int)splitk_depth_t<32>(g, num_sms);
}

void gemm(const GemmArgs& g, int num_sms, cudaStream_t s) {
    if (g.m <= 0 || g.n <= 0) return;
    if (g.k <= 0) {
        // empty contraction: run a zero-K GEMM (epilogue only) through the S=1 path
    }
    if ((g.epi == EPI_GRAM || g.epi == EPI_PARTIALS) && !(g.k > 0 && gemm_tma_ok(g)))
        throw_invalid("gemm: EPI_GRAM / EPI_PARTIALS need the tensor-map path");
    if (g.k > 0 && gemm_tma_ok(g)) {
        if (g.n <= 8) gemm_tma_t<8>(g, num_sms, s);
        else if (g.n <= 16) gemm_tma_t<16>(g, num_sms, s);
        else gemm_tma_t<32>(g, num_sms, s);
        return;
    }
    const int64_t np = (g.n + 7) / 8 * 8;
    if (np <= 8) launch_gemm<8>(g, num_sms, s);
    else if (np <= 16) launch_gemm<16>(g, num_sms, s);
    else if (np <= 32) launch_gemm<32>(g, num_sms, s);
    else launch_gemm<64>(g, num_sms, s);
}

// ---- MTTKRP for the middle (k = 1) / last (k = 2) mode of a 3-way column-major tensor --------
// B_k = T_(k) Z_k: the contraction runs over (i0, outer) with outer = the remaining mode, in tiles
// of 32 consecutive i0 of one outer: the B tile is an A_0 block, the tile's Khatri-Rao row the
// remaining factor's row `outer` (tensor.hpp:158-182: Z_k = A_other (x) A_0, A_0 fastest).  The T
// tile is the transposed unfolding block through a 3-D (k = 1) or 2-D (k = 2) tensor map.
__global__ void rows_of_kernel(const double* __restrict__ f, int64_t ld, int64_t nrows, int64_t r, int64_t ldw,
                               double* __restrict__ wout) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e < nrows * r) wout[(e / r) * ldw + e % r] = f[e / r + ld * (e % r)];  // Wout(o, j) = F(o, j)
}

template <int BN>
void mttkrp_k3_t(const double* t, const int64_t* shape, int k, int64_t r, const double* a0, int64_t ld0,
                 const double* aoth, int64_t ldo, double* b_out, int num_sms, cudaStream_t s, DevBuf<double>& work) {
    const int64_t n0 = shape[0], nk = shape[k], nout = shape[3 - k];
    const int64_t chunks = (n0 + BK - 1) / BK, ktiles = chunks * nout;
    const int mt = (int)((nk + BMM - 1) / BMM), nt = (int)((r + BN - 1) / BN);
    int64_t P = std::max<int64_t>(1, std::min<int64_t>((int64_t)num_sms / (mt * nt), ktiles));
    const size_t need = (size_t)P * nk * r + (size_t)nout * ((r + 1) & ~1LL) + 2;
    if (work.n < need) work.alloc(need);
    double* wout = work.get() + (size_t)P * nk * r;
    rows_of_kernel<<<(unsigned)((nout * r + 255) / 256), 256, 0, s>>>(aoth, ldo, nout, r, (r + 1) & ~1LL, wout);
    CPHIFI_CHECK_LAUNCH();
    CUtensorMap tm_t, tm_b;
    bool ok = encode_tmap_2d_f64(&tm_b, a0, (uint64_t)ld0, (uint64_t)r, (uint64_t)ld0, BK + 4, BN);
    if (k == 1) ok = ok && encode_tmap_3d_f64(&tm_t, t, (uint64_t)n0, (uint64_t)shape[1], (uint64_t)shape[2], BK + 4, BMM, 1);
    else ok = ok && encode_tmap_2d_f64(&tm_t, t, (uint64_t)(n0 * shape[1]), (uint64_t)shape[2], (uint64_t)(n0 * shape[1]),
                                       BK + 4, BMM);
    if (!ok) throw Error(CPHIFI_CUDA_ERROR, "mttkrp: tensor map encoding failed");
    MttkrpArgs a;
    a.d = 3;
    a.shape[0] = nk;   // output rows
    a.shape[1] = n0;   // chunked contraction extent
    a.r = r;
    a.t = t;
    a.fac[1] = a0;
    a.ld[1] = ld0;
    a.off1 = 0;
    a.ldw = (r + 1) & ~1LL;
    constexpr int WC = BN >= 16 ? 16 : BN;
    if (k == 1) launch_v3<BN, 32, WC, false, 1>(a, tm_t, tm_b, mt, P, nt, chunks, ktiles, wout, work.get(), s);
    else launch_v3<BN, 32, WC, false, 2>(a, tm_t, tm_b, mt, P, nt, chunks, ktiles, wout, work.get(), s);
    const int64_t cnt = nk * r;
    reduce_splits_kernel<<<(unsigned)std::min<int64_t>((cnt + 255) / 256, 4 * num_sms), 256, 0, s>>>(work.get(), (int)P,
                                                                                                    cnt, b_out);
    CPHIFI_CHECK_LAUNCH();
}

bool mttkrp_k3_supported(int d, const int64_t* shape, int k, int64_t r) {
    return d == 3 && (k == 1 || k == 2) && shape[0] % 2 == 0 && r <= 64 && r >= 1 &&
           shape[0] * shape[1] < (1LL << 31) && shape[1] < (1LL << 31) && shape[2] < (1LL << 31);
}

void mttkrp_mode_k3(const double* t, const int64_t* shape, int k, int64_t r, const double* a0, int64_t ld0,
                    const double* aoth, int64_t ldo, double* b_out, int num_sms, cudaStream_t s, DevBuf<double>& work) {
    if (r <= 8) mttkrp_k3_t<8>(t, shape, k, r, a0, ld0, aoth, ldo, b_out, num_sms, s, work);
    else if (r <= 16) mttkrp_k3_t<16>(t, shape, k, r, a0, ld0, aoth, ldo, b_out, num_sms, s, work);
    else mttkrp_k3_t<32>(t, shape, k, r, a0, ld0, aoth, ldo, b_out, num_sms, s, work);
}

void mttkrp_mode0(const MttkrpArgs& a, int num_sms, cudaStream_t s, DevBuf<double>& work) {
    const int64_t np = (a.r + 7) / 8 * 8;
    if (np <= 8) launch_mttkrp<8>(a, num_sms, s, work);
    else if (np <= 16) launch_mttkrp<16>(a, num_sms, s, work);
    else if (np <= 32) launch_mttkrp<32>(a, num_sms, s, work);
    else launch_mttkrp<64>(a, num_sms, s, work);
}

void gram_kr(int d, const int64_t* shape, int64_t r, const double* const* fac, int k, double* v,
             cudaStream_t s) {
    if (d > 8) throw_invalid("gram_khatri_rao: order above 8 is not supported");
    GramKrArgs g;
    g.d = d;
    g.k = k;
    g.r = r;
    for (int m = 0; m < d; ++m) {
        g.fac[m] = fac[m];
        g.shape[m] = shape[m];
    }
    gram_kernel<<<blocks_for(r * r * 32, 256), 256, 0, s>>>(g, v);
    CPHIFI_CHECK_LAUNCH();
}

void kernel_matrix(int kind, const double* pts, int64_t n, double param, double* kmat, cudaStream_t s) {
    kernel_matrix_kernel<<<blocks_for(n * n, 256), 256, 0, s>>>(kind, pts, n, param, kmat);
    CPHIFI_CHECK_LAUNCH();
}
void clamp_nonneg(double* v, int64_t n, cudaStream_t s) {
    clamp_kernel<<<blocks_for(n, 256), 256, 0, s>>>(v, n);
    CPHIFI_CHECK_LAUNCH();
}
void max_asym(const double* a, int64_t n, double* out2, cudaStream_t s) {
    CPHIFI_CUDA(cudaMemsetAsync(out2, 0, 2 * sizeof(double), s));  // +0.0: the bit pattern 0
    const unsigned nt = (unsigned)((n + 31) / 32);
    max_asym_kernel<<<dim3(nt, nt), dim3(32, 8), 0, s>>>(a, n, reinterpret_cast<unsigned long long*>(out2));
    CPHIFI_CHECK_LAUNCH();
}
void precond_diag(const double* mu, const double* sv, int64_t n, int64_t r, double gamma, double lambda,
                  double rho, double* dmat, int* flag, cudaStream_t s) {
    precond_diag_kernel<<<blocks_for(n * r, 256), 256, 0, s>>>(mu, sv, n, r, gamma, lambda, rho, dmat, flag);
    CPHIFI_CHECK_LAUNCH();
}
void pack_rows(const double* src_cm, int64_t rows, int64_t ld, int64_t r, int64_t rp, double* dst_rm,
               cudaStream_t s) {
    pack_rows_kernel<<<blocks_for(rows * rp, 256), 256, 0, s>>>(src_cm, rows, ld, r, rp, dst_rm);
    CPHIFI_CHECK_LAUNCH();
}
void rm_to_cm(const double* src_rm, int64_t rows, int64_t rp, int64_t r, double* dst_cm, cudaStream_t s) {
    rm_to_cm_kernel<<<blocks_for(rows * r, 256), 256, 0, s>>>(src_rm, rows, rp, r, dst_cm);
    CPHIFI_CHECK_LAUNCH();
}

}  // namespace cphifi
