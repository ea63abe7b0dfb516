// k_pcgstep.cu — the PCG vector work of one iteration in ONE cooperative launch (large n, eigenbasis
// PCG, r <= 64), sm_100a.
//
// After the operator has produced Ap, solvers.hpp:59-80 does
//     pap = p'Ap  (stop on non-finite / <= 0);  alpha = rz / pap;  x += alpha p;  r -= alpha Ap;
//     rel = ||r|| / ||b||  (stop on rel <= tol or it == max_iter);  z = M^-1 r;
//     rz' = r'z;  beta = rz' / rz;  p = z + beta p
// which the graph body ran as six launches (pap, x/r update + rr, loop control, preconditioner,
// rz, p update).  Here CTA c owns row blocks of 32 rows (all r columns) of every vector, so
// every elementwise step and the eigenbasis preconditioner (row-local: z~(i,:) =
// ((r~(i,:) U_V) o D(i,:)) U_V', unaligned.hpp:135-139) touch only the CTA's own rows; the three
// dot products are the only grid-wide steps: per-CTA partials, a grid barrier, then every CTA
// sums the partials in the same fixed order (bit-identical scalars everywhere, deterministic).
// Lane = row (column-major vectors: each warp access is a contiguous 256-byte column segment),
// warp w = columns [w JT, (w + 1) JT).
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"

namespace cphifi {
namespace {

constexpr int ST = 256, SRB = 32, SW = ST / 32;

__device__ __forceinline__ unsigned long long ld_acquire_u64_s(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// monotonic 64-bit arrival counter (never reset while a solve runs; zeroed with the solve scratch)
__device__ __forceinline__ void grid_sync(unsigned long long* ctr) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long C = gridDim.x;
        __threadfence();
        const unsigned long long old = atomicAdd(ctr, 1ull);
        const unsigned long long target = old - old % C + C;
        while (ld_acquire_u64_s(ctr) < target) {
        }
    }
    __syncthreads();
}

// Sum of the grid's partials in a fixed order; every thread of every CTA gets the same bits.
__device__ __forceinline__ double grid_total(const double* partial, double* sh) {
    if (threadIdx.x < 32) {
        double s = 0.0;
        for (unsigned b = threadIdx.x; b < gridDim.x; b += 32) s += __ldcg(partial + b);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (threadIdx.x == 0) sh[0] = s;
    }
    __syncthreads();
    const double t = sh[0];
    __syncthreads();
    return t;
}

__device__ __forceinline__ double cta_total(double v, double* sh) {  // CTA sum, fixed order, to all
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if ((threadIdx.x & 31) == 0) sh[1 + (threadIdx.x >> 5)] = v;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < SW; ++w) t += sh[1 + w];
    __syncthreads();
    return t;
}

// JT consecutive doubles from shared memory, 16 bytes at a time when JT is even (the callers'
// offsets are multiples of JT doubles from a 16-byte aligned row start)
template <int JT>
__device__ __forceinline__ void ld_vec(double (&v)[JT], const double* p) {
    if constexpr (JT % 2 == 0) {
#pragma unroll
        for (int u = 0; u < JT; u += 2) {
            const double2 t = *reinterpret_cast<const double2*>(p + u);
            v[u] = t.x;
            v[u + 1] = t.y;
        }
    } else {
#pragma unroll
        for (int u = 0; u < JT; ++u) v[u] = p[u];
    }
}

template <int JT>
__global__ void __launch_bounds__(ST) pcg_step_fused_kernel(const PcgStepArgs a) {
    constexpr int RP = JT * SW;
    constexpr int LDU = RP + 2;
    extern __shared__ __align__(16) double smem[];
    double* suv = smem;              // suv[m * LDU + j] = U_V(m, j)
    double* suvt = suv + RP * LDU;   // suvt[m * LDU + j] = U_V(j, m)
    double* sr = suvt + RP * LDU;    // r~ block, then t, column-major [m][q]
    __shared__ double sh[1 + SW];
    const int64_t n = a.n;
    const int r = a.r;
    const int q = threadIdx.x & 31, w = threadIdx.x >> 5, j0 = w * JT;
    const int64_t nblk = (n + SRB - 1) / SRB;
    const int c = blockIdx.x, C = gridDim.x;
    PcgState* st = a.st;
    // a speculatively enqueued iteration after the stopping one (host loop) does nothing
    if (a.ctl && *(volatile const int*)&a.ctl->stop) return;
    const double rz_old = st->rz;
#pragma unroll
    for (int k = 0; k < (RP * RP + ST - 1) / ST; ++k) {  // U_V staged once (used in step 3)
        const int e = threadIdx.x + k * ST;
        const int m = e % RP, j = e / RP;
        if (e < RP * RP) {
            const double u = (m < r && j < r) ? a.uv[m + (int64_t)r * j] : 0.0;
            suv[m * LDU + j] = u;
            suvt[j * LDU + m] = u;
        }
    }
    // Every phase loads all of a thread's JT elements of each operand into registers before any
    // store (the vectors may alias as far as the compiler knows: interleaved load / store chains
    // serialised on L2 latency).
    const double* __restrict__ pp = a.p;
    const double* __restrict__ ap = a.ap;
    const int64_t am = n - a.null_rows;  // rows of the operator GEMM's output
    // Ap(i, j): rho p for the null-space rows; else the operator's output, or its split-K partials
    // reduced in p order with the EPI_ROWSCALE epilogue (bit-identical to reduce_epi_kernel)
    auto ap_at = [&](int64_t i, int j, double pvv) -> double {
        if (i < a.null_rows) return a.rho * pvv;
        if (!a.ap_parts) return ap[i + n * j];
        const int64_t e = (i - a.null_rows) + am * j;
        constexpr int PMAX = 4;  // split-K depth of the operator GEMM (148 SMs / tiles, capped by the host)
        double pt[PMAX];
#pragma unroll
        for (int q2 = 0; q2 < PMAX; ++q2) pt[q2] = q2 < a.ap_p ? __ldcg(a.ap_parts + (int64_t)q2 * am * r + e) : 0.0;
        double v = 0.0;
#pragma unroll
        for (int q2 = 0; q2 < PMAX; ++q2)
            if (q2 < a.ap_p) v += pt[q2];
        return a.mu[i] * (v + a.lambda * pvv) + a.rho * pvv;
    };
    // ---- 1: pap = p'Ap --------------------------------------------------------------------
    double t = 0.0;
    double av0[JT];  // the first own block's Ap, reused by phase 2
    for (int64_t b = c; b < nblk; b += C) {
        const int64_t i = b * SRB + q;
        double pv[JT], av[JT];
#pragma unroll
        for (int u = 0; u < JT; ++u) {
            const bool ok = i < n && j0 + u < r;
            pv[u] = ok ? pp[i + n * (j0 + u)] : 0.0;
            av[u] = ok ? ap_at(i, j0 + u, pv[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < JT; ++u) t = fma(pv[u], av[u], t);
        if (b == c) {
#pragma unroll
            for (int u = 0; u < JT; ++u) av0[u] = av[u];
        }
    }
    t = cta_total(t, sh);
    if (threadIdx.x == 0) a.partial[c] = t;
    grid_sync(a.barrier);
    const double pap = grid_total(a.partial, sh);
    const int flag = !isfinite(pap) ? 1 : (pap <= 0.0 ? 2 : 0);
    const double alpha = rz_old / pap;
    // ---- 2: x += alpha p, r -= alpha Ap, rr ---------------------------------------------------
    t = 0.0;
    for (int64_t b = c; b < nblk; b += C) {
        const int64_t i = b * SRB + q;
        double pv[JT], av[JT], xv[JT], rv[JT];
#pragma unroll
        for (int u = 0; u < JT; ++u) {
            const bool ok = i < n && j0 + u < r;
            const int64_t e = i + n * (j0 + u);
            pv[u] = ok ? pp[e] : 0.0;
            av[u] = !ok ? 0.0 : (b == c ? av0[u] : ap_at(i, j0 + u, pv[u]));
            xv[u] = ok ? a.x[e] : 0.0;
            rv[u] = ok ? a.res[e] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < JT; ++u) {
            xv[u] += alpha * pv[u];
            rv[u] -= alpha * av[u];
            t = fma(rv[u], rv[u], t);
        }
#pragma unroll
        for (int u = 0; u < JT; ++u) {
            if (i < n && j0 + u < r) {
                const int64_t e = i + n * (j0 + u);
                a.x[e] = xv[u];
                a.res[e] = rv[u];
            }
        }
    }
    t = cta_total(t, sh);
    if (threadIdx.x == 0) a.partial[C + c] = t;
    grid_sync(a.barrier);
    const double rr = grid_total(a.partial + C, sh);
    const double rel = sqrt(rr) / st->bnorm;
    if (c == 0 && threadIdx.x == 0) {
        st->pap = pap;
        st->flag = flag;
        st->alpha = alpha;
        st->rr = rr;
        st->rel = rel;
        if (a.ctl) {  // pcg_ctl_kernel's work
            PcgCtl* cc = a.ctl;
            const int it = ++cc->it;
            if (cc->hist && it - 1 < cc->hist_cap) cc->hist[it - 1] = rel;
            if (flag != 0 || !(rel > cc->tol) || it >= cc->max_iter) {
                cc->stop = 1;
                if (a.set_cond) cudaGraphSetConditional(a.h, 0);
            }
        }
    }
    // ---- 3: z = M^-1 r on the own row blocks, rz'; 4: p = z + beta p ----------------------------
    // z and the thread's r values stay in registers for phase 4 when the CTA owns one row block
    double zkeep[JT];  // the first own block's z
    t = 0.0;
    int nb_own = 0;
    for (int64_t b = c; b < nblk; b += C, ++nb_own) {
        const int64_t i = b * SRB + q;
        const bool row_ok = i < n;
        __syncthreads();  // previous block's readers of sr are done
        double rs[JT];
#pragma unroll
        for (int k = 0; k < JT; ++k) {
            const int m = w + k * SW;
            rs[k] = (row_ok && m < r) ? a.res[i + n * m] : 0.0;
        }
        double dv[JT], rmine[JT];
#pragma unroll
        for (int u = 0; u < JT; ++u) {
            const bool ok = row_ok && j0 + u < r;
            dv[u] = ok ? a.dmat[i + n * (j0 + u)] : 0.0;
            rmine[u] = ok ? a.res[i + n * (j0 + u)] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < JT; ++k) sr[(w + k * SW) * SRB + q] = rs[k];
        __syncthreads();
        double acc[JT];
#pragma unroll
        for (int u = 0; u < JT; ++u) acc[u] = 0.0;
#pragma unroll 4
        for (int m = 0; m < r; ++m) {  // JT contiguous U_V(m, j0 ..) as 16-byte broadcast loads
            const double v = sr[m * SRB + q];
            double um[JT];
            ld_vec<JT>(um, suv + m * LDU + j0);
#pragma unroll
            for (int u = 0; u < JT; ++u) acc[u] = fma(v, um[u], acc[u]);
        }
#pragma unroll
        for (int u = 0; u < JT; ++u) acc[u] *= dv[u];
        __syncthreads();
#pragma unroll
        for (int u = 0; u < JT; ++u) sr[(j0 + u) * SRB + q] = acc[u];
        __syncthreads();
#pragma unroll
        for (int u = 0; u < JT; ++u) acc[u] = 0.0;
#pragma unroll 4
        for (int m = 0; m < r; ++m) {  // U_V(j0 .., m) from the transposed copy
            const double v = sr[m * SRB + q];
            double um[JT];
            ld_vec<JT>(um, suvt + m * LDU + j0);
#pragma unroll
            for (int u = 0; u < JT; ++u) acc[u] = fma(v, um[u], acc[u]);
        }
#pragma unroll
        for (int u = 0; u < JT; ++u) {
            if (row_ok && j0 + u < r) {
                a.z[i + n * (j0 + u)] = acc[u];
                t = fma(rmine[u], acc[u], t);
            }
        }
        if (nb_own == 0) {
#pragma unroll
            for (int u = 0; u < JT; ++u) zkeep[u] = acc[u];
        }
    }
    t = cta_total(t, sh);
    if (threadIdx.x == 0) a.partial[2 * C + c] = t;
    grid_sync(a.barrier);
    const double rz_new = grid_total(a.partial + 2 * C, sh);
    const double beta = rz_new / rz_old;
    nb_own = 0;
    for (int64_t b = c; b < nblk; b += C, ++nb_own) {
        const int64_t i = b * SRB + q;
        double zv[JT], pv[JT];
#pragma unroll
        for (int u = 0; u < JT; ++u) {
            const bool ok = i < n && j0 + u < r;
            const int64_t e = i + n * (j0 + u);
            zv[u] = nb_own == 0 ? zkeep[u] : (ok ? a.z[e] : 0.0);
            pv[u] = ok ? a.p[e] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < JT; ++u) {
            if (i < n && j0 + u < r) a.p[i + n * (j0 + u)] = zv[u] + beta * pv[u];
        }
    }
    if (c == 0 && threadIdx.x == 0) {
        st->rz_new = rz_new;
        st->beta = beta;
        st->rz = rz_new;
    }
}

template <int JT>
size_t step_smem() {
    constexpr int RP = JT * SW;
    return sizeof(double) * (2 * RP * (RP + 2) + RP * SRB);
}

template <int JT>
int step_grid(int64_t n, int num_sms) {
    func_attr_once((const void*)pcg_step_fused_kernel<JT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                   (int)step_smem<JT>());
    int occ = 0;  // per device (a query, not cached: cheap next to the cooperative launch)
    CPHIFI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pcg_step_fused_kernel<JT>, ST, step_smem<JT>()));
    const int64_t nblk = (n + SRB - 1) / SRB;
    return (int)std::max<int64_t>(1, std::min<int64_t>(nblk, (int64_t)num_sms * std::min(std::max(occ, 1), 4)));
}

template <int JT>
void launch_step(const PcgStepArgs& a, int num_sms, cudaStream_t s) {
    const int grid = step_grid<JT>(a.n, num_sms);
    static const bool coop = [] {
        const char* e = std::getenv("CPHIFI_PCG_STEP_COOP");  // experiment: plain launch (grid <= SMs)
        return !e || std::atoi(e) != 0;
    }();
    if (!coop) {
        pcg_step_fused_kernel<JT><<<grid, ST, step_smem<JT>(), s>>>(a);
        CPHIFI_CHECK_LAUNCH();
        return;
    }
    void* args[] = {const_cast<PcgStepArgs*>(&a)};
    CPHIFI_CUDA(cudaLaunchCooperativeKernel((const void*)pcg_step_fused_kernel<JT>, dim3(grid), dim3(ST), args,
                                            step_smem<JT>(), s));
}

}  // namespace

int pcg_step_fused_partials(int64_t n, int num_sms) { return 3 * (int)std::min<int64_t>((n + SRB - 1) / SRB, 4 * num_sms); }

void pcg_step_fused(const PcgStepArgs& a, int num_sms, cudaStream_t s) {
    if (a.r <= 8) launch_step<1>(a, num_sms, s);
    else if (a.r <= 16) launch_step<2>(a, num_sms, s);
    else if (a.r <= 32) launch_step<4>(a, num_sms, s);
    else if (a.r <= 64) launch_step<8>(a, num_sms, s);
    else throw_invalid("pcg_step_fused: rank above 64");
}

}  // namespace cphifi
