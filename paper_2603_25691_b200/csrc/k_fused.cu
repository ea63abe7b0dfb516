// k_fused.cu — the unaligned operator as ONE persistent cooperative kernel (sm_100a).
//
//   y = vec(K Yhat + lambda Xhat) + rho x,  Xhat = K X,
//   Yhat(i,:) = sum_{l: i_k(l)=i} (Xhat(i,:) . z_l) z_l,  z_l = prod_{m!=k} A_m(i_m(l),:)
// (unaligned.hpp:101-115 with gather_rows + sampled_mttkrp, observations.hpp:174-198, fused).
//
// Phases, separated by a software grid barrier (all CTAs co-resident: cooperative launch):
//   A  Xhat rows            CTA c computes rows [c n / C, (c+1) n / C)      (small n only)
//   B  scatter-gather       CTA c streams observations [c*chunk, (c+1)*chunk) of the i_k-sorted
//                           set in ROUNDS of NG consecutive observations, one per lane group
//                           (G lanes x VPL doubles = the padded rank).  Each group keeps its
//                           row accumulator in registers; when the round crosses a row boundary
//                           the CTA reduces the groups' accumulators in group order through
//                           shared memory and writes the row: directly to Yhat if the row is
//                           interior to the CTA, else to the CTA's slot A (first row) / B (last).
//   C1 fix-up               rows split across CTAs = slot sums in CTA order
//   C2 y rows               y = K Yhat + lambda Xhat + rho x                  (small n only)
// Every reduction has a fixed order, so results are bit-reproducible for a given launch shape.
// Factor rows are staged in shared memory when they fit (SURVEY §7 hard part 4).
#include <cooperative_groups.h>

#include "kernels.cuh"

namespace cphifi {
namespace {

constexpr int FT = 256;  // threads per CTA

__device__ __forceinline__ void grid_barrier(unsigned* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* vb = bar;
        const unsigned gen = vb[1];
        __threadfence();
        const unsigned arrived = atomicAdd(bar, 1u);
        if (arrived == gridDim.x - 1) {
            vb[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (vb[1] == gen) __nanosleep(40);
        }
        __threadfence();
    }
    __syncthreads();
}

template <int VPL>
__device__ __forceinline__ void ldv(double (&v)[VPL], const double* p) {
    if constexpr (VPL == 1) {
        v[0] = p[0];
    } else if constexpr (VPL == 2) {
        const double2 t = *reinterpret_cast<const double2*>(p);
        v[0] = t.x; v[1] = t.y;
    } else {
#pragma unroll
        for (int u = 0; u < VPL; u += 2) {
            const double2 t = *reinterpret_cast<const double2*>(p + u);
            v[u] = t.x; v[u + 1] = t.y;
        }
    }
}

// Small dense row kernel: out(i, j) = sum_k M(k, i) * V(k, j) for rows i of this CTA (M is
// symmetric n x n column-major, so column i is row i; V(k, j) at v[k*vs_r + j*vs_c]).
// thread t -> column j = t / S, k-slice s = t % S; slices are summed in order.
template <int RP>
__device__ __forceinline__ void rows_times(const FusedArgs& a, int64_t i, const double* __restrict__ v,
                                           int64_t vs_r, int64_t vs_c, double* red, double* out_j) {
    constexpr int S = FT / RP;
    const int j = threadIdx.x / S, s = threadIdx.x % S;
    double t = 0.0;
    if (j < a.r) {
        const double* mcol = a.kmat + i * a.n;
        for (int64_t k = s; k < a.n; k += S) t = fma(mcol[k], v[k * vs_r + j * vs_c], t);
    }
    red[threadIdx.x] = t;
    __syncthreads();
    if (threadIdx.x < RP) {
        double acc = 0.0;
        for (int q = 0; q < S; ++q) acc += red[threadIdx.x * S + q];
        out_j[threadIdx.x] = acc;
    }
    __syncthreads();
}

template <int RP, int DO, bool SMEMF>
__global__ void __launch_bounds__(FT) fused_matvec_kernel(const FusedArgs a) {
    constexpr int G = RP < 32 ? RP : 32;
    constexpr int VPL = RP / G;
    constexpr int NG = FT / G;
    extern __shared__ __align__(16) double smem[];
    double* red = smem;                    // NG * RP doubles (>= FT)
    double* rowbuf = red + (NG * RP > FT ? NG * RP : FT);  // 2 * RP doubles
    double* sfac = rowbuf + 2 * RP;        // staged factors (SMEMF)
    __shared__ int64_t s_rows[2];

    const int c = blockIdx.x, C = gridDim.x;
    const int g = threadIdx.x / G, glane = threadIdx.x % G, jb = glane * VPL;
    const int lane = threadIdx.x & 31;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane - lane % G));

    // stage the packed factors (row-major, rp-padded) in shared memory
    if constexpr (SMEMF) {
        const double2* src = reinterpret_cast<const double2*>(a.fac);
        double2* dst = reinterpret_cast<double2*>(sfac);
        for (int64_t e = threadIdx.x; e < a.fac_total / 2; e += FT) dst[e] = src[e];
    }
    const double* fac = SMEMF ? sfac : a.fac;

    // ---- phase A: Xhat rows (small n) ----------------------------------------------------
    if (a.phases & PH_A) {
        const int64_t i0 = a.n * c / C, i1 = a.n * (c + 1) / C;
        for (int64_t i = i0; i < i1; ++i) {
            rows_times<RP>(a, i, a.x, 1, a.n, red, rowbuf);
            if (threadIdx.x < RP) a.xhat_rm[i * RP + threadIdx.x] = threadIdx.x < a.r ? rowbuf[threadIdx.x] : 0.0;
        }
        grid_barrier(a.barrier);
    }

    // ---- phase B: fused gather / scatter over this CTA's observations ---------------------
    if (a.phases & PH_B) {
        const int64_t ca = min(a.q, (int64_t)c * a.chunk), cb = min(a.q, ca + a.chunk);
        if (ca < cb) {
            if (threadIdx.x == 0) {
                s_rows[0] = a.cta_rows[2 * c];
                s_rows[1] = a.cta_rows[2 * c + 1];
            }
            __syncthreads();
            const int64_t first_row = s_rows[0], last_row = s_rows[1];
            int64_t cur = first_row;
            int64_t cur_end = a.row_ptr[cur + 1];
            const bool dot = a.weights == nullptr;
            double xh[VPL], acc[VPL];
#pragma unroll
            for (int v = 0; v < VPL; ++v) acc[v] = 0.0;
            if (dot) ldv<VPL>(xh, a.xhat_rm + cur * RP + jb);

            auto flush = [&](int64_t row) {
                __syncthreads();
#pragma unroll
                for (int v = 0; v < VPL; ++v) red[g * RP + jb + v] = acc[v];
                __syncthreads();
                if (threadIdx.x < RP) {
                    double s = 0.0;
                    for (int q = 0; q < NG; ++q) s += red[q * RP + threadIdx.x];
                    double* dst = row == first_row ? a.slot_a + (int64_t)c * RP
                                : row == last_row ? a.slot_b + (int64_t)c * RP
                                                  : a.yhat_rm + row * RP;
                    dst[threadIdx.x] = s;
                }
#pragma unroll
                for (int v = 0; v < VPL; ++v) acc[v] = 0.0;
            };

            for (int64_t base = ca; base < cb; base += NG) {
                const int64_t l = base + g;
                const bool valid = l < cb;
                const int64_t last_l = min(base + NG, cb) - 1;
                double z[VPL];
                double w = 0.0;
                if (valid) {
                    ldv<VPL>(z, fac + a.fac_off[0] + (int64_t)__ldg(a.idx + l) * RP + jb);
#pragma unroll
                    for (int m = 1; m < DO; ++m) {
                        double f[VPL];
                        ldv<VPL>(f, fac + a.fac_off[m] + (int64_t)__ldg(a.idx + (int64_t)m * a.q + l) * RP + jb);
#pragma unroll
                        for (int v = 0; v < VPL; ++v) z[v] *= f[v];
                    }
                    if (!dot) w = __ldg(a.weights + l);
                }
                auto contribute = [&]() {
                    double s;
                    if (dot) {
                        double p = 0.0;
#pragma unroll
                        for (int v = 0; v < VPL; ++v) p = fma(xh[v], z[v], p);
#pragma unroll
                        for (int off = G / 2; off > 0; off >>= 1) p += __shfl_xor_sync(gmask, p, off, G);
                        s = p;
                    } else {
                        s = w;
                    }
#pragma unroll
                    for (int v = 0; v < VPL; ++v) acc[v] = fma(s, z[v], acc[v]);
                };
                if (last_l < cur_end) {  // whole round inside the current row (common case)
                    if (valid) contribute();
                } else {
                    bool done = !valid;
                    while (true) {
                        if (!done && l < cur_end) {
                            contribute();
                            done = true;
                        }
                        if (last_l < cur_end) break;
                        flush(cur);
                        // next row holding observation position cur_end (skip empty rows)
                        const int64_t pos = cur_end;
                        do {
                            ++cur;
                            cur_end = a.row_ptr[cur + 1];
                        } while (cur_end <= pos);
                        if (dot) ldv<VPL>(xh, a.xhat_rm + cur * RP + jb);
                    }
                }
            }
            flush(cur);
        }
        if (a.phases & (PH_C1 | PH_C2)) grid_barrier(a.barrier);
    }

    // ---- phase C1: rows split across CTAs = ordered slot sums ----------------------------
    if (a.phases & PH_C1) {
        for (int64_t e = (int64_t)c * FT + threadIdx.x; e < a.n * RP; e += (int64_t)C * FT) {
            const int64_t i = e / RP, j = e % RP;
            const int64_t rb = a.row_ptr[i], re = a.row_ptr[i + 1];
            if (rb == re) {
                a.yhat_rm[e] = 0.0;
                continue;
            }
            const int64_t u0 = rb / a.chunk, u1 = (re - 1) / a.chunk;
            const bool first_of_u0 = rb == u0 * a.chunk;
            if (u0 == u1) {
                const bool last_of_u0 = re == min(a.q, (u0 + 1) * a.chunk);
                if (first_of_u0) a.yhat_rm[e] = a.slot_a[u0 * RP + j];
                else if (last_of_u0) a.yhat_rm[e] = a.slot_b[u0 * RP + j];
                continue;  // else interior: written in phase B
            }
            double s = first_of_u0 ? a.slot_a[u0 * RP + j] : a.slot_b[u0 * RP + j];
            for (int64_t u = u0 + 1; u <= u1; ++u) s += a.slot_a[u * RP + j];
            a.yhat_rm[e] = s;
        }
        if (a.phases & PH_C2) grid_barrier(a.barrier);
    }

    // ---- phase C2: y = (K Yhat + lambda Xhat) + rho x  (small n) ------------------------------
    if (a.phases & PH_C2) {
        const int64_t i0 = a.n * c / C, i1 = a.n * (c + 1) / C;
        for (int64_t i = i0; i < i1; ++i) {
            rows_times<RP>(a, i, a.yhat_rm, RP, 1, red, rowbuf);
            if (threadIdx.x < a.r) {
                const int64_t e = i + a.n * threadIdx.x;
                double out = rowbuf[threadIdx.x] + a.lambda * a.xhat_rm[i * RP + threadIdx.x];
                a.y[e] = out + a.rho * a.x[e];
            }
        }
    }
}

template <int RP, int DO, bool SMEMF>
void launch_fused_t(const FusedArgs& a, int grid, size_t smem, cudaStream_t s) {
    auto kern = fused_matvec_kernel<RP, DO, SMEMF>;
    static bool attr = false;
    if (!attr) {
        CPHIFI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    void* args[] = {const_cast<FusedArgs*>(&a)};
    CPHIFI_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(FT), args, smem, s));
}

template <int RP, bool SMEMF>
void launch_fused_do(const FusedArgs& a, int grid, size_t smem, cudaStream_t s) {
    switch (a.dother) {
        case 1: launch_fused_t<RP, 1, SMEMF>(a, grid, smem, s); break;
        case 2: launch_fused_t<RP, 2, SMEMF>(a, grid, smem, s); break;
        case 3: launch_fused_t<RP, 3, SMEMF>(a, grid, smem, s); break;
        case 4: launch_fused_t<RP, 4, SMEMF>(a, grid, smem, s); break;
        case 5: launch_fused_t<RP, 5, SMEMF>(a, grid, smem, s); break;
        default: throw_invalid("unaligned: tensor order above 6 is not supported");
    }
}

template <int RP>
void launch_fused_rp(const FusedArgs& a, int grid, size_t smem, bool smemf, cudaStream_t s) {
    if (smemf) launch_fused_do<RP, true>(a, grid, smem, s);
    else launch_fused_do<RP, false>(a, grid, smem, s);
}

template <int RP, int DO, bool SMEMF>
int occupancy_t(size_t smem) {
    int blocks = 0;
    CPHIFI_CUDA(cudaFuncSetAttribute(fused_matvec_kernel<RP, DO, SMEMF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     200 * 1024));
    CPHIFI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fused_matvec_kernel<RP, DO, SMEMF>, FT, smem));
    return blocks;
}

__global__ void cta_rows_kernel(const int64_t* row_ptr, int64_t n, int64_t q, int64_t chunk, int C, int64_t* out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    const int64_t ca = min(q, (int64_t)c * chunk), cb = min(q, ca + chunk);
    auto row_of = [&](int64_t pos) {
        int64_t lo = 0, hi = n;
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (row_ptr[mid] <= pos) lo = mid; else hi = mid;
        }
        return lo;
    };
    out[2 * c] = ca < cb ? row_of(ca) : 0;
    out[2 * c + 1] = ca < cb ? row_of(cb - 1) : 0;
}

}  // namespace

size_t fused_smem_bytes(int64_t rp, int64_t fac_total, bool smemf) {
    const int64_t g = rp < 32 ? rp : 32;
    const int64_t ng = FT / g;
    const int64_t red = std::max<int64_t>(ng * rp, FT);
    return sizeof(double) * (red + 2 * rp + (smemf ? fac_total : 0));
}

int fused_grid(int64_t rp, int dother, bool smemf, size_t smem, int num_sms) {
    int occ = 0;
#define OCC(RPV)                                                                    \
    case RPV:                                                                       \
        switch (dother) {                                                           \
            case 1: occ = smemf ? occupancy_t<RPV, 1, true>(smem) : occupancy_t<RPV, 1, false>(smem); break; \
            case 2: occ = smemf ? occupancy_t<RPV, 2, true>(smem) : occupancy_t<RPV, 2, false>(smem); break; \
            case 3: occ = smemf ? occupancy_t<RPV, 3, true>(smem) : occupancy_t<RPV, 3, false>(smem); break; \
            case 4: occ = smemf ? occupancy_t<RPV, 4, true>(smem) : occupancy_t<RPV, 4, false>(smem); break; \
            default: occ = smemf ? occupancy_t<RPV, 5, true>(smem) : occupancy_t<RPV, 5, false>(smem); break; \
        }                                                                           \
        break;
    switch (rp) {
        OCC(4) OCC(8) OCC(16) OCC(32) OCC(64) OCC(128)
        default: throw_invalid("unaligned: rank above 128 is not supported");
    }
#undef OCC
    if (occ < 1) throw_runtime("fused matvec: kernel does not fit on an SM");
    return num_sms * std::min(occ, 4);
}

void fused_cta_rows(const int64_t* row_ptr, int64_t n, int64_t q, int64_t chunk, int C, int64_t* out,
                    cudaStream_t s) {
    cta_rows_kernel<<<(C + 127) / 128, 128, 0, s>>>(row_ptr, n, q, chunk, C, out);
    CPHIFI_CHECK_LAUNCH();
}

void fused_matvec(const FusedArgs& a, int grid, size_t smem, bool smemf, cudaStream_t s) {
    switch (a.rp) {
        case 4: launch_fused_rp<4>(a, grid, smem, smemf, s); break;
        case 8: launch_fused_rp<8>(a, grid, smem, smemf, s); break;
        case 16: launch_fused_rp<16>(a, grid, smem, smemf, s); break;
        case 32: launch_fused_rp<32>(a, grid, smem, smemf, s); break;
        case 64: launch_fused_rp<64>(a, grid, smem, smemf, s); break;
        case 128: launch_fused_rp<128>(a, grid, smem, smemf, s); break;
        default: throw_invalid("unaligned: rank above 128 is not supported");
    }
}

}  // namespace cphifi
