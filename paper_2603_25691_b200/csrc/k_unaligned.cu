// k_unaligned.cu — PCG vector kernels and observation-plan helpers for sm_100a.  (The
// per-observation operator kernel lives in k_fused.cu; its design notes follow.)
//
// K1 fuses the reference's two q-loops — gather_rows (observations.hpp:191-198) and
// sampled_mttkrp (:174-184) — into ONE pass over observations pre-sorted by i_k (CSR):
//     z_l = prod_{m != k} A_m(i_m(l), :)        (ascending mode order, build_zhat :150-156)
//     s_l = Xhat(i_k(l), :) . z_l               (or s_l = value_l for the RHS B, :186-188)
//     Yhat(i_k(l), :) += s_l z_l
// Zhat is never materialised.  Work is split into equal-COUNT units (robust to Zipf skew);
// a unit is one lane group that keeps its Yhat row accumulator in registers and flushes it
// once per row it touches.  Rows fully inside a unit are stored directly; a unit's first /
// last (possibly shared) row goes to slot_a / slot_b and a fix-up kernel sums the slots of
// every shared row in unit order.  No atomics: the result is bit-reproducible.
#include <cub/cub.cuh>

#include "kernels.cuh"

namespace cphifi {
namespace {

constexpr int SG_THREADS = 256;

// ---- PCG vector kernels ------------------------------------------------------------------
constexpr int RED_THREADS = 256;
constexpr int RED_BLOCKS = RED_GRID;  // fixed -> fixed summation tree -> deterministic (2 CTAs per SM)

__device__ __forceinline__ double block_sum(double v, double* sh) {
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double t = 0.0;
    if (w == 0) {
        t = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
        for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    }
    __syncthreads();
    return t;  // valid in thread 0
}

// Last-block-done pattern: every block writes its partial; the last block to finish sums
// the partials in block order (fixed) and runs `fin`.
template <class Fin>
__device__ __forceinline__ void finish_reduce(double local, double* partial, unsigned* ticket, Fin fin) {
    __shared__ double sh[32];
    __shared__ bool last;
    const double bsum = block_sum(local, sh);
    if (threadIdx.x == 0) {
        partial[blockIdx.x] = bsum;
        __threadfence();
        last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (last) {  // the partials in a fixed tree: thread t sums t, t + blockDim, ...; then block_sum
        __threadfence();
        double s = 0.0;
        for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) s += __ldcg(partial + b);
        s = block_sum(s, sh);
        if (threadIdx.x == 0) {
            *ticket = 0;
            fin(s);
        }
    }
}

__global__ void dot_kernel(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                           double* partial, double* out) {
    double t = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        t = fma(x[i], y[i], t);
    finish_reduce(t, partial, reinterpret_cast<unsigned*>(partial + RED_BLOCKS), [&](double s) { *out = s; });
}

// pap = p.ap (grid reduce #1, in this kernel), then step A2 does the updates.
__global__ void pcg_pap_kernel(const double* __restrict__ p, const double* __restrict__ ap, int64_t n,
                               PcgState* st, double* partial) {
    double t = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        t = fma(p[i], ap[i], t);
    finish_reduce(t, partial, reinterpret_cast<unsigned*>(partial + RED_BLOCKS), [&](double s) {
        st->pap = s;
        st->flag = !isfinite(s) ? 1 : (s <= 0.0 ? 2 : 0);
        st->alpha = st->rz / s;
    });
}

__global__ void pcg_xr_kernel(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                              const double* __restrict__ ap, int64_t n, PcgState* st, double* partial) {
    const double alpha = st->alpha;
    double t = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        x[i] += alpha * p[i];
        const double ri = r[i] - alpha * ap[i];
        r[i] = ri;
        t = fma(ri, ri, t);
    }
    finish_reduce(t, partial, reinterpret_cast<unsigned*>(partial + RED_BLOCKS), [&](double s) {
        st->rr = s;
        st->rel = sqrt(s) / st->bnorm;
    });
}

__global__ void pcg_rz_kernel(const double* __restrict__ r, const double* __restrict__ z, int64_t n, PcgState* st,
                              double* partial) {
    double t = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        t = fma(r[i], z[i], t);
    finish_reduce(t, partial, reinterpret_cast<unsigned*>(partial + RED_BLOCKS), [&](double s) {
        st->rz_new = s;
        st->beta = s / st->rz;
        st->rz = s;
    });
}

__global__ void pcg_p_kernel(const double* __restrict__ z, double* __restrict__ p, int64_t n, const PcgState* st) {
    const double beta = st->beta;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = z[i] + beta * p[i];
}

// init: rz = r.z, rr = r.r, rel; p = z
__global__ void pcg_init_kernel(const double* __restrict__ r, const double* __restrict__ z, double* __restrict__ p,
                                int64_t n, PcgState* st, double* partial) {
    double t = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        p[i] = z[i];
        t = fma(r[i], z[i], t);
    }
    finish_reduce(t, partial, reinterpret_cast<unsigned*>(partial + RED_BLOCKS), [&](double s) { st->rz = s; });
}
__global__ void pcg_rr_kernel(const double* __restrict__ r, int64_t n, PcgState* st, double* partial) {
    double t = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        t = fma(r[i], r[i], t);
    finish_reduce(t, partial, reinterpret_cast<unsigned*>(partial + RED_BLOCKS), [&](double s) {
        st->rr = s;
        st->rel = sqrt(s) / st->bnorm;
    });
}

__global__ void pcg_ctl_kernel(const PcgState* st, PcgCtl* c, cudaGraphConditionalHandle h) {
    const int it = ++c->it;
    const double rel = st->rel;
    if (c->hist && it - 1 < c->hist_cap) c->hist[it - 1] = rel;
    if (st->flag != 0 || !(rel > c->tol) || it >= c->max_iter) {
        c->stop = 1;
        cudaGraphSetConditional(h, 0);
    }
}

__global__ void pcg_prologue_kernel(PcgState* st, PcgCtl* c) {
    const double bn = sqrt(st->bnorm);
    st->bnorm = bn;
    c->zero_b = bn == 0.0;
}
__global__ void pcg_x0_kernel(double* __restrict__ x, double* __restrict__ res, const double* __restrict__ b, int64_t n,
                              const PcgCtl* c) {
    const bool warm = c->warm && !c->zero_b;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (!warm) {
            x[i] = 0.0;
            res[i] = b[i];
        }
    }
}
__global__ void pcg_loopctl_kernel(const PcgState* st, PcgCtl* c, cudaGraphConditionalHandle hwhile) {
    c->rel0 = st->rel;
    if (c->zero_b || !(st->rel > c->tol)) cudaGraphSetConditional(hwhile, 0u);
}

// ---- single-CTA fused PCG steps (small n r): one launch instead of two (or three) ----------
constexpr int ONE_T = 1024;
constexpr int64_t ONE_MAX = 32768;  // elements; above this the 64-block kernels are faster
__device__ __forceinline__ double cta_sum(double v, double* sh) {  // all threads get the total
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < ONE_T / 32; ++w) t += sh[w];
    __syncthreads();
    return t;
}
// pap, flag, alpha; x += alpha p, r -= alpha ap; rr, rel; then (ctl) the loop control
__global__ void __launch_bounds__(ONE_T) pcg_step_a1_kernel(double* __restrict__ x, double* __restrict__ r,
                                                            const double* __restrict__ p, const double* __restrict__ ap,
                                                            int64_t n, PcgState* st, PcgCtl* c,
                                                            cudaGraphConditionalHandle h) {
    __shared__ double sh[ONE_T / 32];
    double t = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += ONE_T) t = fma(p[i], ap[i], t);
    const double pap = cta_sum(t, sh);
    const int flag = !isfinite(pap) ? 1 : (pap <= 0.0 ? 2 : 0);
    const double alpha = st->rz / pap;
    t = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += ONE_T) {
        x[i] += alpha * p[i];
        const double ri = r[i] - alpha * ap[i];
        r[i] = ri;
        t = fma(ri, ri, t);
    }
    const double rr = cta_sum(t, sh);
    if (threadIdx.x == 0) {
        st->pap = pap;
        st->flag = flag;
        st->alpha = alpha;
        st->rr = rr;
        const double rel = sqrt(rr) / st->bnorm;
        st->rel = rel;
        if (c) {  // pcg_ctl_kernel's work
            const int it = ++c->it;
            if (c->hist && it - 1 < c->hist_cap) c->hist[it - 1] = rel;
            if (flag != 0 || !(rel > c->tol) || it >= c->max_iter) {
                c->stop = 1;
                cudaGraphSetConditional(h, 0);
            }
        }
    }
}
// rz_new, beta, rz; p = z + beta p
__global__ void __launch_bounds__(ONE_T) pcg_step_b1_kernel(const double* __restrict__ r, const double* __restrict__ z,
                                                            double* __restrict__ p, int64_t n, PcgState* st) {
    __shared__ double sh[ONE_T / 32];
    double t = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += ONE_T) t = fma(r[i], z[i], t);
    const double rz_new = cta_sum(t, sh);
    const double beta = rz_new / st->rz;
    for (int64_t i = threadIdx.x; i < n; i += ONE_T) p[i] = z[i] + beta * p[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        st->rz_new = rz_new;
        st->beta = beta;
        st->rz = rz_new;
    }
}

// 16-byte copies (either side may be mapped host memory: one PCIe stream instead of a DMA node)
__global__ void copy16_kernel(double2* __restrict__ dst, const double2* __restrict__ src, int64_t n2) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

__global__ void axpby_kernel(double* y, const double* a, double alpha, const double* b, double beta, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = alpha * a[i] + beta * b[i];
}

// y(i, j) = alpha x(i, j) for rows i < z of column-major n x r blocks
__global__ void scale_row_block_kernel(double* __restrict__ y, const double* __restrict__ x, int64_t z, int64_t n,
                                       int64_t r, double alpha) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < z * r; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % z, j = e / z;
        y[i + n * j] = alpha * x[i + n * j];
    }
}

// ---- observation plan helpers -------------------------------------------------------------
__global__ void check_range_kernel(const int32_t* idx, int d, int64_t q, const int64_t* shape, int* flag) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)d * q;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int m = (int)(e / q);
        const int32_t v = idx[e];
        if (v < 0 || (int64_t)v >= shape[m]) *flag = 1;
    }
}
__global__ void linear_index_kernel(const int32_t* idx, int d, int64_t q, const int64_t* stride, uint64_t* lin) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < q; l += (int64_t)gridDim.x * blockDim.x) {
        uint64_t s = 0;
        for (int m = 0; m < d; ++m) s += (uint64_t)idx[(int64_t)m * q + l] * (uint64_t)stride[m];
        lin[l] = s;
    }
}
__global__ void adjacent_equal_kernel(const uint64_t* a, int64_t q, int* flag) {
    for (int64_t l = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < q; l += (int64_t)gridDim.x * blockDim.x)
        if (a[l] == a[l - 1]) *flag = 1;
}
__global__ void iota_kernel(int32_t* p, int64_t q) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < q; l += (int64_t)gridDim.x * blockDim.x)
        p[l] = (int32_t)l;
}
__global__ void gather_i32_kernel(const int32_t* src, const int32_t* perm, int64_t lo, int64_t cnt, int32_t* dst) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < cnt; l += (int64_t)gridDim.x * blockDim.x)
        dst[l] = src[perm[lo + l]];
}
__global__ void gather_f64_kernel(const double* src, const int32_t* perm, int64_t lo, int64_t cnt, double* dst) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < cnt; l += (int64_t)gridDim.x * blockDim.x)
        dst[l] = src[perm[lo + l]];
}
// row_ptr[i] = lower_bound(keys, i) for i in [0, n]
__global__ void csr_kernel(const int32_t* keys, int64_t q, int64_t n, int64_t* row_ptr) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > n) return;
    int64_t lo = 0, hi = q;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)keys[mid] < i) lo = mid + 1; else hi = mid;
    }
    row_ptr[i] = lo;
}

// row_ptr[i] = lower_bound(keys, i * span) for i in [0, n] (keys = lexicographic u64 keys with
// the row index i_k as the most significant digit, span = product of the other mode sizes)
__global__ void csr64_kernel(const uint64_t* keys, int64_t q, int64_t n, uint64_t span, int64_t* row_ptr) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > n) return;
    const uint64_t key = (uint64_t)i * span;
    int64_t lo = 0, hi = q;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (keys[mid] < key) lo = mid + 1; else hi = mid;
    }
    row_ptr[i] = lo;
}

// cnt[i] += the number of DISTINCT keys of row i (sorted keys, row = key / span): each warp walks a
// contiguous stretch 32 keys at a time; a stretch inside one row (the common case) adds one ballot
// count to a warp-held running sum, flushed by one atomic per row change
__global__ void row_distinct_kernel(const uint64_t* keys, int64_t q, uint64_t span, unsigned long long* cnt) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t per = ((q + nwarp - 1) / nwarp + 31) / 32 * 32;
    const int64_t lo = warp * per, hi = min(q, lo + per);
    int64_t cur = -1;
    unsigned long long acc = 0;
    for (int64_t b = lo; b < hi; b += 32) {
        const int64_t l = b + lane;
        const bool in = l < hi;
        const uint64_t key = in ? keys[l] : 0;
        const bool first = in && (l == 0 || keys[l - 1] != key);
        const int64_t row = in ? (int64_t)(key / span) : -1;
        const int64_t r0 = __shfl_sync(0xffffffffu, row, 0);
        if (__all_sync(0xffffffffu, !in || row == r0)) {
            if (r0 != cur) {
                if (lane == 0 && acc) atomicAdd(cnt + cur, acc);
                cur = r0;
                acc = 0;
            }
            acc += (unsigned long long)__popc(__ballot_sync(0xffffffffu, first));
        } else if (first) {
            atomicAdd(cnt + row, 1ull);
        }
    }
    if (lane == 0 && acc) atomicAdd(cnt + cur, acc);
}

// Row-sharded output operand: B(i,:) = Yhat(i,:) + lambda X(i,:) on the rows this rank owns, Yhat(i,:)
// on the other rows of [lo, hi) (X column-major n x r, Yhat / B row-major with stride rp)
__global__ void shard_operand_kernel(const double* __restrict__ yhat, const double* __restrict__ x, int64_t n,
                                     int64_t r, int64_t rp, int64_t lo, int64_t hi, int64_t own_lo, int64_t own_hi,
                                     double lambda, double* __restrict__ b) {
    const int64_t cnt = (hi - lo) * rp;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < cnt; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = lo + e / rp, c = e % rp;
        double v = yhat[i * rp + c];
        if (c < r && i >= own_lo && i < own_hi) v += lambda * x[i + n * c];
        b[i * rp + c] = v;
    }
}

__global__ void decode_keys_kernel(const uint64_t* keys, int64_t nu, int d, int k, const int64_t* stride,
                                   const int64_t* shape, int32_t* idx_o, int64_t ldq) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < nu; l += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t key = keys[l];
        int mm = 0;
        for (int m = 0; m < d; ++m) {
            if (m == k) continue;
            idx_o[(int64_t)mm * ldq + l] = (int32_t)((key / (uint64_t)stride[m]) % (uint64_t)shape[m]);
            ++mm;
        }
    }
}

inline unsigned grid_for(int64_t n, int t, int cap = 8192) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + t - 1) / t, cap));
}

}  // namespace

void dot_to(const double* x, const double* y, int64_t n, double* partial, double* out, cudaStream_t s) {
    dot_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(x, y, n, partial, out);
    CPHIFI_CHECK_LAUNCH();
}
void pcg_step_a(double* x, double* r, const double* p, const double* ap, int64_t n, PcgState* st,
                double* partial, cudaStream_t s) {
    if (n <= ONE_MAX) {
        pcg_step_a1_kernel<<<1, ONE_T, 0, s>>>(x, r, p, ap, n, st, nullptr, cudaGraphConditionalHandle{});
    } else {
        pcg_pap_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(p, ap, n, st, partial);
        pcg_xr_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(x, r, p, ap, n, st, partial);
    }
    CPHIFI_CHECK_LAUNCH();
}
void pcg_step_a_ctl(double* x, double* r, const double* p, const double* ap, int64_t n, PcgState* st, double* partial,
                    PcgCtl* c, cudaGraphConditionalHandle h, cudaStream_t s) {
    if (n <= ONE_MAX) {
        pcg_step_a1_kernel<<<1, ONE_T, 0, s>>>(x, r, p, ap, n, st, c, h);
        CPHIFI_CHECK_LAUNCH();
    } else {
        pcg_step_a(x, r, p, ap, n, st, partial, s);
        pcg_ctl(st, c, h, s);
    }
}
void pcg_step_b(const double* r, const double* z, double* p, int64_t n, PcgState* st, double* partial,
                cudaStream_t s) {
    if (n <= ONE_MAX) {
        pcg_step_b1_kernel<<<1, ONE_T, 0, s>>>(r, z, p, n, st);
    } else {
        pcg_rz_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(r, z, n, st, partial);
        pcg_p_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(z, p, n, st);
    }
    CPHIFI_CHECK_LAUNCH();
}
void pcg_init(const double* r, const double* z, double* p, int64_t n, PcgState* st, double* partial,
              cudaStream_t s) {
    pcg_init_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(r, z, p, n, st, partial);
    pcg_rr_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(r, n, st, partial);
    CPHIFI_CHECK_LAUNCH();
}
void pcg_prologue(PcgState* st, PcgCtl* c, cudaStream_t s) {
    pcg_prologue_kernel<<<1, 1, 0, s>>>(st, c);
    CPHIFI_CHECK_LAUNCH();
}
void pcg_x0(double* x, double* res, const double* b, int64_t n, const PcgCtl* c, cudaStream_t s) {
    pcg_x0_kernel<<<grid_for(n, 256), 256, 0, s>>>(x, res, b, n, c);
    CPHIFI_CHECK_LAUNCH();
}
void pcg_loopctl(const PcgState* st, PcgCtl* c, cudaGraphConditionalHandle hwhile, cudaStream_t s) {
    pcg_loopctl_kernel<<<1, 1, 0, s>>>(st, c, hwhile);
    CPHIFI_CHECK_LAUNCH();
}
void pcg_ctl(const PcgState* st, PcgCtl* c, cudaGraphConditionalHandle h, cudaStream_t s) {
    pcg_ctl_kernel<<<1, 1, 0, s>>>(st, c, h);
    CPHIFI_CHECK_LAUNCH();
}
void copy_doubles(double* dst, const double* src, int64_t n, cudaStream_t s) {
    if (n % 2 != 0 || reinterpret_cast<uintptr_t>(dst) % 16 != 0 || reinterpret_cast<uintptr_t>(src) % 16 != 0) {
        CPHIFI_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyDefault, s));
        return;
    }
    const int64_t n2 = n / 2;
    copy16_kernel<<<(unsigned)std::min<int64_t>((n2 + 255) / 256, 64), 256, 0, s>>>(
        reinterpret_cast<double2*>(dst), reinterpret_cast<const double2*>(src), n2);
    CPHIFI_CHECK_LAUNCH();
}
void axpby(double* y, const double* a, double alpha, const double* b, double beta, int64_t n, cudaStream_t s) {
    axpby_kernel<<<grid_for(n, 256), 256, 0, s>>>(y, a, alpha, b, beta, n);
    CPHIFI_CHECK_LAUNCH();
}

void scale_row_block(double* y, const double* x, int64_t z, int64_t n, int64_t r, double alpha, cudaStream_t s) {
    if (z <= 0 || r <= 0) return;
    scale_row_block_kernel<<<grid_for(z * r, 256), 256, 0, s>>>(y, x, z, n, r, alpha);
    CPHIFI_CHECK_LAUNCH();
}

void check_range(const int32_t* idx, int d, int64_t q, const int64_t* shape_dev, int* flag, cudaStream_t s) {
    if (q == 0) return;
    check_range_kernel<<<grid_for((int64_t)d * q, 256), 256, 0, s>>>(idx, d, q, shape_dev, flag);
    CPHIFI_CHECK_LAUNCH();
}
void linear_index(const int32_t* idx, int d, int64_t q, const int64_t* stride, uint64_t* lin, cudaStream_t s) {
    if (q == 0) return;
    linear_index_kernel<<<grid_for(q, 256), 256, 0, s>>>(idx, d, q, stride, lin);
    CPHIFI_CHECK_LAUNCH();
}
void adjacent_equal(const uint64_t* sorted, int64_t q, int* flag, cudaStream_t s) {
    if (q < 2) return;
    adjacent_equal_kernel<<<grid_for(q, 256), 256, 0, s>>>(sorted, q, flag);
    CPHIFI_CHECK_LAUNCH();
}
void iota32(int32_t* p, int64_t q, cudaStream_t s) {
    if (q == 0) return;
    iota_kernel<<<grid_for(q, 256), 256, 0, s>>>(p, q);
    CPHIFI_CHECK_LAUNCH();
}
void gather_i32(const int32_t* src, const int32_t* perm, int64_t lo, int64_t cnt, int32_t* dst, cudaStream_t s) {
    if (cnt == 0) return;
    gather_i32_kernel<<<grid_for(cnt, 256), 256, 0, s>>>(src, perm, lo, cnt, dst);
    CPHIFI_CHECK_LAUNCH();
}
void gather_f64(const double* src, const int32_t* perm, int64_t lo, int64_t cnt, double* dst, cudaStream_t s) {
    if (cnt == 0) return;
    gather_f64_kernel<<<grid_for(cnt, 256), 256, 0, s>>>(src, perm, lo, cnt, dst);
    CPHIFI_CHECK_LAUNCH();
}
namespace {
__global__ void block_key_kernel(const int32_t* col, int64_t q, int32_t rows, int32_t* key) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < q; l += (int64_t)gridDim.x * blockDim.x)
        key[l] = col[l] / rows;
}
__global__ void row_of_kernel(const int64_t* row_ptr, int64_t n, int64_t q, int32_t* rows) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < q; l += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = n;  // largest i with row_ptr[i] <= l
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (row_ptr[mid] <= l) lo = mid;
            else hi = mid - 1;
        }
        rows[l] = (int32_t)lo;
    }
}
__global__ void add_i32_kernel(int32_t* p, int64_t cnt, int32_t delta) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < cnt; l += (int64_t)gridDim.x * blockDim.x)
        p[l] += delta;
}
}  // namespace

void block_key(const int32_t* col, int64_t q, int32_t rows, int32_t* key, cudaStream_t s) {
    if (q == 0) return;
    block_key_kernel<<<grid_for(q, 256), 256, 0, s>>>(col, q, rows, key);
    CPHIFI_CHECK_LAUNCH();
}
void row_of_entries(const int64_t* row_ptr, int64_t n, int64_t q, int32_t* rows, cudaStream_t s) {
    if (q == 0) return;
    row_of_kernel<<<grid_for(q, 256), 256, 0, s>>>(row_ptr, n, q, rows);
    CPHIFI_CHECK_LAUNCH();
}
void add_i32(int32_t* p, int64_t cnt, int32_t delta, cudaStream_t s) {
    if (cnt == 0 || delta == 0) return;
    add_i32_kernel<<<grid_for(cnt, 256), 256, 0, s>>>(p, cnt, delta);
    CPHIFI_CHECK_LAUNCH();
}

namespace {
__global__ void run_flag_kernel(const int32_t* rows, const int32_t* col0, int64_t q, unsigned char* flag) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < q; l += (int64_t)gridDim.x * blockDim.x)
        flag[l] = l == 0 || rows[l] != rows[l - 1] || col0[l] != col0[l - 1];
}
}  // namespace

int64_t build_run_starts(const int32_t* rows, const int32_t* col0, int64_t q, int32_t* run_start, cudaStream_t s) {
    if (q == 0) return 0;
    DevBuf<unsigned char> flag(q);
    DevBuf<int32_t> iota(q);
    DevBuf<int64_t> nsel(1);
    run_flag_kernel<<<grid_for(q, 256), 256, 0, s>>>(rows, col0, q, flag.get());
    CPHIFI_CHECK_LAUNCH();
    iota32(iota.get(), q, s);
    size_t bytes = 0;
    CPHIFI_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, iota.get(), flag.get(), run_start, nsel.get(), q, s));
    DevBuf<unsigned char> tmp(bytes);
    CPHIFI_CUDA(cub::DeviceSelect::Flagged(tmp.get(), bytes, iota.get(), flag.get(), run_start, nsel.get(), q, s));
    int64_t nr = 0;
    CPHIFI_CUDA(cudaMemcpyAsync(&nr, nsel.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CPHIFI_CUDA(cudaStreamSynchronize(s));
    return nr;
}

void csr_from_sorted(const int32_t* keys, int64_t q, int64_t n, int64_t* row_ptr, cudaStream_t s) {
    csr_kernel<<<(unsigned)((n + 1 + 255) / 256), 256, 0, s>>>(keys, q, n, row_ptr);
    CPHIFI_CHECK_LAUNCH();
}

void csr_from_sorted64(const uint64_t* keys, int64_t q, int64_t n, uint64_t span, int64_t* row_ptr, cudaStream_t s) {
    csr64_kernel<<<(unsigned)((n + 1 + 255) / 256), 256, 0, s>>>(keys, q, n, span, row_ptr);
    CPHIFI_CHECK_LAUNCH();
}

void row_distinct_counts(const uint64_t* keys, int64_t q, int64_t n, uint64_t span, unsigned long long* cnt,
                         cudaStream_t s) {
    CPHIFI_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * n, s));
    if (q == 0) return;
    row_distinct_kernel<<<grid_for(q, 256 * 32), 256, 0, s>>>(keys, q, span, cnt);
    CPHIFI_CHECK_LAUNCH();
}

void shard_operand(const double* yhat, const double* x, int64_t n, int64_t r, int64_t rp, int64_t lo, int64_t hi,
                   int64_t own_lo, int64_t own_hi, double lambda, double* b, cudaStream_t s) {
    if (hi <= lo) return;
    shard_operand_kernel<<<grid_for((hi - lo) * rp, 256), 256, 0, s>>>(yhat, x, n, r, rp, lo, hi, own_lo, own_hi,
                                                                      lambda, b);
    CPHIFI_CHECK_LAUNCH();
}

size_t radix_sort_pairs_bytes(int64_t q, int bits) {
    size_t bytes = 0;
    CPHIFI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                                (const int32_t*)nullptr, (int32_t*)nullptr, q, 0, bits));
    return bytes;
}
void radix_sort_pairs(void* temp, size_t temp_bytes, const int32_t* keys_in, int32_t* keys_out,
                      const int32_t* vals_in, int32_t* vals_out, int64_t q, int bits, cudaStream_t s) {
    CPHIFI_CUDA(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in, vals_out, q, 0,
                                                bits, s));
}
size_t radix_sort_pairs64_bytes(int64_t q, int bits) {
    size_t bytes = 0;
    CPHIFI_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                                (const int32_t*)nullptr, (int32_t*)nullptr, q, 0, bits));
    return bytes;
}
void radix_sort_pairs64(void* temp, size_t temp_bytes, const uint64_t* keys_in, uint64_t* keys_out,
                        const int32_t* vals_in, int32_t* vals_out, int64_t q, int bits, cudaStream_t s) {
    CPHIFI_CUDA(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in, vals_out, q, 0,
                                                bits, s));
}
int64_t coalesce_sorted(const uint64_t* keys, const double* vals, int64_t q, uint64_t* ukeys, int32_t* counts,
                        double* vsum, cudaStream_t s) {
    if (q == 0) return 0;
    DevBuf<int64_t> nrun(2);
    size_t b1 = 0, b2 = 0;
    CPHIFI_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, b1, keys, ukeys, counts, nrun.get(), q, s));
    CPHIFI_CUDA(cub::DeviceReduce::ReduceByKey(nullptr, b2, keys, ukeys, vals, vsum, nrun.get() + 1, cub::Sum(), q, s));
    DevBuf<unsigned char> tmp(std::max(b1, b2));
    CPHIFI_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.get(), b1, keys, ukeys, counts, nrun.get(), q, s));
    CPHIFI_CUDA(cub::DeviceReduce::ReduceByKey(tmp.get(), b2, keys, ukeys, vals, vsum, nrun.get() + 1, cub::Sum(), q, s));
    int64_t h[2] = {0, 0};
    CPHIFI_CUDA(cudaMemcpyAsync(h, nrun.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    CPHIFI_CUDA(cudaStreamSynchronize(s));
    if (h[0] != h[1]) throw_runtime("ObservationSet: coalescing run counts disagree");
    return h[0];
}
void decode_keys(const uint64_t* keys, int64_t nu, int d, int k, const int64_t* stride_dev, const int64_t* shape_dev,
                 int32_t* idx_o, int64_t ldq, cudaStream_t s) {
    if (nu == 0) return;
    decode_keys_kernel<<<grid_for(nu, 256), 256, 0, s>>>(keys, nu, d, k, stride_dev, shape_dev, idx_o, ldq);
    CPHIFI_CHECK_LAUNCH();
}
size_t radix_sort_keys64_bytes(int64_t q) {
    size_t bytes = 0;
    CPHIFI_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, (const uint64_t*)nullptr, (uint64_t*)nullptr, q));
    return bytes;
}
void radix_sort_keys64(void* temp, size_t temp_bytes, const uint64_t* in, uint64_t* out, int64_t q,
                       cudaStream_t s) {
    CPHIFI_CUDA(cub::DeviceRadixSort::SortKeys(temp, temp_bytes, in, out, q, 0, 64, s));
}

}  // namespace cphifi
