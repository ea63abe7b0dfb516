// k_unaligned.cu — the per-observation hot loop of the unaligned operator
// plus PCG vector kernels and observation-plan helpers, for sm_100a.
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

__device__ __forceinline__ int64_t row_of(const int64_t* __restrict__ row_ptr, int64_t n, int64_t pos) {
    // largest i with row_ptr[i] <= pos  (upper_bound - 1)
    int64_t lo = 0, hi = n;  // row_ptr[0] = 0 <= pos < row_ptr[n]
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(row_ptr + mid) <= pos) lo = mid; else hi = mid;
    }
    return lo;
}

template <int VPL>
struct Vec;
template <> struct Vec<1> {
    double v[1];
    __device__ __forceinline__ void load(const double* p) { v[0] = __ldg(p); }
};
template <> struct Vec<2> {
    double v[2];
    __device__ __forceinline__ void load(const double* p) {
        const double2 t = __ldg(reinterpret_cast<const double2*>(p));
        v[0] = t.x; v[1] = t.y;
    }
};
template <> struct Vec<4> {
    double v[4];
    __device__ __forceinline__ void load(const double* p) {
        const double2 t0 = __ldg(reinterpret_cast<const double2*>(p));
        const double2 t1 = __ldg(reinterpret_cast<const double2*>(p) + 1);
        v[0] = t0.x; v[1] = t0.y; v[2] = t1.x; v[3] = t1.y;
    }
};

// RP = padded rank (power of two >= 4); DO = number of other modes (d - 1).
template <int RP, int DO>
__global__ void __launch_bounds__(SG_THREADS) scatter_gather_kernel(const SgArgs a) {
    constexpr int G = RP < 32 ? RP : 32;  // lanes per observation group
    constexpr int VPL = RP / G;           // values per lane
    const int lane = threadIdx.x & 31;
    const int glane = lane % G;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane - glane));
    const int64_t unit = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
    if (unit >= a.units) return;
    const int64_t beg = unit * a.chunk;
    const int64_t end = min(a.q, beg + a.chunk);
    if (beg >= end) return;
    const int jb = glane * VPL;

    int64_t row = row_of(a.row_ptr, a.n, beg);
    const int64_t first_row = row;
    const int64_t last_row = row_of(a.row_ptr, a.n, end - 1);
    int64_t row_end = __ldg(a.row_ptr + row + 1);

    Vec<VPL> xh;
    double acc[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) acc[v] = 0.0;
    const bool dot = a.weights == nullptr;
    if (dot) xh.load(a.xhat + row * RP + jb);

    auto flush = [&](int64_t rr) {
        double* dst;
        if (rr == first_row) dst = a.slot_a + unit * RP;
        else if (rr == last_row) dst = a.slot_b + unit * RP;
        else dst = a.yhat + rr * RP;
#pragma unroll
        for (int v = 0; v < VPL; ++v) dst[jb + v] = acc[v];
    };

    for (int64_t l = beg; l < end; ++l) {
        if (l >= row_end) {
            flush(row);
#pragma unroll
            for (int v = 0; v < VPL; ++v) acc[v] = 0.0;
            do {
                ++row;
                row_end = __ldg(a.row_ptr + row + 1);
            } while (l >= row_end);
            if (dot) xh.load(a.xhat + row * RP + jb);
        }
        // z = A_{m0}(i) * A_{m1}(i) * ...   (ascending modes, starting from the first factor)
        Vec<VPL> z;
        {
            const int64_t ix = __ldg(a.idx + l);
            z.load(a.fac + a.fac_off[0] + ix * RP + jb);
        }
#pragma unroll
        for (int m = 1; m < DO; ++m) {
            const int64_t ix = __ldg(a.idx + (int64_t)m * a.q + l);
            Vec<VPL> f;
            f.load(a.fac + a.fac_off[m] + ix * RP + jb);
#pragma unroll
            for (int v = 0; v < VPL; ++v) z.v[v] *= f.v[v];
        }
        double s;
        if (dot) {
            double p = 0.0;
#pragma unroll
            for (int v = 0; v < VPL; ++v) p = fma(xh.v[v], z.v[v], p);
#pragma unroll
            for (int off = G / 2; off > 0; off >>= 1) p += __shfl_xor_sync(gmask, p, off, G);
            s = p;
        } else {
            s = __ldg(a.weights + l);
        }
#pragma unroll
        for (int v = 0; v < VPL; ++v) acc[v] = fma(s, z.v[v], acc[v]);
    }
    flush(row);
}

// Fix-up: one thread per (row, column j < rp).  See the file comment for the slot rules.
__global__ void sg_fixup_kernel(const SgArgs a) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= a.n * a.rp) return;
    const int64_t i = e / a.rp, j = e % a.rp;
    const int64_t rb = a.row_ptr[i], re = a.row_ptr[i + 1];
    if (rb == re) {
        a.yhat[e] = 0.0;
        return;
    }
    const int64_t u0 = rb / a.chunk, u1 = (re - 1) / a.chunk;
    auto uend = [&](int64_t u) { return min(a.q, (u + 1) * a.chunk); };
    if (u0 == u1) {
        const bool is_first = (rb == u0 * a.chunk);
        const bool is_last = (re == uend(u0));
        if (is_first) a.yhat[e] = a.slot_a[u0 * a.rp + j];
        else if (is_last) a.yhat[e] = a.slot_b[u0 * a.rp + j];
        // else interior: written directly by the unit
        return;
    }
    double s = (rb == u0 * a.chunk) ? a.slot_a[u0 * a.rp + j] : a.slot_b[u0 * a.rp + j];
    for (int64_t u = u0 + 1; u <= u1; ++u) s += a.slot_a[u * a.rp + j];
    a.yhat[e] = s;
}

template <int RP>
void launch_sg_rp(const SgArgs& a, unsigned blocks, cudaStream_t s) {
    switch (a.dother) {
        case 1: scatter_gather_kernel<RP, 1><<<blocks, SG_THREADS, 0, s>>>(a); break;
        case 2: scatter_gather_kernel<RP, 2><<<blocks, SG_THREADS, 0, s>>>(a); break;
        case 3: scatter_gather_kernel<RP, 3><<<blocks, SG_THREADS, 0, s>>>(a); break;
        case 4: scatter_gather_kernel<RP, 4><<<blocks, SG_THREADS, 0, s>>>(a); break;
        case 5: scatter_gather_kernel<RP, 5><<<blocks, SG_THREADS, 0, s>>>(a); break;
        default: throw_invalid("unaligned: tensor order above 6 is not supported");
    }
}

// ---- PCG vector kernels ------------------------------------------------------------------
constexpr int RED_THREADS = 256;
constexpr int RED_BLOCKS = 64;  // fixed -> fixed summation tree -> deterministic

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
    if (last && threadIdx.x == 0) {
        __threadfence();
        double s = 0.0;
        for (unsigned b = 0; b < gridDim.x; ++b) s += ((volatile double*)partial)[b];
        *ticket = 0;
        fin(s);
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

__global__ void axpby_kernel(double* y, const double* a, double alpha, const double* b, double beta, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = alpha * a[i] + beta * b[i];
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

inline unsigned grid_for(int64_t n, int t, int cap = 8192) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + t - 1) / t, cap));
}

}  // namespace

void sg_plan(int64_t q, int64_t rp, int num_sms, int64_t* units, int64_t* chunk) {
    const int64_t g = rp < 32 ? rp : 32;
    const int64_t groups_per_block = SG_THREADS / g;
    // enough resident groups to fill every SM several times, but >= 16 observations each
    int64_t u = (int64_t)num_sms * 8 * groups_per_block;
    u = std::min<int64_t>(u, std::max<int64_t>(1, (q + 15) / 16));
    int64_t c = std::max<int64_t>(1, (q + u - 1) / u);
    u = std::max<int64_t>(1, (q + c - 1) / c);
    *units = u;
    *chunk = c;
}

void scatter_gather(const SgArgs& a, cudaStream_t s) {
    sg_main(a, s);
    sg_fixup(a, s);
}

void sg_main(const SgArgs& a, cudaStream_t s) {
    if (a.q > 0) {
        const int64_t g = a.rp < 32 ? a.rp : 32;
        const int64_t threads = a.units * g;
        const unsigned blocks = (unsigned)((threads + SG_THREADS - 1) / SG_THREADS);
        switch (a.rp) {
            case 4: launch_sg_rp<4>(a, blocks, s); break;
            case 8: launch_sg_rp<8>(a, blocks, s); break;
            case 16: launch_sg_rp<16>(a, blocks, s); break;
            case 32: launch_sg_rp<32>(a, blocks, s); break;
            case 64: launch_sg_rp<64>(a, blocks, s); break;
            case 128: launch_sg_rp<128>(a, blocks, s); break;
            default: throw_invalid("unaligned: rank above 128 is not supported");
        }
        CPHIFI_CHECK_LAUNCH();
    }
}

void sg_fixup(const SgArgs& a, cudaStream_t s) {
    sg_fixup_kernel<<<grid_for(a.n * a.rp, 256, 1 << 20), 256, 0, s>>>(a);
    CPHIFI_CHECK_LAUNCH();
}

void dot_to(const double* x, const double* y, int64_t n, double* partial, double* out, cudaStream_t s) {
    dot_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(x, y, n, partial, out);
    CPHIFI_CHECK_LAUNCH();
}
void pcg_step_a(double* x, double* r, const double* p, const double* ap, int64_t n, PcgState* st,
                double* partial, cudaStream_t s) {
    pcg_pap_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(p, ap, n, st, partial);
    pcg_xr_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(x, r, p, ap, n, st, partial);
    CPHIFI_CHECK_LAUNCH();
}
void pcg_step_b(const double* r, const double* z, double* p, int64_t n, PcgState* st, double* partial,
                cudaStream_t s) {
    pcg_rz_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(r, z, n, st, partial);
    pcg_p_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(z, p, n, st);
    CPHIFI_CHECK_LAUNCH();
}
void pcg_init(const double* r, const double* z, double* p, int64_t n, PcgState* st, double* partial,
              cudaStream_t s) {
    pcg_init_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(r, z, p, n, st, partial);
    pcg_rr_kernel<<<RED_BLOCKS, RED_THREADS, 0, s>>>(r, n, st, partial);
    CPHIFI_CHECK_LAUNCH();
}
void axpby(double* y, const double* a, double alpha, const double* b, double beta, int64_t n, cudaStream_t s) {
    axpby_kernel<<<grid_for(n, 256), 256, 0, s>>>(y, a, alpha, b, beta, n);
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
void csr_from_sorted(const int32_t* keys, int64_t q, int64_t n, int64_t* row_ptr, cudaStream_t s) {
    csr_kernel<<<(unsigned)((n + 1 + 255) / 256), 256, 0, s>>>(keys, q, n, row_ptr);
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
