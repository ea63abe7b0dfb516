// k_gram.cu — the row-Gram form of the unaligned operator (sm_100a).
//
// For every row i of the infinite mode, the reference's gather + scatter
// (observations.hpp:174-198, called per PCG iteration by unaligned.hpp:110-111) is
//     Yhat(i,:) = sum_{l: i_k(l)=i} (Xhat(i,:) . z_l) z_l = Xhat(i,:) G_i,
//     G_i = sum_{l: i_k(l)=i} z_l z_l'      (rp x rp, symmetric, independent of X)
// — an exact algebraic identity.  G is built ONCE per subproblem (O(q rp^2) flops, one pass over
// the observations) and every operator application then costs O(n rp^2) instead of O(q d r).
// Duplicated multi-indices (multiset configs) add z z' once per copy, or once with weight
// mult_l in a coalesced plan.
//
// gram_build_kernel: CTA c walks the same row-aligned observation ranges as the fused kernel,
//   building z for batches of GB observations of one row in shared memory and accumulating
//   Z'Z in registers (each thread owns a BLK x BLK block of G).  Rows split across CTAs are
//   finished by the last CTA (per-row arrival counter, ordered slot sum) — deterministic.
// gram_apply_kernel: Yhat(i, a) = sum_b G_i(b, a) Xhat(i, b); thread (i, a), consecutive a
//   read consecutive G entries (G_i symmetric, so its row-major and column-major layouts agree).
#include <cstdlib>

#include "kernels.cuh"

namespace cphifi {
namespace {

constexpr int GT = 256;  // threads per CTA
constexpr int GB = 32;   // observations per z batch

__device__ __forceinline__ unsigned atom_add_acqrel_g(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

template <int RP, int DO>
__global__ void __launch_bounds__(GT) gram_build_kernel(const GramArgs a) {
    constexpr int BLK = RP >= 64 ? 4 : (RP >= 32 ? 2 : 1);  // thread block of G entries
    constexpr int NB = RP / BLK;                           // blocks per dimension
    constexpr int NACT = NB * NB;                          // active threads (<= GT)
    static_assert(NACT <= GT, "G tile does not fit the CTA");
    __shared__ __align__(16) double zs[GB][RP + 2];
    __shared__ double ws[GB];  // entry weights (coalesced plan multiplicities)
    __shared__ int s_last;
    const int c = blockIdx.x;
    const int64_t ca = a.cta_beg[c], cb = a.cta_beg[c + 1];
    if (ca >= cb) return;
    const int tid = threadIdx.x;
    const bool act = tid < NACT;
    const int ba = (tid / NB) * BLK, bb = (tid % NB) * BLK;
    const int64_t first_row = a.cta_rows[2 * c];
    double acc[BLK][BLK];
#pragma unroll
    for (int x = 0; x < BLK; ++x)
#pragma unroll
        for (int y = 0; y < BLK; ++y) acc[x][y] = 0.0;

    int64_t row = first_row;
    int64_t row_end = a.row_ptr[row + 1];
    auto finish_row = [&](int64_t rr) {
        const int ncta = a.row_ncta[rr];
        double* dst = ncta == 1 ? a.g + rr * RP * RP
                    : rr == first_row ? a.slot_a + (int64_t)c * RP * RP
                                      : a.slot_b + (int64_t)c * RP * RP;
        if (act) {
#pragma unroll
            for (int x = 0; x < BLK; ++x)
#pragma unroll
                for (int y = 0; y < BLK; ++y) dst[(ba + x) * RP + bb + y] = acc[x][y];
        }
#pragma unroll
        for (int x = 0; x < BLK; ++x)
#pragma unroll
            for (int y = 0; y < BLK; ++y) acc[x][y] = 0.0;
        if (ncta > 1) {  // the last CTA of a split row sums the slots in CTA order
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                s_last = atom_add_acqrel_g(a.rowcnt + rr, 1u) == (unsigned)ncta - 1;
                if (s_last) a.rowcnt[rr] = 0;
            }
            __syncthreads();
            if (s_last) {
                const int u0 = a.row_first_cta[rr];
                const bool starts = a.row_ptr[rr] == a.cta_beg[u0];
                for (int e = tid; e < RP * RP; e += GT) {
                    double s = starts ? __ldcg(a.slot_a + (int64_t)u0 * RP * RP + e)
                                      : __ldcg(a.slot_b + (int64_t)u0 * RP * RP + e);
                    for (int u = u0 + 1; u < u0 + ncta; ++u) s += __ldcg(a.slot_a + (int64_t)u * RP * RP + e);
                    a.g[rr * RP * RP + e] = s;
                }
            }
        }
    };

    int64_t pos = ca;
    while (pos < cb) {
        while (pos >= row_end) {  // advance to the row holding `pos` (skip empty rows)
            finish_row(row);
            do {
                ++row;
                row_end = a.row_ptr[row + 1];
            } while (row_end <= pos);
        }
        const int cnt = (int)min((int64_t)GB, min(cb, row_end) - pos);
        __syncthreads();  // previous batch consumed
        for (int e = tid; e < GB * RP; e += GT) {
            const int t = e / RP, j = e % RP;
            double z = 0.0;
            if (t < cnt) {
                const int64_t l = pos + t;
                z = a.fac[a.fac_off[0] + (int64_t)__ldg(a.idx + l) * RP + j];
#pragma unroll
                for (int m = 1; m < DO; ++m) z *= a.fac[a.fac_off[m] + (int64_t)__ldg(a.idx + (int64_t)m * a.q + l) * RP + j];
            }
            zs[t][j] = z;
            if (j == 0) ws[t] = (a.mult && t < cnt) ? (double)__ldg(a.mult + pos + t) : 1.0;
        }
        __syncthreads();
        if (act) {
            for (int t = 0; t < cnt; ++t) {
                double za[BLK], zb[BLK];
#pragma unroll
                const double w = ws[t];
#pragma unroll
                for (int x = 0; x < BLK; ++x) {
                    za[x] = zs[t][ba + x] * w;
                    zb[x] = zs[t][bb + x];
                }
#pragma unroll
                for (int x = 0; x < BLK; ++x)
#pragma unroll
                    for (int y = 0; y < BLK; ++y) acc[x][y] = fma(za[x], zb[y], acc[x][y]);
            }
        }
        pos += cnt;
    }
    __syncthreads();
    finish_row(row);
}

// ---- DMMA build: G_i += (W Z)' Z per batch of GB observations ------------------------------
// The batch's Khatri-Rao rows Z (GB x RP, one row of i_k) are gathered into shared memory (the
// other-mode factors staged there when they fit), then G's upper-triangle 8x8 tiles accumulate
// DMMA m8n8k4 products over the batch (k = observations): nt(nt+1)/2 tiles (nt = RP/8) spread
// over the 8 warps, A fragments pre-weighted by the entry weights.  Row boundaries flush the
// tiles (and their mirror) exactly like the FMA build; same split-row protocol, deterministic.
// (FMA build: 85 ms at config 3 — shared-memory operand traffic, one LDS per FMA.)
__device__ __forceinline__ void dmma_g(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}
template <int RP, int DO, bool SF>
__global__ void __launch_bounds__(GT) gram_build_dmma_kernel(const GramArgs a) {
    constexpr int NT = RP / 8;                  // 8x8 tiles per dimension
    constexpr int NUP = NT * (NT + 1) / 2;      // upper-triangle tiles
    constexpr int NW = GT / 32;
    constexpr int TPW = (NUP + NW - 1) / NW;    // tiles per warp
    constexpr int ZP = RP + 4;                  // z row pitch: == 4 mod 16 doubles, conflict-free fragments
    extern __shared__ __align__(16) double gsm[];
    double* zs = gsm;                           // GB x ZP
    double* zw = zs + GB * ZP;                  // GB x ZP (weighted)
    double* sfac = zw + GB * ZP;                // staged factors (SF)
    __shared__ int sidx[DO][GB];
    __shared__ double sw[GB];
    __shared__ int s_last;
    const int c = blockIdx.x;
    const int64_t ca = a.cta_beg[c], cb = a.cta_beg[c + 1];
    if (ca >= cb) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, kq = lane & 3;
    if constexpr (SF) {
        for (int64_t e = tid; e < a.fac_total; e += GT) sfac[e] = a.fac[e];
    }
    const double* fac = SF ? sfac : a.fac;
    // this warp's tiles (ti <= tj), in a fixed enumeration
    int tiles_i[TPW], tiles_j[TPW];
#pragma unroll
    for (int u = 0; u < TPW; ++u) {
        int t = warp + NW * u, ti = 0;
        tiles_i[u] = -1;
        tiles_j[u] = -1;
        if (t < NUP) {
            while (t >= NT - ti) {
                t -= NT - ti;
                ++ti;
            }
            tiles_i[u] = ti;
            tiles_j[u] = ti + t;
        }
    }
    double acc[TPW][2];
#pragma unroll
    for (int u = 0; u < TPW; ++u) acc[u][0] = acc[u][1] = 0.0;
    const int64_t first_row = a.cta_rows[2 * c];
    int64_t row = first_row;
    int64_t row_end = a.row_ptr[row + 1];
    auto finish_row = [&](int64_t rr) {
        const int ncta = a.row_ncta[rr];
        double* dst = ncta == 1 ? a.g + rr * RP * RP
                    : rr == first_row ? a.slot_a + (int64_t)c * RP * RP
                                      : a.slot_b + (int64_t)c * RP * RP;
#pragma unroll
        for (int u = 0; u < TPW; ++u) {
            if (tiles_i[u] < 0) continue;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int ii = tiles_i[u] * 8 + g, jj = tiles_j[u] * 8 + 2 * kq + h;
                dst[ii * RP + jj] = acc[u][h];
                if (tiles_i[u] != tiles_j[u]) dst[jj * RP + ii] = acc[u][h];
            }
            acc[u][0] = acc[u][1] = 0.0;
        }
        if (ncta > 1) {  // the last CTA of a split row sums the slots in CTA order
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                s_last = atom_add_acqrel_g(a.rowcnt + rr, 1u) == (unsigned)ncta - 1;
                if (s_last) a.rowcnt[rr] = 0;
            }
            __syncthreads();
            if (s_last) {
                const int u0 = a.row_first_cta[rr];
                const bool starts = a.row_ptr[rr] == a.cta_beg[u0];
                for (int e = tid; e < RP * RP; e += GT) {
                    double sv = starts ? __ldcg(a.slot_a + (int64_t)u0 * RP * RP + e)
                                       : __ldcg(a.slot_b + (int64_t)u0 * RP * RP + e);
                    for (int u = u0 + 1; u < u0 + ncta; ++u) sv += __ldcg(a.slot_a + (int64_t)u * RP * RP + e);
                    a.g[rr * RP * RP + e] = sv;
                }
            }
        }
    };
    __syncthreads();  // staged factors
    int64_t pos = ca;
    while (pos < cb) {
        while (pos >= row_end) {
            finish_row(row);
            do {
                ++row;
                row_end = a.row_ptr[row + 1];
            } while (row_end <= pos);
        }
        const int cnt = (int)min((int64_t)GB, min(cb, row_end) - pos);
        __syncthreads();  // previous batch consumed (zs, zw, sidx, sw)
        for (int e = tid; e < GB * (DO + 1); e += GT) {  // the batch's indices and weights, once
            const int t = e % GB, m = e / GB;
            if (m < DO) sidx[m][t] = t < cnt ? __ldg(a.idx + (int64_t)m * a.q + pos + t) : 0;
            else sw[t] = t < cnt ? (a.mult ? (double)__ldg(a.mult + pos + t) : 1.0) : 0.0;
        }
        __syncthreads();
        {
            // all of the thread's factor loads in flight before the first use
            constexpr int IT = (GB * RP + GT - 1) / GT;
            double zr[IT][DO];
#pragma unroll
            for (int k = 0; k < IT; ++k) {
                const int e = tid + k * GT;
                const int t = min(e / RP, GB - 1), j = e % RP;
#pragma unroll
                for (int m = 0; m < DO; ++m) zr[k][m] = fac[a.fac_off[m] + (int64_t)sidx[m][t] * RP + j];
            }
#pragma unroll
            for (int k = 0; k < IT; ++k) {
                const int e = tid + k * GT;
                if (e < GB * RP) {
                    const int t = e / RP, j = e % RP;
                    double z = zr[k][0];
#pragma unroll
                    for (int m = 1; m < DO; ++m) z *= zr[k][m];
                    if (t >= cnt) z = 0.0;
                    zs[t * ZP + j] = z;
                    zw[t * ZP + j] = z * sw[t];
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int k0 = 0; k0 < GB; k0 += 4) {
            const int t = k0 + kq;
#pragma unroll
            for (int u = 0; u < TPW; ++u) {
                if (tiles_i[u] < 0) continue;
                const double av = zw[t * ZP + tiles_i[u] * 8 + g];   // A(i, t) = w_t z_t(i)
                const double bv = zs[t * ZP + tiles_j[u] * 8 + g];   // B(t, j) = z_t(j)
                dmma_g(acc[u], av, bv);
            }
        }
        pos += cnt;
    }
    __syncthreads();
    finish_row(row);
}

// ---- DMMA build v2: 2x2 register blocks of 8x8 tiles -------------------------------------------
// v1 loads one A and one B fragment (two 64-bit LDS, four shared-memory wavefronts) per DMMA,
// which caps it near half the FP64 tensor rate.  Here a warp owns a 2 x 2 block of tiles of the
// upper triangle (blocks bi <= bj; the lower tile of a diagonal block is computed and dropped) and
// reuses each fragment twice: 4 LDS per 4 DMMA.  RP = 64: 10 blocks = 10 warps; RP = 32 / 16:
// 3 / 1 blocks x KS warps splitting the batch's k-steps, whose partial tiles are summed in ks order
// at row flush (deterministic).  The batch's indices are staged once in shared memory and the
// Khatri-Rao rows built two columns per thread (16-byte factor loads).
template <int RP>
struct Gv2 {
    static constexpr int NT = RP / 8, NB = NT / 2, NBLK = NB * (NB + 1) / 2;
    static constexpr int KS = RP >= 64 ? 1 : (RP >= 32 ? 4 : 8);
    static constexpr int NWARP = NBLK * KS, T = 32 * NWARP;
    static constexpr int ZP = RP + 4;
};
template <int RP, int DO, bool SF>
__global__ void __launch_bounds__(Gv2<RP>::T, 2) gram_build_dmma2_kernel(const GramArgs a) {
    using V = Gv2<RP>;
    constexpr int ZP = V::ZP, KS = V::KS, T = V::T, NB = V::NB;
    extern __shared__ __align__(16) double gsm[];
    double* zs = gsm;                           // GB x ZP
    double* zw = zs + GB * ZP;                  // GB x ZP (weighted)
    double* red = zw + GB * ZP;                 // KS > 1: KS x RP x RP partial tiles at flush
    double* sfac = red + (KS > 1 ? KS * RP * RP : 0);  // staged factors (SF)
    __shared__ int sidx[DO][GB];
    __shared__ double sw[GB];
    __shared__ int s_last;
    const int c = blockIdx.x;
    const int64_t ca = a.cta_beg[c], cb = a.cta_beg[c + 1];
    if (ca >= cb) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, kq = lane & 3;
    // SF: the factors of modes 1.. staged in shared memory (mode 0 — the first other mode, constant
    // along the plan's runs — is read through L1)
    if constexpr (SF) {
        for (int64_t e = tid; e < a.fac_total - a.fac_off[1]; e += T) sfac[e] = a.fac[a.fac_off[1] + e];
    }
    auto fac_m = [&](int m) -> const double* {
        return SF ? sfac + (a.fac_off[m] - a.fac_off[1]) : a.fac + a.fac_off[m];
    };
    const int blk = warp / KS, ks = warp % KS;
    int bi = 0, bj = 0;
    {
        int t = blk;
        while (t >= NB - bi) {
            t -= NB - bi;
            ++bi;
        }
        bj = bi + t;
    }
    double acc[2][2][2];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 2; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
    const int64_t first_row = a.cta_rows[2 * c];
    int64_t row = first_row;
    int64_t row_end = a.row_ptr[row + 1];
    auto finish_row = [&](int64_t rr) {
        const int ncta = a.row_ncta[rr];
        double* dst = ncta == 1 ? a.g + rr * RP * RP
                    : rr == first_row ? a.slot_a + (int64_t)c * RP * RP
                                      : a.slot_b + (int64_t)c * RP * RP;
        if constexpr (KS == 1) {
#pragma unroll
            for (int x = 0; x < 2; ++x)
#pragma unroll
                for (int y = 0; y < 2; ++y) {
                    const int ti = 2 * bi + x, tj = 2 * bj + y;
                    if (ti <= tj) {
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int ii = ti * 8 + g, jj = tj * 8 + 2 * kq + h;
                            dst[ii * RP + jj] = acc[x][y][h];
                            if (ti != tj) dst[jj * RP + ii] = acc[x][y][h];
                        }
                    }
                }
        } else {
            __syncthreads();
#pragma unroll
            for (int x = 0; x < 2; ++x)
#pragma unroll
                for (int y = 0; y < 2; ++y)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int ii = (2 * bi + x) * 8 + g, jj = (2 * bj + y) * 8 + 2 * kq + h;
                        red[(ks * RP + ii) * RP + jj] = acc[x][y][h];
                    }
            __syncthreads();
            for (int e = tid; e < RP * RP; e += T) {  // upper triangle: sum the k-splits in order
                const int ii = e / RP, jj = e % RP;
                if (ii / 8 > jj / 8) continue;
                double sv = 0.0;
#pragma unroll
                for (int k2 = 0; k2 < KS; ++k2) sv += red[(k2 * RP + ii) * RP + jj];
                if (ii / 8 < jj / 8 || ii <= jj) {
                    dst[ii * RP + jj] = sv;
                    dst[jj * RP + ii] = sv;
                }
            }
        }
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
            for (int y = 0; y < 2; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
        if (ncta > 1) {  // the last CTA of a split row sums the slots in CTA order
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                s_last = atom_add_acqrel_g(a.rowcnt + rr, 1u) == (unsigned)ncta - 1;
                if (s_last) a.rowcnt[rr] = 0;
            }
            __syncthreads();
            if (s_last) {
                const int u0 = a.row_first_cta[rr];
                const bool starts = a.row_ptr[rr] == a.cta_beg[u0];
                for (int e = tid; e < RP * RP; e += T) {
                    double sv = starts ? __ldcg(a.slot_a + (int64_t)u0 * RP * RP + e)
                                       : __ldcg(a.slot_b + (int64_t)u0 * RP * RP + e);
                    for (int u = u0 + 1; u < u0 + ncta; ++u) sv += __ldcg(a.slot_a + (int64_t)u * RP * RP + e);
                    a.g[rr * RP * RP + e] = sv;
                }
            }
        }
    };
    __syncthreads();  // staged factors
    int64_t pos = ca;
    while (pos < cb) {
        while (pos >= row_end) {
            finish_row(row);
            do {
                ++row;
                row_end = a.row_ptr[row + 1];
            } while (row_end <= pos);
        }
        const int cnt = (int)min((int64_t)GB, min(cb, row_end) - pos);
        __syncthreads();  // previous batch consumed (zs, zw, sidx, sw)
        for (int e = tid; e < GB * (DO + 1); e += T) {
            const int t = e % GB, m = e / GB;
            if (m < DO) sidx[m][t] = t < cnt ? __ldg(a.idx + (int64_t)m * a.q + pos + t) : 0;
            else sw[t] = t < cnt ? (a.mult ? (double)__ldg(a.mult + pos + t) : 1.0) : 0.0;
        }
        __syncthreads();
        {
            // all of the thread's factor loads in flight before the first use (the loop over
            // elements with interleaved shared-memory stores serialised them on L2 latency)
            constexpr int IT = (GB * RP / 2 + T - 1) / T;
            double2 zr[IT], fr[IT][DO > 1 ? DO - 1 : 1];
#pragma unroll
            for (int k = 0; k < IT; ++k) {
                const int e = tid + k * T;
                const int t = min(e / (RP / 2), GB - 1), j = 2 * (e % (RP / 2));
                zr[k] = __ldg(reinterpret_cast<const double2*>(a.fac + a.fac_off[0] + (int64_t)sidx[0][t] * RP + j));
#pragma unroll
                for (int m = 1; m < DO; ++m)
                    fr[k][m - 1] = *reinterpret_cast<const double2*>(fac_m(m) + (int64_t)sidx[m][t] * RP + j);
            }
#pragma unroll
            for (int k = 0; k < IT; ++k) {
                const int e = tid + k * T;
                if (e < GB * RP / 2) {
                    const int t = e / (RP / 2), j = 2 * (e % (RP / 2));
                    double2 z = zr[k];
#pragma unroll
                    for (int m = 1; m < DO; ++m) {
                        z.x *= fr[k][m - 1].x;
                        z.y *= fr[k][m - 1].y;
                    }
                    const double w = sw[t];  // 0 beyond cnt: padded observations contribute exactly zero
                    if (t >= cnt) z.x = z.y = 0.0;
                    *reinterpret_cast<double2*>(zs + t * ZP + j) = z;
                    *reinterpret_cast<double2*>(zw + t * ZP + j) = make_double2(z.x * w, z.y * w);
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int k0 = 4 * ks; k0 < GB; k0 += 4 * KS) {
            const int t = k0 + kq;
            double av[2], bv[2];
#pragma unroll
            for (int x = 0; x < 2; ++x) av[x] = zw[t * ZP + (2 * bi + x) * 8 + g];  // A(i, t) = w_t z_t(i)
#pragma unroll
            for (int y = 0; y < 2; ++y) bv[y] = zs[t * ZP + (2 * bj + y) * 8 + g];  // B(t, j) = z_t(j)
#pragma unroll
            for (int x = 0; x < 2; ++x)
#pragma unroll
                for (int y = 0; y < 2; ++y) dmma_g(acc[x][y], av[x], bv[y]);
        }
        pos += cnt;
    }
    __syncthreads();
    finish_row(row);
}

// Yhat(i, a) = sum_b G_i(b, a) Xhat(i, b) for rows with observations (others stay zero).
// The b loop is unrolled at compile-time RP so every thread has its G column loads in flight at
// once (the runtime-bound loop issued one dependent load per FMA: latency-bound at ~57 % of HBM).
template <int RP>
__global__ void gram_apply_kernel(const double* __restrict__ g, const double* __restrict__ xhat, const int64_t* row_ptr,
                                  int64_t n, double* __restrict__ yhat) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n * RP) return;
    const int64_t i = e / RP;
    const int aa = (int)(e % RP);
    if (row_ptr[i + 1] == row_ptr[i]) return;
    const double* gi = g + i * RP * RP + aa;
    const double* xi = xhat + i * RP;
    constexpr int U = RP < 16 ? RP : 16;
    double s = 0.0;
#pragma unroll
    for (int b0 = 0; b0 < RP; b0 += U) {
        double gv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) gv[u] = __ldcs(gi + (b0 + u) * RP);  // streamed once per apply
#pragma unroll
        for (int u = 0; u < U; ++u) s = fma(gv[u], xi[b0 + u], s);
    }
    yhat[e] = s;
}

// grid == -1: partition-density query (CTAs per SM for the kernel gram_build would launch,
// from its occupancy), answered through g_occ instead of launching
thread_local int g_occ = 0;
template <class K>
bool occ_query(K kern, int grid, int threads, size_t smem) {
    if (grid != -1) return false;
    CPHIFI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_occ, kern, threads, smem));
    return true;
}

template <int RP, int DO>
void launch_dmma_do(const GramArgs& a, int grid, cudaStream_t s) {
    const size_t zbytes = sizeof(double) * 2 * GB * (RP + 4);
    size_t sf_cap = 200 * 1024;  // factors staged in shared memory below this (CPHIFI_GRAM_SF_KB)
    if (const char* e = std::getenv("CPHIFI_GRAM_SF_KB")) sf_cap = (size_t)std::atoi(e) * 1024;
    const bool sf = zbytes + sizeof(double) * a.fac_total <= sf_cap;
    const size_t smem = zbytes + (sf ? sizeof(double) * a.fac_total : 0);
    auto kern = sf ? gram_build_dmma_kernel<RP, DO, true> : gram_build_dmma_kernel<RP, DO, false>;
    CPHIFI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (occ_query(kern, grid, GT, smem)) {
        g_occ *= 2;  // v1: two waves' worth of CTAs — the finer row partition balanced better (config 3
        return;      // 27.4 -> 24.7 ms), while v2's one wave avoids a partial second wave (config 4)
    }
    kern<<<grid, GT, smem, s>>>(a);
}

template <int RP, int DO>
void launch_dmma2_do(const GramArgs& a, int grid, cudaStream_t s) {
    using V = Gv2<RP>;
    const size_t zbytes = sizeof(double) * (2 * GB * V::ZP + (V::KS > 1 ? V::KS * RP * RP : 0));
    size_t sf_cap = 100 * 1024;  // staging only while two CTAs still fit an SM (one CTA per SM: no
                                 // gather / DMMA overlap, measured 1.6x slower at config 3)
    if (const char* e = std::getenv("CPHIFI_GRAM_SF_KB")) sf_cap = (size_t)std::atoi(e) * 1024;
    const int64_t staged = DO > 1 ? a.fac_total - a.fac_off[1] : 0;  // modes 1.. (v2 stages no mode 0)
    const bool sf = DO > 1 && zbytes + sizeof(double) * staged <= sf_cap;
    const size_t smem = zbytes + (sf ? sizeof(double) * staged : 0);
    auto kern = sf ? gram_build_dmma2_kernel<RP, DO, true> : gram_build_dmma2_kernel<RP, DO, false>;
    CPHIFI_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (occ_query(kern, grid, V::T, smem)) return;
    kern<<<grid, V::T, smem, s>>>(a);
}

template <int RP>
void launch_build_rp(const GramArgs& a, int grid, cudaStream_t s) {
    if constexpr (RP >= 16) {
        // default for RP = 64 only: measured 82.8 -> 68.5 ms at config 4 (RP 64), 33.7 -> 35.4 ms
        // at config 3 (RP 32, three gathered modes: v1 keeps more CTAs per SM); CPHIFI_GRAM_V2=1
        // forces it for RP 16 / 32
        bool v2 = RP >= 64 && reinterpret_cast<uintptr_t>(a.fac) % 16 == 0;  // 16-byte factor-row loads
        if (const char* e = std::getenv("CPHIFI_GRAM_V2"))
            if (std::atoi(e) != 0) v2 = reinterpret_cast<uintptr_t>(a.fac) % 16 == 0;
        for (int m = 0; m < a.dother; ++m) v2 = v2 && a.fac_off[m] % 2 == 0;
        if (const char* e = std::getenv("CPHIFI_GRAM_V2")) v2 = v2 && std::atoi(e) != 0;
        if (v2) {
            switch (a.dother) {
                case 1: launch_dmma2_do<RP, 1>(a, grid, s); return;
                case 2: launch_dmma2_do<RP, 2>(a, grid, s); return;
                case 3: launch_dmma2_do<RP, 3>(a, grid, s); return;
                case 4: launch_dmma2_do<RP, 4>(a, grid, s); return;
                case 5: launch_dmma2_do<RP, 5>(a, grid, s); return;
                default: throw_invalid("unaligned: tensor order above 6 is not supported");
            }
        }
    }
    bool dm = RP >= 8;
    if (const char* e = std::getenv("CPHIFI_GRAM_DMMA")) dm = dm && std::atoi(e) != 0;
    if constexpr (RP >= 8) {
        if (dm) {
            switch (a.dother) {
                case 1: launch_dmma_do<RP, 1>(a, grid, s); return;
                case 2: launch_dmma_do<RP, 2>(a, grid, s); return;
                case 3: launch_dmma_do<RP, 3>(a, grid, s); return;
                case 4: launch_dmma_do<RP, 4>(a, grid, s); return;
                case 5: launch_dmma_do<RP, 5>(a, grid, s); return;
                default: throw_invalid("unaligned: tensor order above 6 is not supported");
            }
        }
    }
    if (grid == -1) {  // FMA build: the query reports the default partition density
        g_occ = 4;
        return;
    }
    switch (a.dother) {
        case 1: gram_build_kernel<RP, 1><<<grid, GT, 0, s>>>(a); break;
        case 2: gram_build_kernel<RP, 2><<<grid, GT, 0, s>>>(a); break;
        case 3: gram_build_kernel<RP, 3><<<grid, GT, 0, s>>>(a); break;
        case 4: gram_build_kernel<RP, 4><<<grid, GT, 0, s>>>(a); break;
        case 5: gram_build_kernel<RP, 5><<<grid, GT, 0, s>>>(a); break;
        default: throw_invalid("unaligned: tensor order above 6 is not supported");
    }
}

}  // namespace

int gram_build_occupancy(const GramArgs& a) {
    g_occ = 0;
    switch (a.rp) {
        case 4: launch_build_rp<4>(a, -1, nullptr); break;
        case 8: launch_build_rp<8>(a, -1, nullptr); break;
        case 16: launch_build_rp<16>(a, -1, nullptr); break;
        case 32: launch_build_rp<32>(a, -1, nullptr); break;
        case 64: launch_build_rp<64>(a, -1, nullptr); break;
        default: throw_invalid("gram operator: padded rank above 64 is not supported");
    }
    return std::max(g_occ, 1);
}

void gram_build(const GramArgs& a, int grid, cudaStream_t s) {
    switch (a.rp) {
        case 4: launch_build_rp<4>(a, grid, s); break;
        case 8: launch_build_rp<8>(a, grid, s); break;
        case 16: launch_build_rp<16>(a, grid, s); break;
        case 32: launch_build_rp<32>(a, grid, s); break;
        case 64: launch_build_rp<64>(a, grid, s); break;
        default: throw_invalid("gram operator: padded rank above 64 is not supported");
    }
    CPHIFI_CHECK_LAUNCH();
}

void gram_apply(const double* g, const double* xhat_rm, const int64_t* row_ptr, int64_t n, int64_t rp, double* yhat_rm,
                cudaStream_t s) {
    const unsigned grid = (unsigned)((n * rp + 255) / 256);
    switch (rp) {
        case 4: gram_apply_kernel<4><<<grid, 256, 0, s>>>(g, xhat_rm, row_ptr, n, yhat_rm); break;
        case 8: gram_apply_kernel<8><<<grid, 256, 0, s>>>(g, xhat_rm, row_ptr, n, yhat_rm); break;
        case 16: gram_apply_kernel<16><<<grid, 256, 0, s>>>(g, xhat_rm, row_ptr, n, yhat_rm); break;
        case 32: gram_apply_kernel<32><<<grid, 256, 0, s>>>(g, xhat_rm, row_ptr, n, yhat_rm); break;
        case 64: gram_apply_kernel<64><<<grid, 256, 0, s>>>(g, xhat_rm, row_ptr, n, yhat_rm); break;
        case 128: gram_apply_kernel<128><<<grid, 256, 0, s>>>(g, xhat_rm, row_ptr, n, yhat_rm); break;
        default: throw_invalid("gram_apply: padded rank must be a power of two in [4, 128]");
    }
    CPHIFI_CHECK_LAUNCH();
}

}  // namespace cphifi
