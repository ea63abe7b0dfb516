// k_fused.cu — the unaligned operator as ONE persistent cooperative kernel (sm_100a).
//
//   y = vec(K Yhat + lambda Xhat) + rho x,  Xhat = K X,
//   Yhat(i,:) = sum_{l: i_k(l)=i} (Xhat(i,:) . z_l) z_l,  z_l = prod_{m!=k} A_m(i_m(l),:)
// (unaligned.hpp:101-115 with gather_rows + sampled_mttkrp, observations.hpp:174-198, fused;
// Zhat is never materialised).
//
// Phases (small n, one GPU: a single launch with ONE grid barrier):
//   AL  Xhat rows     each CTA computes the (<= MAXLOC) rows its own observations touch, from
//                     X and K columns prefetched into shared memory at entry
//   (A  fallback      rows distributed over CTAs + a grid barrier)
//   B   scatter-gather CTA c streams observations [beg[c], beg[c+1]) of the i_k-sorted set (a
//                     host-planned ROW-ALIGNED partition: whole rows packed per CTA, only rows
//                     longer than the target load split across CTAs)
//                     in ROUNDS of NG consecutive observations, one per lane group (G lanes x
//                     VPL doubles = the padded rank), four rounds in flight per group.  Each
//                     group keeps its row accumulator in registers; at a row boundary the CTA
//                     reduces the groups in group order (fixed tree) and writes the row:
//                     directly to Yhat if the row is interior to the CTA; otherwise to the CTA's
//                     slot (A = first row, B = last row), and the LAST CTA to finish a split row
//                     (per-row arrival counter) sums its slots in CTA order into Yhat.
//   --  grid barrier
//   C2  y rows        y = K Yhat + lambda Xhat + rho x for rows [c n / C, (c+1) n / C)
// Every reduction has a fixed order, so results are bit-reproducible for a launch shape.
// Large n: the DMMA GEMM kernels compute Xhat and y; this kernel runs phase B only.
//
// Memory pipeline: the observation stream (int32 index columns, fp64 weights) is staged in
// shared memory tile by tile with cp.async (tiles 0 and 1 issued at kernel entry, so their HBM
// latency hides behind phase AL); packed factor rows are staged in shared memory when they fit
// (SURVEY §7 hard part 4), so the round loop runs from shared memory.
#include "kernels.cuh"
#include "lanegroup.cuh"
#include "tma.cuh"

namespace cphifi {
namespace {

constexpr int FT = 512;    // threads per CTA
constexpr int TILE = 1024; // observations per staged tile
constexpr int MAXLOC = 4;  // PH_AL: max rows one CTA computes Xhat for
constexpr int MAX_SMEM = 226 * 1024;  // dynamic shared memory cap (227 KB opt-in minus static)
constexpr int UNR = 4;     // observations in flight per lane group in the fast path

__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Software grid barrier (all CTAs co-resident: cooperative launch) on ONE 64-bit counter that
// is never reset: a CTA arrives with a relaxed add after a gpu-scope fence (cumulative over the
// CTA's writes, ordered by bar.sync) and waits until the counter reaches the next multiple of the
// grid size.  Two L2 round trips on the critical path (the arrival and the observing load); the
// former two-level counter tree + generation word took ~3 us from the last arrival to release.
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void grid_barrier(unsigned* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long* ctr = reinterpret_cast<unsigned long long*>(bar);
        const unsigned long long C = gridDim.x;
        __threadfence();
        const unsigned long long old = atomicAdd(ctr, 1ull);
        const unsigned long long target = old - old % C + C;
        while (ld_acquire_u64(ctr) < target) {
        }
    }
    __syncthreads();
}

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void stamp(const FusedArgs& a, int slot) {
    if (a.trace && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[(size_t)blockIdx.x * TRACE_SLOTS + slot] = t;
    }
}

template <int VPL>
__device__ __forceinline__ void ldv(double (&v)[VPL], const double* p) {
    if constexpr (VPL == 1) {
        v[0] = p[0];
    } else {
#pragma unroll
        for (int u = 0; u < VPL; u += 2) {
            const double2 t = *reinterpret_cast<const double2*>(p + u);
            v[u] = t.x;
            v[u + 1] = t.y;
        }
    }
}

// out[j] = sum_k kc[k] * V(k, j), j < r, for one row (kc = the row's K column, length n).
// thread t -> column j = t % RP, k-slice s = t / RP: consecutive lanes read consecutive
// columns, so a warp load of a row-major V covers contiguous row segments; kc[k] is a
// broadcast.  Loads go out in predicated batches of 8 (V may live in L2).  Lanes sharing j are
// combined by xor shuffles, then the per-warp (or per-slice) partials in a fixed order.
template <int RP>
__device__ __forceinline__ void row_dot(const FusedArgs& a, const double* __restrict__ kc, const double* __restrict__ v,
                                        int64_t vs_r, int64_t vs_c, double* red, double* out) {
    constexpr int S = FT / RP;
    const int j = threadIdx.x % RP, s = threadIdx.x / RP;
    double t = 0.0;
    if (j < a.r) {
        const double* vj = v + j * vs_c;
        for (int64_t k0 = s; k0 < a.n; k0 += 8 * S) {
            double kv[8], vv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t k = k0 + (int64_t)u * S;
                const bool ok = k < a.n;
                kv[u] = ok ? kc[k] : 0.0;
                vv[u] = ok ? vj[k * vs_r] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) t = fma(kv[u], vv[u], t);
        }
    }
    if constexpr (RP < 32) {
#pragma unroll
        for (int off = 16; off >= RP; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    }
    constexpr int PW = RP < 32 ? FT / 32 : S;  // partials per column
    const int pidx = RP < 32 ? (int)(threadIdx.x >> 5) : s;
    if (RP >= 32 || (threadIdx.x & 31) < RP) red[pidx * RP + j] = t;
    __syncthreads();
    if (threadIdx.x < RP) {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < PW; ++q) acc += red[q * RP + threadIdx.x];
        out[threadIdx.x] = threadIdx.x < a.r ? acc : 0.0;
    }
    __syncthreads();
}

template <int RP, int DO, bool SMEMF>
__global__ void __launch_bounds__(FT, 2) fused_matvec_kernel(const FusedArgs a) {
    // 2 doubles per lane: one LDS.128 per factor row, and every 8-lane phase of the warp reads
    // one contiguous 128-byte row segment -> conflict-free gathers (the loop is bound by
    // shared-memory wavefronts, SURVEY §7 hard part 4)
    constexpr int VPL = (RP >= 8 && RP <= 64) ? 2 : 4;  // G = RP / VPL <= 32 lanes
    constexpr int G = RP / VPL;           // lanes per observation: few shuffle steps per dot
    constexpr int NG = FT / G;            // observations per round
    constexpr int NW = FT / 32;
    extern __shared__ __align__(16) double smem[];
    double* red = smem;                   // RP x (NG + 1) doubles (transposed group partials)
    double* red2 = red + FT * VPL + RP;   // FT doubles
    double* rowbuf = red2 + FT;           // 2 * RP doubles
    double* xloc = rowbuf + 2 * RP;       // MAXLOC * RP: this CTA's Xhat rows (PH_AL)
    double* sw = xloc + MAXLOC * RP;      // 2 x TILE weights (RHS mode)
    int32_t* sidx = reinterpret_cast<int32_t*>(sw + 2 * TILE);       // 2 x DO x TILE
    double* sfac = reinterpret_cast<double*>(sidx + 2 * DO * TILE);   // staged factors (SMEMF)
    // X staged column-major with an odd column stride: the j-fastest lanes of row_dot and the
    // element-order staging writes both hit distinct banks
    const int64_t ldx = fused_ldx(a.n);
    double* xs = sfac + (SMEMF ? a.fac_total : 0);                   // X, ldx x r (prefetch)
    double* kcs = xs + (a.prefetch ? ldx * a.r : 0);                 // K columns (prefetch)
    __shared__ int64_t s_rows[2];
    __shared__ int s_last;
    __shared__ __align__(8) uint64_t s_fbar;  // plan-independent TMA prefetch (factors, X, C2 K columns)

    const int c = blockIdx.x, C = gridDim.x;
    const int64_t i0 = a.n * c / C, i1 = a.n * (c + 1) / C;  // this CTA's y rows (PH_C2)
    const double* kc2 = a.kmat_c2 ? a.kmat_c2 : a.kmat;      // PH_C2 columns (U in the eigenbasis)
    const bool pf = a.prefetch && a.x != nullptr && (a.phases & (PH_AL | PH_C2));
    // ---- entry, before any dependent load: one thread issues the bulk copies that need no plan
    // data (even n: 16-byte aligned columns), so their HBM latency overlaps the plan reads
    const bool tma_entry = (a.n % 2) == 0;
    const bool tma_fac = tma_entry && SMEMF && (a.phases & PH_B) && !a.gram;
    const bool tma_any = tma_fac || (tma_entry && pf);
    if (tma_any && threadIdx.x == 0) {
        tma::mbar_init(&s_fbar, 1);
        tma::fence_mbar_init();
        const unsigned colb = (unsigned)(a.n * 8);
        unsigned bytes = 0;
        if (tma_fac) bytes += (unsigned)(a.fac_total * 8);
        if (pf) bytes += colb * (unsigned)a.r;
        if (pf && (a.phases & PH_C2)) bytes += colb * (unsigned)(i1 - i0);
        tma::mbar_expect_tx(&s_fbar, bytes);
        if (tma_fac)
            for (int64_t b0 = 0; b0 < a.fac_total * 8; b0 += 32768)
                tma::bulk_g2s(reinterpret_cast<unsigned char*>(sfac) + b0, reinterpret_cast<const unsigned char*>(a.fac) + b0,
                              (unsigned)min((int64_t)32768, a.fac_total * 8 - b0), &s_fbar);
        if (pf) {
            for (int j = 0; j < (int)a.r; ++j) tma::bulk_g2s(xs + ldx * j, a.x + a.n * j, colb, &s_fbar);
            if (a.phases & PH_C2)
                for (int64_t i = i0; i < i1; ++i)
                    tma::bulk_g2s(kcs + (MAXLOC + i - i0) * a.n, kc2 + i * a.n, colb, &s_fbar);
        }
    }
    const int g = threadIdx.x / G, glane = threadIdx.x % G, jb = glane * VPL;
    const int lane = threadIdx.x & 31;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane - lane % G));
    const bool dot = a.weights == nullptr;
    const bool mult = dot && a.mult != nullptr;
    const int64_t ca = a.cta_beg[c], cb = a.cta_beg[c + 1];  // row-aligned partition (host plan)
    const bool has_obs = (a.phases & PH_B) && ca < cb;
    const int ntiles = has_obs && !a.gram ? (int)((cb - ca + TILE - 1) / TILE) : 0;

    auto issue_tile = [&](int t) {
        const int buf = t & 1;
        const int64_t t0 = ca + (int64_t)t * TILE;
        const int cnt = (int)min((int64_t)TILE, cb - t0);
#pragma unroll
        for (int m = 0; m < DO; ++m)
            for (int o = threadIdx.x; o < cnt; o += FT)
                cp_async4(sidx + (buf * DO + m) * TILE + o, a.idx + (int64_t)m * a.q + t0 + o);
        if (!dot)
            for (int o = threadIdx.x; o < cnt; o += FT) cp_async8(sw + buf * TILE + o, a.weights + t0 + o);
        else if (mult)  // the weight buffer is free in dot mode
            for (int o = threadIdx.x; o < cnt; o += FT)
                cp_async4(reinterpret_cast<int32_t*>(sw + buf * TILE) + o, a.mult + t0 + o);
    };

    stamp(a, 0);
    __shared__ unsigned s_c2_empty;  // bit t: y row i0 + t has no observation in this shard
    if (threadIdx.x < 32) {
        const bool e = (a.phases & PH_C2) && i0 + threadIdx.x < i1 &&
                       a.row_ptr[i0 + threadIdx.x + 1] == a.row_ptr[i0 + threadIdx.x];
        const unsigned m = __ballot_sync(0xffffffffu, e);
        if (threadIdx.x == 0) s_c2_empty = m;
    }
    if (has_obs && threadIdx.x == 0) {
        s_rows[0] = a.cta_rows[2 * c];
        s_rows[1] = a.cta_rows[2 * c + 1];
    }
    __syncthreads();
    const int64_t first_row = s_rows[0], last_row = s_rows[1];
    int dbg_n = 0;
    auto dbg_mark = [&](int ev) {  // debug timeline (thread 0): (event, clock64) pairs
        if (a.dbg && threadIdx.x == 0 && dbg_n < DBG_SLOTS / 2) {
            a.dbg[(size_t)blockIdx.x * DBG_SLOTS + 2 * dbg_n] = ev;
            a.dbg[(size_t)blockIdx.x * DBG_SLOTS + 2 * dbg_n + 1] = clock64();
            ++dbg_n;
        }
    };
    dbg_mark(0);
    const bool do_al = (a.phases & PH_AL) && has_obs && dot;
    const int nal = do_al ? (int)(last_row - first_row + 1) : 0;

    // ---- entry: async prefetch (group 0: factors, X, K columns, tile 0; group 1: tile 1) ----
    if (ntiles > 0 && !tma_fac) {
        if constexpr (SMEMF) {
            const double2* src = reinterpret_cast<const double2*>(a.fac);
            for (int64_t e = threadIdx.x; e < a.fac_total / 2; e += FT) cp_async16(sfac + 2 * e, src + e);
        }
    }
    if (pf) {
        if (!tma_entry) {
            const int nn = (int)a.n, nr = (int)(a.n * a.r), odd = (int)(ldx - a.n);  // small n: n * r <= 8192
            for (int e = threadIdx.x; e < nr; e += FT) cp_async8(xs + e + odd * (e / nn), a.x + e);
            if (a.phases & PH_C2)
                for (int64_t i = i0; i < i1; ++i)
                    for (int64_t k = threadIdx.x; k < a.n; k += FT)
                        cp_async8(kcs + (MAXLOC + i - i0) * a.n + k, kc2 + i * a.n + k);
        }
        for (int rr = 0; rr < nal; ++rr)
            for (int64_t k = threadIdx.x; k < a.n; k += FT) cp_async8(kcs + rr * a.n + k, a.kmat + (first_row + rr) * a.n + k);
    }
    if (ntiles > 0) issue_tile(0);
    cp_commit();
    if (ntiles > 1) {
        issue_tile(1);
        cp_commit();
    }
    const double* fac = SMEMF ? sfac : a.fac;
    dbg_mark(8);  // prefetch issued

    // ---- phase A: Xhat rows -----------------------------------------------------------------
    if (a.phases & PH_AL) {  // only the rows this CTA's observations touch, from shared memory
        if (ntiles > 1) cp_wait<1>();
        else cp_wait<0>();
        if (tma_any) tma::mbar_wait(&s_fbar, 0);
        __syncthreads();
        dbg_mark(9);  // prefetch landed
        for (int rr = 0; rr < nal; ++rr) {
            row_dot<RP>(a, kcs + rr * a.n, xs, 1, ldx, red, xloc + rr * RP);
            if (threadIdx.x < RP) a.xhat_rm[(first_row + rr) * RP + threadIdx.x] = xloc[rr * RP + threadIdx.x];
        }
        dbg_mark(10);
        stamp(a, 1);
    } else if (a.phases & PH_A) {  // rows distributed over CTAs, then a grid barrier
        for (int64_t i = i0; i < i1; ++i) {
            row_dot<RP>(a, a.kmat + i * a.n, a.x, 1, a.n, red, rowbuf);
            if (threadIdx.x < RP) a.xhat_rm[i * RP + threadIdx.x] = rowbuf[threadIdx.x];
        }
        stamp(a, 1);
        grid_barrier(a.barrier);
        stamp(a, 2);
    }
    const bool local_x = (a.phases & PH_AL) != 0;

    // ---- phase B (row-Gram form): Yhat(i,:) = G_i Xhat(i,:) for the rows this CTA owns -----
    if (has_obs && a.gram) {
        for (int64_t row = first_row; row <= last_row; ++row) {
            if (a.row_ptr[row + 1] == a.row_ptr[row] || a.row_first_cta[row] != c) continue;
            const double* xr = local_x ? xloc + (row - first_row) * RP : a.xhat_rm + row * RP;
            if (threadIdx.x < RP) {
                const double* gi = a.gram + row * RP * RP;
                double s = 0.0;
                for (int b = 0; b < RP; ++b) s = fma(gi[b * RP + threadIdx.x], xr[b], s);
                a.yhat_rm[row * RP + threadIdx.x] = s;
            }
        }
    }

    // ---- phase B: fused gather / scatter over this CTA's observations ---------------------
    if (ntiles > 0) {
        int64_t cur = first_row;
        int64_t cur_end = a.row_ptr[cur + 1];
        double xh[VPL], acc[VPL];
#pragma unroll
        for (int v = 0; v < VPL; ++v) acc[v] = 0.0;
        auto load_xh = [&]() {
            if (dot) ldv<VPL>(xh, local_x ? xloc + (cur - first_row) * RP + jb : a.xhat_rm + cur * RP + jb);
        };
        load_xh();

        // Row reduction over the NG groups in a FIXED order: group partials are stored
        // transposed (red[j][g]); warp w reduces columns j = w, w + NW, ...: each lane sums the
        // groups g = lane, lane + 32, ... in order, then a 5-step xor-shuffle tree.
        auto flush = [&](int64_t row) {
            __syncthreads();
#pragma unroll
            for (int v = 0; v < VPL; ++v) red[(jb + v) * (NG + 1) + g] = acc[v];
            __syncthreads();
            for (int j = threadIdx.x >> 5; j < RP; j += NW) {
                double s = 0.0;
                for (int q = lane; q < NG; q += 32) s += red[j * (NG + 1) + q];
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
                if (lane == 0) red2[j] = s;
            }
            __syncthreads();
            const int ncta = a.row_ncta[row];
            const bool split = ncta > 1;  // the row continues in other CTAs
            if (threadIdx.x < RP) {
                double* dst = !split ? a.yhat_rm + row * RP
                            : row == first_row ? a.slot_a + (int64_t)c * RP
                                               : a.slot_b + (int64_t)c * RP;
                dst[threadIdx.x] = red2[threadIdx.x];
            }
#pragma unroll
            for (int v = 0; v < VPL; ++v) acc[v] = 0.0;
            if (split) {  // the last of the row's CTAs to arrive sums the slots in CTA order
                __syncthreads();
                if (threadIdx.x == 0) {
                    __threadfence();
                    s_last = atom_add_acqrel(a.rowcnt + row, 1u) == (unsigned)ncta - 1;
                    if (s_last) a.rowcnt[row] = 0;  // ready for the next launch
                }
                __syncthreads();
                if (s_last && threadIdx.x < RP) {
                    const int j = threadIdx.x;
                    const int u0 = a.row_first_cta[row];
                    double s = a.row_ptr[row] == a.cta_beg[u0] ? __ldcg(a.slot_a + (int64_t)u0 * RP + j)
                                                               : __ldcg(a.slot_b + (int64_t)u0 * RP + j);
                    for (int u = u0 + 1; u < u0 + ncta; ++u) s += __ldcg(a.slot_a + (int64_t)u * RP + j);
                    a.yhat_rm[row * RP + j] = s;
                }
            }
        };

        for (int t = 0; t < ntiles; ++t) {
            if (t + 1 < ntiles) cp_wait<1>();
            else cp_wait<0>();
            if (t == 0 && tma_any) tma::mbar_wait(&s_fbar, 0);
            __syncthreads();
            if (t == 0) stamp(a, 2);
            dbg_mark(1);  // tile ready
            const int buf = t & 1;
            const int64_t t0 = ca + (int64_t)t * TILE;
            const int64_t t1 = min(cb, t0 + TILE);
            const int32_t* ti = sidx + buf * DO * TILE;
            const double* tw = sw + buf * TILE;
            const int32_t* tm = reinterpret_cast<const int32_t*>(tw);  // multiplicities (dot mode)
            // z = the Khatri-Rao row, modes ascending (observations.hpp:150-156)
            auto build_z = [&](int o, double (&z)[VPL]) {
                ldv<VPL>(z, fac + a.fac_off[0] + (int64_t)ti[o] * RP + jb);
#pragma unroll
                for (int m = 1; m < DO; ++m) {
                    double f[VPL];
                    ldv<VPL>(f, fac + a.fac_off[m] + (int64_t)ti[m * TILE + o] * RP + jb);
#pragma unroll
                    for (int v = 0; v < VPL; ++v) z[v] *= f[v];
                }
            };
            auto partial_dot = [&](const double (&z)[VPL]) {
                double p = 0.0;
#pragma unroll
                for (int v = 0; v < VPL; ++v) p = fma(xh[v], z[v], p);
                return p;
            };
            // Row segments: [seg, seg_end) lies in row `cur`; a tight strided loop with two
            // observations in flight per group and no per-round row bookkeeping.
            int64_t seg = t0;
            while (seg < t1) {
                const int64_t seg_end = min(t1, cur_end);
                const int o_end = (int)(seg_end - t0);
                int o = (int)(seg - t0) + g;
                // UNR observations per lane group per round, every group of the warp running the
                // warp's maximum round count (padding observations contribute exactly zero), so
                // the partial dots reduce with full-mask shuffles as one transposed butterfly
                // (lanegroup.cuh).  Accumulation order per group: o, o + NG, o + 2 NG, ...
                const int mine = o < o_end ? (o_end - o + NG - 1) / NG : 0;
                const int rounds = (int)__reduce_max_sync(0xffffffffu, (unsigned)((mine + UNR - 1) / UNR));
                for (int rd = 0; rd < rounds; ++rd, o += UNR * NG) {
                    double z[UNR][VPL], sv[UNR];
                    bool val[UNR];
#pragma unroll
                    for (int u = 0; u < UNR; ++u) {
                        val[u] = o + u * NG < o_end;
                        build_z(val[u] ? o + u * NG : o_end - 1, z[u]);
                    }
                    if (dot) {
#pragma unroll
                        for (int u = 0; u < UNR; ++u) sv[u] = partial_dot(z[u]);
                        group_reduce<UNR, G>(sv, lane);
                        if (mult) {  // coalesced plan: entry weight = multiplicity
#pragma unroll
                            for (int u = 0; u < UNR; ++u) sv[u] *= (double)tm[val[u] ? o + u * NG : o_end - 1];
                        }
                    } else {
#pragma unroll
                        for (int u = 0; u < UNR; ++u) sv[u] = tw[val[u] ? o + u * NG : o_end - 1];
                    }
#pragma unroll
                    for (int u = 0; u < UNR; ++u) {
                        if (val[u]) {
#pragma unroll
                            for (int v = 0; v < VPL; ++v) acc[v] = fma(sv[u], z[u][v], acc[v]);
                        }
                    }
                }
                seg = seg_end;
                dbg_mark(2);  // segment done
                if (seg_end == cur_end && seg_end < cb) {  // row complete, more rows follow
                    flush(cur);
                    dbg_mark(3);  // flush done
                    do {
                        ++cur;
                        cur_end = a.row_ptr[cur + 1];
                    } while (cur_end <= seg_end);
                    load_xh();
                }
            }
            __syncthreads();  // all groups are done with buffer t & 1
            if (t + 2 < ntiles) {
                issue_tile(t + 2);
                cp_commit();
            }
        }
        stamp(a, 3);
        flush(cur);
    }
    stamp(a, 4);

    // ---- phase C2: y = (K Yhat + lambda Xhat) + rho x  (small n) ------------------------------
    if (a.phases & PH_C2) {
        if (a.phases & PH_B) grid_barrier(a.barrier);
        stamp(a, 5);
        dbg_mark(4);
        cp_wait<0>();
        if (tma_any) tma::mbar_wait(&s_fbar, 0);
        __syncthreads();
        for (int64_t i = i0; i < i1; ++i) {
            const double* kc = pf ? kcs + (MAXLOC + i - i0) * a.n : kc2 + i * a.n;
            if (a.mu_rot) {  // eigenbasis: y~(i,:) = mu_i (U(:,i)' Yhat + lambda x~(i,:)) + rho x~(i,:)
                row_dot<RP>(a, kc, a.yhat_c2, RP, 1, red, rowbuf);
                if (threadIdx.x < a.r) {
                    const int64_t e = i + a.n * threadIdx.x;
                    const double xt = pf ? xs[i + ldx * threadIdx.x] : a.x[e];
                    a.y[e] = a.mu_rot[i] * (rowbuf[threadIdx.x] + a.lambda * xt) + a.rho * xt;
                }
                __syncthreads();
                continue;
            }
            // no observation on row i here -> no CTA produced Xhat(i,:): recompute it below
            const bool empty = local_x && (i - i0 < 32 ? ((s_c2_empty >> (i - i0)) & 1u) != 0
                                                       : a.row_ptr[i + 1] == a.row_ptr[i]);
            double xr = 0.0;  // issued before the Yhat dot so the two L2 round trips overlap
            if (!empty && threadIdx.x < RP) xr = __ldcg(a.xhat_rm + i * RP + threadIdx.x);
            dbg_mark(5);
            row_dot<RP>(a, kc, a.yhat_c2, RP, 1, red, rowbuf);
            dbg_mark(6);
            if (empty) {
                row_dot<RP>(a, kc, pf ? xs : a.x, 1, pf ? ldx : a.n, red, rowbuf + RP);
            } else {
                if (threadIdx.x < RP) rowbuf[RP + threadIdx.x] = xr;
                __syncthreads();
            }
            if (threadIdx.x < a.r) {
                const int64_t e = i + a.n * threadIdx.x;
                const double out = rowbuf[threadIdx.x] + a.lambda * rowbuf[RP + threadIdx.x];
                a.y[e] = out + a.rho * (pf ? xs[i + ldx * threadIdx.x] : a.x[e]);
            }
            __syncthreads();
        }
    } else {
        cp_wait<0>();
    }
    dbg_mark(7);
    stamp(a, 7);
}

template <int RP, int DO, bool SMEMF>
void launch_fused_t(const FusedArgs& a, int grid, size_t smem, cudaStream_t s) {
    auto kern = fused_matvec_kernel<RP, DO, SMEMF>;
    func_attr_once((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, MAX_SMEM);
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

template <int RP, int DO, bool SMEMF>
int occupancy_t(size_t smem) {
    int blocks = 0;
    CPHIFI_CUDA(cudaFuncSetAttribute(fused_matvec_kernel<RP, DO, SMEMF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     MAX_SMEM));
    CPHIFI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fused_matvec_kernel<RP, DO, SMEMF>, FT, smem));
    return blocks;
}

template <int RP, bool SMEMF>
int occupancy_do(int dother, size_t smem) {
    switch (dother) {
        case 1: return occupancy_t<RP, 1, SMEMF>(smem);
        case 2: return occupancy_t<RP, 2, SMEMF>(smem);
        case 3: return occupancy_t<RP, 3, SMEMF>(smem);
        case 4: return occupancy_t<RP, 4, SMEMF>(smem);
        default: return occupancy_t<RP, 5, SMEMF>(smem);
    }
}

template <int RP>
int occupancy_rp(int dother, bool smemf, size_t smem) {
    return smemf ? occupancy_do<RP, true>(dother, smem) : occupancy_do<RP, false>(dother, smem);
}

}  // namespace

size_t fused_smem_bytes(int64_t rp, int dother, int64_t fac_total, bool smemf, int64_t prefetch_elems) {
    const int64_t vpl = (rp >= 8 && rp <= 64) ? 2 : 4;  // must match fused_matvec_kernel
    return sizeof(double) * (FT * vpl + rp + FT + 2 * rp + MAXLOC * rp + 2 * TILE) + sizeof(int32_t) * 2 * dother * TILE +
           sizeof(double) * ((smemf ? fac_total : 0) + prefetch_elems);
}

int fused_maxloc() { return MAXLOC; }

int fused_grid(int64_t rp, int dother, bool smemf, size_t smem, int num_sms) {
    int occ = 0;
    switch (rp) {
        case 4: occ = occupancy_rp<4>(dother, smemf, smem); break;
        case 8: occ = occupancy_rp<8>(dother, smemf, smem); break;
        case 16: occ = occupancy_rp<16>(dother, smemf, smem); break;
        case 32: occ = occupancy_rp<32>(dother, smemf, smem); break;
        case 64: occ = occupancy_rp<64>(dother, smemf, smem); break;
        case 128: occ = occupancy_rp<128>(dother, smemf, smem); break;
        default: throw_invalid("unaligned: rank above 128 is not supported");
    }
    if (occ < 1) throw_runtime("fused matvec: kernel does not fit on an SM");
    int cap = 2;  // CTAs per SM (tunable for experiments: CPHIFI_FUSED_OCC)
    if (const char* e = std::getenv("CPHIFI_FUSED_OCC")) cap = std::max(1, std::atoi(e));
    return num_sms * std::min(occ, cap);
}

void fused_matvec(const FusedArgs& a, int grid, size_t smem, bool smemf, cudaStream_t s) {
#define RPCASE(RPV)                                                        \
    case RPV:                                                              \
        if (smemf) launch_fused_do<RPV, true>(a, grid, smem, s);           \
        else launch_fused_do<RPV, false>(a, grid, smem, s);                \
        break;
    switch (a.rp) {
        RPCASE(4) RPCASE(8) RPCASE(16) RPCASE(32) RPCASE(64) RPCASE(128)
        default: throw_invalid("unaligned: rank above 128 is not supported");
    }
#undef RPCASE
}

}  // namespace cphifi
