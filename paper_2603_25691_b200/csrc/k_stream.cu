// k_stream.cu — the unaligned scatter-gather for LARGE plans (sm_100a): one streaming pass over
// the observations with the first other mode hoisted out of the per-observation work.
//
// The reference computes, per operator application (observations.hpp:174-198 via
// unaligned.hpp:110-111, Zhat materialised by observations.hpp:142-158),
//     Yhat(i,:) = sum_{l: i_k(l)=i} (Xhat(i,:) . z_l) z_l,   z_l = A_1(a_l,:) o A_2(b_l,:) o ...
// The plan is in lexicographic order (i_k, a, b, ...) (capi.cu, obs_create), so observations of
// one row form RUNS of equal a.  Within a run (i, a) with p = Xhat(i,:) o A_1(a,:) and
// t_l = A_2(b_l,:) o ... (the remaining modes):
//     x_l = p . t_l,      Yhat(i,:) += A_1(a,:) o sum_{l in run} w_l x_l t_l
// (w_l = multiplicity of a coalesced entry; RHS mode: x_l w_l -> the observed value).  The
// per-observation work is then one (d-2)-row product, one dot and one axpy on rows that live in
// shared memory; A_1 rows are touched once per run.
//
// Schedule: CTA c streams observations [cta_beg[c], cta_beg[c+1]) of the host-planned row-aligned
// partition (capi.cu plan_partition; no co-residency needed, split rows are finished by their
// last CTA).  Tiles of STILE observations (index columns + multiplicity/weight column) are moved
// by the TMA bulk-copy engine (cp.async.bulk, completion on an mbarrier) into a double buffer; the
// per-observation factors are bulk-copied into shared memory once per CTA when they fit (SF),
// otherwise read through L1.
//
// Lane groups: G = 8 lanes per observation, VPL = RP / 8 doubles per lane, columns interleaved
// so that one quarter-warp LDS.128 reads one contiguous 128-byte row segment (conflict-free).
// Each lane group walks a CONTIGUOUS sub-chunk of every row segment in batches of B observations
// (B = 4 for VPL <= 4, 2 for VPL = 8): the B index sets arrive as one vector LDS per mode (the plan's
// index columns have a stride that is a multiple of 4, so every staged column shares one
// alignment), and the B partial dot products are reduced together by a transposed butterfly
// (reduce-scatter then all-gather: 7 double shuffles for 4 dots instead of 12).  The run
// accumulator stays in registers; runs are folded into a per-lane-group row accumulator in shared
// memory; rows are reduced over lane groups in a fixed order.  Results are bit-reproducible for a
// given plan.
#include <cstdlib>

#include "kernels.cuh"

namespace cphifi {
namespace {

constexpr int ST = 512;      // threads per CTA
constexpr int STILE = 1024;  // observations per staged tile
constexpr int NSTAGE = 4;    // tile ring depth (warps drift up to NSTAGE - 2 tiles apart)
constexpr int SPAD = 8;      // staged-column slack (alignment of the bulk copies)
constexpr int SMEM_CAP = 226 * 1024;  // opt-in maximum (227 KB) minus the static shared memory
constexpr int G = 8;         // lanes per observation

template <int RP>
struct Shape {
    static constexpr int VPL = RP / G;                 // doubles per lane per row (RP >= 16)
    static constexpr int B = VPL <= 4 ? 4 : 2;         // observations per batch
    static constexpr int NG = ST / G;                  // lane groups per CTA
    static constexpr int RS = RP + 2;                  // row stride of the accumulators
};

__device__ __forceinline__ unsigned atom_add_acqrel_s(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// TMA bulk copy global -> shared (bytes % 16 == 0, both addresses 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Staged column: elements [e0, e0 + cnt) of `base` (16-byte aligned) land at smem + (e0 mod AL).
template <typename T>
__device__ __forceinline__ unsigned col_bytes(int64_t e0, int cnt) {
    constexpr int AL = 16 / (int)sizeof(T);
    const int off = (int)(e0 & (AL - 1));
    return (unsigned)((((off + cnt) * (int)sizeof(T)) + 15) & ~15);
}
template <typename T>
__device__ __forceinline__ void stage_col(T* smem, const T* base, int64_t e0, int cnt, uint64_t* bar) {
    constexpr int AL = 16 / (int)sizeof(T);
    bulk_g2s(smem, base + (e0 & ~(int64_t)(AL - 1)), col_bytes<T>(e0, cnt), bar);
}

// Lane `gl` of a lane group owns the row columns 2 u G + 2 gl + {0, 1}, u < VPL / 2.
template <int RP, bool SMEM>
__device__ __forceinline__ void ld_row(double (&v)[Shape<RP>::VPL], const double* row, int gl) {
#pragma unroll
    for (int u = 0; u < Shape<RP>::VPL / 2; ++u) {
        double2 t;
        if constexpr (SMEM) t = *reinterpret_cast<const double2*>(row + 2 * u * G + 2 * gl);
        else t = __ldg(reinterpret_cast<const double2*>(row + 2 * u * G + 2 * gl));
        v[2 * u] = t.x;
        v[2 * u + 1] = t.y;
    }
}

// Sum each of d[0..B) over the G lanes of the lane group; every lane ends with all B totals.
// Reduce-scatter over offsets G/2 .. G/B (each step halves the values a lane carries), butterfly
// over the remaining offsets, then all-gather in reverse.  Fixed order: deterministic.
template <int B>
__device__ __forceinline__ void group_reduce(double (&d)[B], unsigned gmask, int lane) {
    if constexpr (B == 1) {
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) d[0] += __shfl_xor_sync(gmask, d[0], off, G);
    } else {
        // reduce-scatter
        double v[B];
#pragma unroll
        for (int i = 0; i < B; ++i) v[i] = d[i];
        int w = B;
        int off = G / 2;
#pragma unroll
        for (int st = 0; (1 << st) < B; ++st) {
            const bool hi = (lane & off) != 0;
            const int h = w / 2;
#pragma unroll
            for (int i = 0; i < h; ++i) {
                const double keep = hi ? v[i + h] : v[i];
                const double send = hi ? v[i] : v[i + h];
                v[i] = keep + __shfl_xor_sync(gmask, send, off, G);
            }
            w = h;
            off >>= 1;
        }
#pragma unroll
        for (; off > 0; off >>= 1) v[0] += __shfl_xor_sync(gmask, v[0], off, G);
        // all-gather (offsets G/B .. G/2)
        int wg = 1;
        int og = G / B;
#pragma unroll
        for (int st = 0; (1 << st) < B; ++st) {
            const bool hi = (lane & og) != 0;
#pragma unroll
            for (int i = 0; i < wg; ++i) {
                const double other = __shfl_xor_sync(gmask, v[i], og, G);
                const double mine = v[i];
                v[i] = hi ? other : mine;
                v[i + wg] = hi ? mine : other;
            }
            wg *= 2;
            og *= 2;
        }
#pragma unroll
        for (int i = 0; i < B; ++i) d[i] = v[i];
    }
}

template <int B>
__device__ __forceinline__ void ld_idx(int (&v)[B], const int32_t* p) {
    if constexpr (B == 4) {
        const int4 t = *reinterpret_cast<const int4*>(p);
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    } else if constexpr (B == 2) {
        const int2 t = *reinterpret_cast<const int2*>(p);
        v[0] = t.x; v[1] = t.y;
    } else {
        v[0] = *p;
    }
}

// aux: 0 = none (operator, uncoalesced), 1 = int32 multiplicities (operator, coalesced plan),
// 2 = fp64 weights (RHS: the observed values)
__device__ __forceinline__ void cpa16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cpa_commit_s() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cpa_wait1_s() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cpa_wait0_s() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// PF: the mode-1 factor rows of the NEXT batch are copied (cp.async, each lane its own 16-byte
// chunks, so no lane-group synchronisation) into a 2-slot per-lane-group ring while the current
// batch computes: factors read through L1 (config 4: 256 KB, not shared-memory resident) stop
// being a chain of dependent L1-miss -> L2 round trips.
template <int RP, int DO, bool SF, int AUX, bool PF>
__global__ void __launch_bounds__(ST, 1) stream_kernel(const FusedArgs a) {
    using S = Shape<RP>;
    constexpr int VPL = S::VPL, NG = S::NG, RS = S::RS, B = S::B;
    constexpr int NW = ST / 32;
    constexpr int CI = STILE + SPAD;  // staged column capacity (elements)
    constexpr bool DOT = AUX != 2;
    constexpr int AUXB = AUX == 0 ? 0 : (AUX == 1 ? 4 : 8);
    extern __shared__ __align__(128) unsigned char smem_raw[];
    // barriers: full[NSTAGE] (TMA bytes landed), empty[NSTAGE] (every warp done), factors
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* empty = full + NSTAGE;
    uint64_t* fbar = empty + NSTAGE;
    double* red2 = reinterpret_cast<double*>(smem_raw + 128);        // RP
    double* acc_s = red2 + RP;                                       // NG x RS lane-group row accumulators
    int32_t* idx_s = reinterpret_cast<int32_t*>(acc_s + NG * RS);    // NSTAGE x DO x CI
    unsigned char* aux_s = reinterpret_cast<unsigned char*>(idx_s + NSTAGE * DO * CI);  // NSTAGE x CI x AUXB
    double* sfac = reinterpret_cast<double*>(aux_s + NSTAGE * CI * AUXB);               // staged factors
    __shared__ int s_last;

    const int c = blockIdx.x;
    const int64_t ca = a.cta_beg[c], cb = a.cta_beg[c + 1];
    if (ca >= cb) return;
    const int tid = threadIdx.x;
    const int g = tid / G, gl = tid % G, lane = tid & 31;
    const unsigned gmask = ((1u << G) - 1u) << (lane - lane % G);
    const int ntiles = (int)((cb - ca + STILE - 1) / STILE);

    // factor sizes (rows of other mode m = (next offset - offset) / RP)
    int64_t frows[DO];
#pragma unroll
    for (int m = 0; m < DO; ++m) frows[m] = ((m + 1 < DO ? a.fac_off[m + 1] : a.fac_total) - a.fac_off[m]) / RP;

    for (int e = tid; e < NG * RS; e += ST) acc_s[e] = 0.0;
    if (tid == 0) {
        for (int b = 0; b < NSTAGE; ++b) {
            mbar_init(full + b, 1);
            mbar_init(empty + b, NW);
        }
        mbar_init(fbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // Every int32 column shares the staged offset t0 mod 4 (a.q % 4 == 0, aligned bases).
    auto issue_tile = [&](int t) {  // thread 0
        const int buf = t % NSTAGE;
        uint64_t* bar = full + buf;
        const int64_t t0 = ca + (int64_t)t * STILE;
        const int cnt = (int)min((int64_t)STILE, cb - t0);
        unsigned bytes = DO * col_bytes<int32_t>(t0, cnt);
        if constexpr (AUX == 1) bytes += col_bytes<int32_t>(t0, cnt);
        if constexpr (AUX == 2) bytes += col_bytes<double>(t0, cnt);
        mbar_expect_tx(bar, bytes);
#pragma unroll
        for (int m = 0; m < DO; ++m) stage_col(idx_s + (buf * DO + m) * CI, a.idx, (int64_t)m * a.q + t0, cnt, bar);
        if constexpr (AUX == 1) stage_col(reinterpret_cast<int32_t*>(aux_s) + buf * CI, a.mult, t0, cnt, bar);
        if constexpr (AUX == 2) stage_col(reinterpret_cast<double*>(aux_s) + buf * CI, a.weights, t0, cnt, bar);
    };

    if (tid == 0) {
        fence_proxy_async();
        if constexpr (SF) {  // per-observation factors (other modes 1..DO-1), once per CTA
            unsigned bytes = 0;
#pragma unroll
            for (int m = 1; m < DO; ++m) bytes += (unsigned)(frows[m] * RP * 8);
            mbar_expect_tx(fbar, bytes);
            int64_t so = 0;
#pragma unroll
            for (int m = 1; m < DO; ++m) {
                const int64_t tot = frows[m] * RP * 8;
                for (int64_t b0 = 0; b0 < tot; b0 += 32768) {
                    const unsigned nb = (unsigned)min((int64_t)32768, tot - b0);
                    bulk_g2s(reinterpret_cast<unsigned char*>(sfac + so) + b0,
                             reinterpret_cast<const unsigned char*>(a.fac + a.fac_off[m]) + b0, nb, fbar);
                }
                so += frows[m] * RP;
            }
        }
        for (int t = 0; t < min(ntiles, NSTAGE); ++t) issue_tile(t);
    }
    const double* fac_m[DO];  // base of the factor rows (smem or global)
    {
        int64_t so = 0;
#pragma unroll
        for (int m = 0; m < DO; ++m) {
            if (SF && m > 0) {
                fac_m[m] = sfac + so;
                so += frows[m] * RP;
            } else {
                fac_m[m] = a.fac + a.fac_off[m];
            }
        }
    }
    if constexpr (SF) mbar_wait(fbar, 0);

    int64_t cur = a.cta_rows[2 * c];
    int64_t cur_end = a.row_ptr[cur + 1];
    int cur_a = -1;
    double p[VPL], accg[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
        p[v] = 0.0;
        accg[v] = 0.0;
    }
    double* my_acc = acc_s + g * RS;

    // fold the run accumulator into this lane group's row accumulator: acc += A_1(cur_a,:) o accg
    auto run_flush = [&]() {
        if (cur_a >= 0) {
            double a1[VPL];
            ld_row<RP, false>(a1, fac_m[0] + (int64_t)cur_a * RP, gl);
#pragma unroll
            for (int u = 0; u < VPL / 2; ++u) {
                double2* d = reinterpret_cast<double2*>(my_acc + 2 * u * G + 2 * gl);
                double2 t = *d;
                t.x = fma(a1[2 * u], accg[2 * u], t.x);
                t.y = fma(a1[2 * u + 1], accg[2 * u + 1], t.y);
                *d = t;
            }
#pragma unroll
            for (int v = 0; v < VPL; ++v) accg[v] = 0.0;
        }
    };
    auto run_start = [&](int an) {
        if constexpr (DOT) {
            double a1[VPL], xh[VPL];
            ld_row<RP, false>(a1, fac_m[0] + (int64_t)an * RP, gl);
            ld_row<RP, false>(xh, a.xhat_rm + cur * RP, gl);
#pragma unroll
            for (int v = 0; v < VPL; ++v) p[v] = xh[v] * a1[v];
        }
        cur_a = an;
    };
    // reduce the lane-group row accumulators in a fixed order and emit row `row`
    auto row_flush = [&](int64_t row) {
        __syncthreads();
        for (int j = tid >> 5; j < RP; j += NW) {
            double s = 0.0;
            for (int q = lane; q < NG; q += 32) s += acc_s[q * RS + j];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
            if (lane == 0) red2[j] = s;
        }
        __syncthreads();
        for (int e = tid; e < NG * RS; e += ST) acc_s[e] = 0.0;
        const int ncta = a.row_ncta[row];
        const bool split = ncta > 1;
        const int64_t first_row = a.cta_rows[2 * c];
        if (tid < RP) {
            if (!split) {
                double* dst = a.yhat_rm + row * RP + tid;
                *dst = a.accumulate ? *dst + red2[tid] : red2[tid];
            } else {
                double* dst = row == first_row ? a.slot_a + (int64_t)c * RP : a.slot_b + (int64_t)c * RP;
                dst[tid] = red2[tid];
            }
        }
        if (split) {  // the last of the row's CTAs to arrive sums the slots in CTA order
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                s_last = atom_add_acqrel_s(a.rowcnt + row, 1u) == (unsigned)ncta - 1;
                if (s_last) a.rowcnt[row] = 0;
            }
            __syncthreads();
            if (s_last && tid < RP) {
                const int u0 = a.row_first_cta[row];
                double s = a.row_ptr[row] == a.cta_beg[u0] ? __ldcg(a.slot_a + (int64_t)u0 * RP + tid)
                                                           : __ldcg(a.slot_b + (int64_t)u0 * RP + tid);
                for (int u = u0 + 1; u < u0 + ncta; ++u) s += __ldcg(a.slot_a + (int64_t)u * RP + tid);
                double* dst = a.yhat_rm + row * RP + tid;
                *dst = a.accumulate ? *dst + s : s;
            }
        }
    };

    for (int t = 0; t < ntiles; ++t) {
        const int buf = t % NSTAGE;
        // producer: refill the slot tile t-1 used once every warp has released it
        if (tid == 0 && t >= 1 && t - 1 + NSTAGE < ntiles) {
            mbar_wait(empty + (t - 1) % NSTAGE, (unsigned)(((t - 1) / NSTAGE) & 1));
            fence_proxy_async();
            issue_tile(t - 1 + NSTAGE);
        }
        mbar_wait(full + buf, (unsigned)((t / NSTAGE) & 1));
        const int64_t t0 = ca + (int64_t)t * STILE;
        const int64_t t1 = min(cb, t0 + STILE);
        const int off = (int)(t0 & 3);  // staged position P = tile-local index + off (int32 columns)
        const int32_t* ti[DO];
#pragma unroll
        for (int m = 0; m < DO; ++m) ti[m] = idx_s + (buf * DO + m) * CI;
        const int32_t* tm = reinterpret_cast<const int32_t*>(aux_s) + buf * CI;
        const double* tw = reinterpret_cast<const double*>(aux_s) + buf * CI + (off & 1) - off;  // tw[P]

        // Every lane group runs the same number of single / batch rounds (warp maxima), so the
        // shuffles below always see the whole warp converged; `valid` masks the padding rounds.
        // single observation at staged position P (run change handled inline, no collectives)
        auto one = [&](int P, bool valid) {
            int ix[DO];
#pragma unroll
            for (int m = 0; m < DO; ++m) ix[m] = valid ? ti[m][P] : 0;
            double z[VPL];
            ld_row<RP, SF>(z, fac_m[1] + (int64_t)ix[1] * RP, gl);
#pragma unroll
            for (int m = 2; m < DO; ++m) {
                double f[VPL];
                ld_row<RP, SF>(f, fac_m[m] + (int64_t)ix[m] * RP, gl);
#pragma unroll
                for (int v = 0; v < VPL; ++v) z[v] *= f[v];
            }
            if (valid && ix[0] != cur_a) {
                run_flush();
                run_start(ix[0]);
            }
            double s[1];
            if constexpr (DOT) {
                s[0] = 0.0;
#pragma unroll
                for (int v = 0; v < VPL; ++v) s[0] = fma(p[v], z[v], s[0]);
                group_reduce<1>(s, 0xffffffffu, lane);
                if constexpr (AUX == 1) s[0] *= valid ? (double)tm[P] : 0.0;
            } else {
                s[0] = valid ? tw[P] : 0.0;
            }
            if (valid) {
#pragma unroll
                for (int v = 0; v < VPL; ++v) accg[v] = fma(s[0], z[v], accg[v]);
            }
        };
        // PF ring: slot (g, sl) holds B rows of RP doubles
        double* pf_base = sfac + (int64_t)g * 2 * B * RP;
        auto prefetch = [&](int P, bool valid, int sl) {
            if constexpr (PF) {
                int ib[B];
                if (valid) ld_idx<B>(ib, ti[1] + P);
                else {
#pragma unroll
                    for (int b = 0; b < B; ++b) ib[b] = 0;
                }
#pragma unroll
                for (int b = 0; b < B; ++b)
#pragma unroll
                    for (int u = 0; u < VPL / 2; ++u)
                        cpa16(pf_base + (sl * B + b) * RP + 2 * u * G + 2 * gl,
                              fac_m[1] + (int64_t)ib[b] * RP + 2 * u * G + 2 * gl);
                cpa_commit_s();
            }
        };
        // B observations at aligned staged position P, all in one run (else `need` defers them)
        auto batch = [&](int P, bool valid, int sl) {
            int ia[B];
            if (valid) ld_idx<B>(ia, ti[0] + P);
            else {
#pragma unroll
                for (int b = 0; b < B; ++b) ia[b] = cur_a;
            }
            // a is nondecreasing inside a row segment: equal ends = one run
            if (ia[0] == ia[B - 1] && ia[0] != cur_a) {
                run_flush();
                run_start(ia[0]);
            }
            const bool need = ia[0] != ia[B - 1];  // a run starts inside: redo as singles
            const bool use = valid && !need;
            double z[B][VPL];
            {
                int ib[B];
                if (use) ld_idx<B>(ib, ti[1] + P);
                else {
#pragma unroll
                    for (int b = 0; b < B; ++b) ib[b] = 0;
                }
                if constexpr (PF) {
                    cpa_wait1_s();  // this lane's copies of this batch have landed
#pragma unroll
                    for (int b = 0; b < B; ++b) ld_row<RP, true>(z[b], pf_base + (sl * B + b) * RP, gl);
                } else {
#pragma unroll
                    for (int b = 0; b < B; ++b) ld_row<RP, SF>(z[b], fac_m[1] + (int64_t)ib[b] * RP, gl);
                }
            }
#pragma unroll
            for (int m = 2; m < DO; ++m) {
                int ib[B];
                if (use) ld_idx<B>(ib, ti[m] + P);
                else {
#pragma unroll
                    for (int b = 0; b < B; ++b) ib[b] = 0;
                }
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    double f[VPL];
                    ld_row<RP, SF>(f, fac_m[m] + (int64_t)ib[b] * RP, gl);
#pragma unroll
                    for (int v = 0; v < VPL; ++v) z[b][v] *= f[v];
                }
            }
            double s[B];
            if constexpr (DOT) {
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    s[b] = 0.0;
#pragma unroll
                    for (int v = 0; v < VPL; ++v) s[b] = fma(p[v], z[b][v], s[b]);
                }
                group_reduce<B>(s, 0xffffffffu, lane);
                if constexpr (AUX == 1) {
                    int mu[B];
                    if (use) ld_idx<B>(mu, tm + P);
#pragma unroll
                    for (int b = 0; b < B; ++b) s[b] *= use ? (double)mu[b] : 0.0;
                }
            } else {
#pragma unroll
                for (int b = 0; b < B; ++b) s[b] = use ? tw[P + b] : 0.0;
            }
            if (use) {
#pragma unroll
                for (int b = 0; b < B; ++b)
#pragma unroll
                    for (int v = 0; v < VPL; ++v) accg[v] = fma(s[b], z[b][v], accg[v]);
            }
            const bool redo = valid && need;
            if (__any_sync(0xffffffffu, redo)) {
#pragma unroll 1
                for (int b = 0; b < B; ++b) one(P + b, redo);
            }
        };

        int64_t seg = t0;
        while (seg < t1) {
            const int64_t seg_end = min(t1, cur_end);
            // lane group g: a contiguous sub-chunk [pb, pe) of the segment's staged positions;
            // inner boundaries are multiples of 4 so batches load their indices as one vector
            const int p0 = (int)(seg - t0) + off, p1 = (int)(seg_end - t0) + off;
            const int len = p1 - p0;
            const int pb = g == 0 ? p0 : max(p0, (p0 + (len * g) / NG) & ~3);
            const int pe = g == NG - 1 ? p1 : max(p0, (p0 + (len * (g + 1)) / NG) & ~3);
            const int pa = min(pe, (pb + B - 1) & ~(B - 1));   // first aligned position
            const int nbat = (pe - pa) / B;
            const int pt = pa + nbat * B;                       // tail start
            const int nh = __reduce_max_sync(0xffffffffu, (unsigned)(pa - pb));
            const int nb = __reduce_max_sync(0xffffffffu, (unsigned)nbat);
            const int nt = __reduce_max_sync(0xffffffffu, (unsigned)(pe - pt));
#pragma unroll 1
            for (int h = 0; h < nh; ++h) one(pb + h, pb + h < pa);
#pragma unroll 1
            if constexpr (PF) {
                if (nb > 0) prefetch(pa, 0 < nbat, 0);
                for (int j = 0; j < nb; ++j) {
                    if (j + 1 < nb) prefetch(pa + (j + 1) * B, j + 1 < nbat, (j + 1) & 1);
                    else cpa_commit_s();  // keep one group per batch: wait_group 1 = this batch
                    batch(pa + j * B, j < nbat, j & 1);
                }
                cpa_wait0_s();
            } else {
                for (int j = 0; j < nb; ++j) batch(pa + j * B, j < nbat, 0);
            }
#pragma unroll 1
            for (int h = 0; h < nt; ++h) one(pt + h, pt + h < pe);
            seg = seg_end;
            if (seg_end == cur_end) {  // row complete (possibly the CTA's last, split row)
                run_flush();
                cur_a = -1;
                row_flush(cur);
                if (seg_end < cb) {
                    do {
                        ++cur;
                        cur_end = a.row_ptr[cur + 1];
                    } while (cur_end <= seg_end);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + buf);  // this warp is done with the buffer
    }
    if (cur_end > cb) {  // the CTA's range ends inside row `cur` (split row)
        run_flush();
        row_flush(cur);
    }
}

int aux_kind(const FusedArgs& a) { return a.weights ? 2 : (a.mult ? 1 : 0); }

template <int RP, int DO, bool SF, int AUX, bool PF>
void launch_t(const FusedArgs& a, int grid, size_t smem, cudaStream_t s) {
    auto kern = stream_kernel<RP, DO, SF, AUX, PF>;
    func_attr_once((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_CAP);
    kern<<<grid, ST, smem, s>>>(a);
}

template <int RP, int DO, bool SF, bool PF>
void launch_sf(const FusedArgs& a, int grid, size_t smem, cudaStream_t s) {
    switch (aux_kind(a)) {
        case 0: launch_t<RP, DO, SF, 0, PF>(a, grid, smem, s); break;
        case 1: launch_t<RP, DO, SF, 1, PF>(a, grid, smem, s); break;
        default: launch_t<RP, DO, SF, 2, PF>(a, grid, smem, s); break;
    }
}

template <int RP, int DO>
void launch_do(const FusedArgs& a, int grid, size_t smem, bool sf, bool pf, cudaStream_t s) {
    if (sf) launch_sf<RP, DO, true, false>(a, grid, smem, s);
    else if (pf) launch_sf<RP, DO, false, true>(a, grid, smem, s);
    else launch_sf<RP, DO, false, false>(a, grid, smem, s);
}

template <int RP>
void launch_rp(const FusedArgs& a, int grid, size_t smem, bool sf, bool pf, cudaStream_t s) {
    switch (a.dother) {
        case 2: launch_do<RP, 2>(a, grid, smem, sf, pf, s); break;
        case 3: launch_do<RP, 3>(a, grid, smem, sf, pf, s); break;
        case 4: launch_do<RP, 4>(a, grid, smem, sf, pf, s); break;
        case 5: launch_do<RP, 5>(a, grid, smem, sf, pf, s); break;
        default: throw_invalid("stream scatter-gather: needs 2..5 other modes");
    }
}

template <int RP>
size_t pf_bytes() { return sizeof(double) * (size_t)Shape<RP>::NG * 2 * Shape<RP>::B * RP; }

}  // namespace

bool stream_supported(int64_t rp, int dother) { return rp >= 16 && rp <= 64 && dother >= 2 && dother <= 5; }

size_t stream_smem_bytes(int64_t rp, int dother, int64_t sf_doubles, int aux_bytes) {
    const int64_t ng = ST / G;
    const int64_t ci = STILE + SPAD;
    return 128 + sizeof(double) * (rp + ng * (rp + 2)) + sizeof(int32_t) * NSTAGE * dother * ci +
           NSTAGE * ci * aux_bytes + sizeof(double) * sf_doubles;
}

size_t stream_smem_cap() { return SMEM_CAP; }

void stream_scatter_gather(const FusedArgs& a, int grid, int64_t sf_doubles, cudaStream_t s) {
    const int ab = a.weights ? 8 : (a.mult ? 4 : 0);
    // factors through L1 when this launch's tiles leave no room for them (e.g. the RHS build)
    if (stream_smem_bytes(a.rp, a.dother, sf_doubles, ab) > SMEM_CAP) sf_doubles = 0;
    size_t smem = stream_smem_bytes(a.rp, a.dother, sf_doubles, ab);
    const bool sf = sf_doubles > 0;
    // factors through L1: prefetch ring for the per-observation rows when shared memory allows
    const size_t pfb = a.rp == 16 ? pf_bytes<16>() : (a.rp == 32 ? pf_bytes<32>() : pf_bytes<64>());
    bool pf = !sf && smem + pfb <= SMEM_CAP;
    if (const char* e = std::getenv("CPHIFI_STREAM_PF")) pf = pf && std::atoi(e) != 0;
    if (pf) smem += pfb;
    switch (a.rp) {
        case 16: launch_rp<16>(a, grid, smem, sf, pf, s); break;
        case 32: launch_rp<32>(a, grid, smem, sf, pf, s); break;
        case 64: launch_rp<64>(a, grid, smem, sf, pf, s); break;
        default: throw_invalid("stream scatter-gather: padded rank must be in [16, 64]");
    }
    CPHIFI_CHECK_LAUNCH();
}

}  // namespace cphifi
