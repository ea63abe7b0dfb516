// k_gram3.cu — row-Gram build, register-fragment form (sm_100a DMMA).
//
// G_i = sum_{l: i_k(l) = i} w_l z_l z_l',  z_l = A_1(a_l,:) o A_2(b_l,:) o ...   (the identity behind
// the row-Gram operator, k_gram.cu; the reference's per-observation gather + scatter,
// observations.hpp:174-198, applied to every basis vector at once).
//
// The single-pass builds of k_gram.cu stage a batch of Khatri-Rao rows in shared memory and read
// the DMMA fragments back from it: one or two 8-byte loads per DMMA (4 wavefronts), plus the batch's
// own stores, which holds them near half the FP64 tensor rate (config 3: 24.5 ms for a 5.7 ms
// floor).  Here each lane builds exactly the fragment values it feeds the tensor core, in registers,
// straight from the factor rows:
//   * G's rows / columns are tiled so that tile t holds the indices c = NT g + t (g = 0..7,
//     NT = RP / 8).  For a k-step of 4 entries, lane (g, kq) then needs z_kq(NT g + t) for every t:
//     NT CONSECUTIVE doubles of each factor row (NT / 2 16-byte loads per mode), and the warp's loads
//     of one mode cover the 4 entries' rows exactly (conflict-free);
//   * A(i, k) = w_k z_k(NT i + ti), B(k, j) = z_k(NT j + tj): lane (g, kq) holds both for all tiles,
//     so every upper-triangle tile pair (ti <= tj) is one DMMA on registers — NT (NT + 1) / 2 DMMA per
//     k-step with no shared-memory traffic besides the factor rows;
//   * TW warps (a team) walk the same entries and split the tile pairs; a CTA holds (its warps) / TW
//     teams, each with its own contiguous entry range (equal-count, split rows finished by the last
//     arrival summing the units' slots in unit order: deterministic).  TW = 1 throughout: at RP = 64
//     a warp holds all 36 tile pairs with 8 warps per CTA (g3_threads; CPHIFI_GRAM3_TW=4 splits them
//     over 4 warps of 16, measured 54.3 against 40.7 ms at config 4);
//   * the plan's indices and multiplicities arrive 32 entries at a time, one coalesced load per
//     column, one batch ahead, and are handed to the k-step's lanes by shuffles; the factors are
//     staged in shared memory when they fit (config 3: 3 x 64 KB), else read through L1.
// k-steps sit at fixed 4-aligned positions; a step that straddles a row end is run once per row
// with the other row's entries masked (rows hold ~1e5 entries, so this is rare).
//
// STAGE 3 (3-way factor-block parts, config 4: the factors do not fit shared memory): the first
// other mode is HOISTED per run instead of gathered per entry.  The plan is lexicographic, so the
// entries of a row form runs of equal a, and over a run
//     sum_l w_l z_l z_l' = (A_1(a,:)' A_1(a,:)) o M,   M = sum_{l in run} w_l t_l t_l',  t_l = A_2(b_l,:)
// (z_l = A_1(a,:) o t_l): the k-steps accumulate M from the staged block's rows alone (no mode-0 load
// per entry), and a run end folds G += (a a') o M on the accumulator registers (each lane scales its
// own fragment elements by A_1(a, ii) A_1(a, jj)) and clears M.  A k-step that straddles a run end is
// run once per run with the other entries masked (a is non-decreasing inside a row); the A_1 rows of
// the next batch's runs are prefetched into L1 when the batch is loaded.  MEASURED SLOWER (opt-in,
// CPHIFI_GRAM3_PARTS=3): config 4 72.6 ms against 54.4 ms for STAGE 1 (profiles/round2/
// gram_parts_config4.log) — with ~28-entry runs per part a quarter of the k-steps straddle a run end
// (a second masked DMMA pass), every run end pays a fold whose A_1 loads wait on L1 / L2, and the
// two accumulator sets spill at 128 registers.
#include <climits>
#include <cstdlib>
#include <type_traits>

#include "kernels.cuh"

namespace cphifi {
namespace {

// threads per CTA: 16 warps of single-warp teams (TW = 1) up to RP = 32; at RP = 64 a single warp
// holds all 36 upper-triangle tile pairs (72 accumulator doubles) only with up to 255 registers, so
// 8 warps per CTA (2 per scheduler: one warp's 36 DMMAs cover the other's z build) — TW > 1 (warps
// splitting the pairs, each rebuilding the same z) spends ~75 instructions per 9 DMMAs
template <int RP, int TW>
constexpr int g3_threads() { return (RP == 64 && TW == 1) ? 256 : 512; }

__device__ __forceinline__ void dmma3(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ unsigned atom_add_acqrel3(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

template <int RP, int TW>
struct G3 {
    static constexpr int NT = RP / 8;
    static constexpr int NUP = NT * (NT + 1) / 2;
    static constexpr int TPW = (NUP + TW - 1) / TW;  // tile pairs per warp
    static constexpr int THREADS = g3_threads<RP, TW>();
    static constexpr int TEAMS = THREADS / 32 / TW;
};

// index of tile pair (ti, tj), ti <= tj, row-major over the upper triangle of NT x NT tiles
template <int NT>
__host__ __device__ constexpr int pair_index(int ti, int tj) {
    return ti * NT - ti * (ti - 1) / 2 + (tj - ti);
}

// STAGE: 2 = every factor staged in shared memory; 1 = modes 1.. staged (a factor-block part: mode 0,
// constant along the plan's runs, read through L1); 3 = as 1 with mode 0 hoisted per run (DO = 2);
// 0 = none staged
template <int RP, int DO, int TW, int STAGE>
__global__ void __launch_bounds__(g3_threads<RP, TW>(), 1) gram3_kernel(const GramArgs a, int units) {
    constexpr bool SF = STAGE > 0;
    constexpr bool HOIST = STAGE == 3;
    static_assert(!HOIST || DO == 2, "gram build v3: the hoisted form is for 3-way plans");
    using C = G3<RP, TW>;
    constexpr int NT = C::NT, TPW = C::TPW;
    extern __shared__ __align__(16) double g3s[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, kq = lane & 3;
    // Staged rows: a 16-byte load instruction is served a quarter-warp (8 lanes: g in {2p, 2p+1} x
    // kq) at a time, i.e. 4 different factor rows x 2 lanes.  Lane (g, kq) reads its CPL chunks in the
    // order rotated by kq (instruction c: chunk (c + kq) mod CPL), so the 4 rows of a quarter hit
    // different bank groups (RP 64: conflict-free; RP 32: pairs of rows share one), and the chunks of
    // row R are stored XOR-swizzled by sw(R) (RP 32: R's parity flips the 64-byte halves, so those
    // pairs collide only when their rows have equal parity; RP 16: two bits of R).  The rotation is
    // undone in registers once per k-step.
    constexpr int CPL = NT / 2;  // 16-byte chunks per lane per row
    auto sw = [](int64_t grow) -> int {
        return CPL == 2 ? (int)((grow & 1) << 2) : CPL == 1 ? (int)((grow & 3) << 1) : 0;
    };
    const int64_t sbeg = STAGE == 2 ? 0 : a.fac_off[1];  // first staged double (a row boundary)
    if constexpr (SF) {
        const double2* src = reinterpret_cast<const double2*>(a.fac + sbeg);
        for (int64_t e = tid; e < (a.fac_total - sbeg) / 2; e += C::THREADS) {
            const int jj = (int)(e % (RP / 2));
            const int64_t grow = e / (RP / 2);
            reinterpret_cast<double2*>(g3s)[e] = __ldg(src + (e - jj) + (jj ^ sw(grow)));
        }
    }
    __syncthreads();  // the only CTA-wide barrier: teams are independent from here on
    const int team = warp / TW, tw = warp % TW;
    const int u = blockIdx.x * C::TEAMS + team;
    if (u >= units) return;
    const int64_t beg = a.cta_beg[u], end = a.cta_beg[u + 1];
    if (beg >= end) return;

    // The warp's tile pairs (uu % TW == tw) must be a compile-time set: with a runtime tw every
    // DMMA of the k-step is issued predicated, with a register select per accumulator and a
    // convergence barrier around each (measured at TW = 4: 10 % of the instructions DMMA, the
    // tensor pipe at a third of its FP64 rate).  The body is instantiated per tw.
    auto body = [&](auto twc) {
        constexpr int TWI = decltype(twc)::value;
        double acc[TPW][2];
        double accm[HOIST ? TPW : 1][2];  // HOIST: the current run's M (acc holds G)
    #pragma unroll
        for (int x = 0; x < TPW; ++x) acc[x][0] = acc[x][1] = 0.0;
    #pragma unroll
        for (int x = 0; x < (HOIST ? TPW : 1); ++x) accm[x][0] = accm[x][1] = 0.0;

        const int64_t first_row = a.cta_rows[2 * u];
        int64_t row = first_row;
        int64_t row_beg = a.row_ptr[row], row_end = a.row_ptr[row + 1];

        auto flush = [&](int64_t rr) {
            const int nu = a.row_ncta[rr];
            double* dst = nu == 1 ? a.g + rr * RP * RP
                        : rr == first_row ? a.slot_a + (int64_t)u * RP * RP
                                          : a.slot_b + (int64_t)u * RP * RP;
    #pragma unroll
            for (int ti = 0; ti < NT; ++ti)
    #pragma unroll
                for (int tj = ti; tj < NT; ++tj) {
                    const int uu = pair_index<NT>(ti, tj);
                    if (uu % TW != TWI) continue;
    #pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int ii = NT * g + ti, jj = NT * (2 * kq + h) + tj;
                        const double v = acc[uu / TW][h] + (a.accumulate && nu == 1 ? dst[ii * RP + jj] : 0.0);
                        dst[ii * RP + jj] = v;
                        if (ti != tj) dst[jj * RP + ii] = v;
                    }
                }
    #pragma unroll
            for (int x = 0; x < TPW; ++x) acc[x][0] = acc[x][1] = 0.0;
            if (nu > 1) {  // the last of the row's units (TW warps each) sums the unit slots in unit order
                __syncwarp();
                unsigned last = 0;
                if (lane == 0) {
                    __threadfence();
                    last = atom_add_acqrel3(a.rowcnt + rr, 1u) == (unsigned)(nu * TW) - 1;
                    if (last) a.rowcnt[rr] = 0;
                }
                last = __shfl_sync(0xffffffffu, last, 0);
                if (last) {
                    const int u0 = a.row_first_cta[rr];
                    const bool starts = a.row_ptr[rr] == a.cta_beg[u0];
                    for (int e = lane; e < RP * RP; e += 32) {
                        double s = starts ? __ldcg(a.slot_a + (int64_t)u0 * RP * RP + e)
                                          : __ldcg(a.slot_b + (int64_t)u0 * RP * RP + e);
                        for (int v = u0 + 1; v < u0 + nu; ++v) s += __ldcg(a.slot_a + (int64_t)v * RP * RP + e);
                        a.g[rr * RP * RP + e] = a.accumulate ? a.g[rr * RP * RP + e] + s : s;
                    }
                }
            }
        };

        // index / multiplicity batches: lane L holds entry b0 + L of every column (cur), and the next
        // batch (nxt) is in flight.  Positions below are 32-bit offsets from p0 (units hold < 2^31
        // entries); iterations take 8 entries (two k-steps) at 8-aligned offsets, inside one batch.
        const int64_t p0 = beg & ~(int64_t)31;
        const int nrel = (int)(end - p0);
        int b0 = 0;
        int32_t cur[DO + 1], nxt[DO + 1];
        auto load_batch = [&](int base, int32_t (&v)[DO + 1]) {
            const int64_t e = p0 + base + lane;
            const bool ok = e >= beg && e < end;
    #pragma unroll
            for (int m = 0; m < DO; ++m) v[m] = ok ? __ldg(a.idx + (int64_t)m * a.q + e) : 0;
            v[DO] = ok ? (a.mult ? (__ldg(a.mult + e) & RUN_MULT_MASK) : 1) : 0;
            if constexpr (HOIST) {  // the A_1 rows of the runs starting in this batch, into L1
                const int32_t prev = __shfl_up_sync(0xffffffffu, v[0], 1);
                if (ok && (lane == 0 || prev != v[0])) {
                    const char* row = reinterpret_cast<const char*>(a.fac + a.fac_off[0] + (int64_t)v[0] * RP);
    #pragma unroll
                    for (int c = 0; c < RP * 8; c += 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(row + c));
                }
            }
        };
        load_batch(0, cur);
        load_batch(32, nxt);
        // per-mode row bases (shared-memory byte addresses when staged) and the swizzle phase of row 0
        uint32_t sbase[DO];
        const double* gbase[DO];
        int opar[DO];
    #pragma unroll
        for (int m = 0; m < DO; ++m) {
            gbase[m] = a.fac + a.fac_off[m];
            sbase[m] = (uint32_t)__cvta_generic_to_shared(g3s) + (uint32_t)((a.fac_off[m] - sbeg) * 8);
            opar[m] = (int)(((a.fac_off[m] - sbeg) / RP) & 3);
        }
        int rb = (int)(row_beg - p0), re = (int)(min(row_end, end) - p0);  // current row, relative
        const int ulo = (int)(beg - p0);  // the unit's first entry, relative

        // z of entry (kq) of the k-step at batch lane offset src
        auto build_z = [&](int src, double (&z)[NT], int32_t& wm, int32_t& ea) {
            int32_t ix[DO];
    #pragma unroll
            for (int m = 0; m < DO; ++m) ix[m] = __shfl_sync(0xffffffffu, cur[m], src);
            wm = __shfl_sync(0xffffffffu, cur[DO], src);  // 0 outside [beg, end)
            ea = ix[0];
    #pragma unroll
            for (int m = HOIST ? 1 : 0; m < DO; ++m) {
                const bool st = STAGE == 2 || (STAGE != 0 && m >= 1);  // this mode in shared memory
                const int swm = st ? sw(opar[m] + ix[m]) : 0;
    #pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    // logical chunk (columns 2 lc, 2 lc + 1), every mode in the same kq-rotated order
                    const int lc = CPL * g + (SF ? ((c + kq) & (CPL - 1)) : c);
                    double2 f;
                    if (st) {
                        const uint32_t ad = sbase[m] + (uint32_t)ix[m] * (RP * 8) + (uint32_t)((lc ^ swm) * 16);
                        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(f.x), "=d"(f.y) : "r"(ad));
                    } else {
                        f = __ldg(reinterpret_cast<const double2*>(gbase[m] + (int64_t)ix[m] * RP) + lc);
                    }
                    if (m == (HOIST ? 1 : 0)) {
                        z[2 * c] = f.x;
                        z[2 * c + 1] = f.y;
                    } else {
                        z[2 * c] *= f.x;
                        z[2 * c + 1] *= f.y;
                    }
                }
            }
            if constexpr (SF && CPL > 1) {  // logical chunk j sits in register chunk (j - kq) mod CPL
                if (kq & 1) {
                    const double t0 = z[2 * CPL - 2], t1 = z[2 * CPL - 1];
    #pragma unroll
                    for (int c = CPL - 1; c > 0; --c) {
                        z[2 * c] = z[2 * c - 2];
                        z[2 * c + 1] = z[2 * c - 1];
                    }
                    z[0] = t0;
                    z[1] = t1;
                }
                if (CPL == 4 && (kq & 2)) {
    #pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const double t0 = z[2 * c], t1 = z[2 * c + 1];
                        z[2 * c] = z[2 * c + 4];
                        z[2 * c + 1] = z[2 * c + 5];
                        z[2 * c + 4] = t0;
                        z[2 * c + 5] = t1;
                    }
                }
            }
        };
        // A = w z.  The FP64 multiplies share the pipe with DMMA, so a plan without multiplicities
        // (w = 1 on the unit's entries, 0 off them) masks with selects instead
        const bool weighted = a.mult != nullptr;
        auto mma_step = [&](const double (&z)[NT], int32_t w) {
            double zw[NT];
            const double wd = (double)w;
    #pragma unroll
            for (int t = 0; t < NT; ++t) zw[t] = weighted ? wd * z[t] : (w ? z[t] : 0.0);
            // tile pair uu goes to warp uu % TW of the team (accumulator uu / TW): every register index
            // is a compile-time constant
    #pragma unroll
            for (int ti = 0; ti < NT; ++ti)
    #pragma unroll
                for (int tj = ti; tj < NT; ++tj) {
                    const int uu = pair_index<NT>(ti, tj);
                    if (uu % TW == TWI) {
                        if constexpr (HOIST) dmma3(accm[uu / TW], zw[ti], z[tj]);
                        else dmma3(acc[uu / TW], zw[ti], z[tj]);
                    }
                }
        };
        // HOIST: the current run's first-mode index (-1: none yet) and its fold G += (a a') o M
        int cur_a = -1;
        auto fold = [&]() {
            if constexpr (HOIST) {
                if (cur_a >= 0) {
                    const double* ar = a.fac + a.fac_off[0] + (int64_t)cur_a * RP;
    #pragma unroll
                    for (int ti = 0; ti < NT; ++ti)
    #pragma unroll
                        for (int tj = ti; tj < NT; ++tj) {
                            const int uu = pair_index<NT>(ti, tj);
                            if (uu % TW != TWI) continue;
                            const double ai = __ldg(ar + NT * g + ti);
    #pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                const double s = ai * __ldg(ar + NT * (2 * kq + h) + tj);
                                acc[uu / TW][h] = fma(s, accm[uu / TW][h], acc[uu / TW][h]);
                                accm[uu / TW][h] = 0.0;
                            }
                        }
                }
            }
        };
        // the next non-empty row after the current one (it starts at the current row's end)
        auto next_row = [&]() {
            fold();
            cur_a = -1;
            flush(row);
            do {
                ++row;
                row_beg = a.row_ptr[row];
                row_end = a.row_ptr[row + 1];
            } while (row_end == row_beg);
            rb = (int)(row_beg - p0);
            re = (int)(min(row_end, end) - p0);
        };

        for (int P = (int)(beg - p0) & ~7; P < nrel; P += 8) {
            if (P >= b0 + 32) {
                b0 += 32;
    #pragma unroll
                for (int m = 0; m <= DO; ++m) cur[m] = nxt[m];
                load_batch(b0 + 32, nxt);
            }
            const int src = P - b0 + kq;
            if constexpr (HOIST) {  // one k-step at a time (registers: G and M accumulators)
    #pragma unroll 1
                for (int h = 0; h < 8; h += 4) {
                    const int Q = P + h;
                    if (Q >= nrel) break;
                    double z[NT];
                    int32_t wm, ea;
                    build_z(src + h, z, wm, ea);
                    if (Q >= rb && Q >= ulo && Q + 4 <= re && __all_sync(0xffffffffu, ea == cur_a)) {  // one run
                        mma_step(z, wm);
                        continue;
                    }
                    // a run or row end (or the unit's start / end) inside: once per run of each row
                    const int e = Q + kq;
                    for (;;) {
                        for (;;) {  // runs of the current row in this k-step, in ascending a
                            const bool in = e >= rb && e >= ulo && e < re;
                            if (__any_sync(0xffffffffu, in && ea == cur_a)) mma_step(z, in && ea == cur_a ? wm : 0);
                            const int nx = (int)__reduce_min_sync(0xffffffffu, (unsigned)(in && ea > cur_a ? ea : INT_MAX));
                            if (nx == INT_MAX) break;
                            fold();
                            cur_a = nx;
                        }
                        if (Q + 4 <= re || row_end >= end) break;
                        next_row();  // the step straddles the row end: the next row's entries of this step
                    }
                }
                continue;
            }
            if (P >= rb && P + 8 <= re) {  // both k-steps inside the current row
                double za[NT], zb[NT];
                int32_t wa, wb, ka, kb;
                build_z(src, za, wa, ka);
                build_z(src + 4, zb, wb, kb);
                mma_step(za, wa);
                mma_step(zb, wb);
                continue;
            }
            // a row end (or the unit's start / end) inside: one k-step at a time, one pass per row
    #pragma unroll 1
            for (int h = 0; h < 8; h += 4) {
                const int Q = P + h;
                if (Q >= nrel) break;
                double z[NT];
                int32_t wm, ea;
                build_z(src + h, z, wm, ea);
                const int e = Q + kq;
                for (;;) {
                    mma_step(z, (e >= rb && e < re) ? wm : 0);
                    if (Q + 4 <= re || row_end >= end) break;
                    next_row();  // the step straddles the row end: the next row's entries of this step
                }
            }
        }
        fold();
        flush(row);
    };
    switch (tw) {
        case 0: body(std::integral_constant<int, 0>{}); break;
        case 1: if constexpr (TW > 1) body(std::integral_constant<int, 1 % TW>{}); break;
        case 2: if constexpr (TW > 2) body(std::integral_constant<int, 2 % TW>{}); break;
        default: if constexpr (TW > 3) body(std::integral_constant<int, 3 % TW>{}); break;
    }
}

template <int RP, int DO, int TW>
void launch_g3(const GramArgs& a, int units, int stage, cudaStream_t s) {
    using C = G3<RP, TW>;
    const int grid = (units + C::TEAMS - 1) / C::TEAMS;
    const size_t fbytes = sizeof(double) * (size_t)(a.fac_total - (stage == 2 ? 0 : a.fac_off[1]));
    if (stage == 2) {
        auto kern = gram3_kernel<RP, DO, TW, 2>;
        func_attr_once((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        kern<<<grid, C::THREADS, fbytes, s>>>(a, units);
    } else if (stage == 1) {
        auto kern = gram3_kernel<RP, DO, TW, 1>;
        func_attr_once((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        kern<<<grid, C::THREADS, fbytes, s>>>(a, units);
    } else if (stage == 3) {
        if constexpr (DO == 2) {
            auto kern = gram3_kernel<RP, DO, TW, 3>;
            func_attr_once((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
            kern<<<grid, C::THREADS, fbytes, s>>>(a, units);
        } else {
            throw_invalid("gram build v3: the hoisted form needs a 3-way plan");
        }
    }
    CPHIFI_CHECK_LAUNCH();
}

template <int RP, int TW>
void launch_g3_do(const GramArgs& a, int units, int stage, cudaStream_t s) {
    switch (a.dother) {
        case 2: launch_g3<RP, 2, TW>(a, units, stage, s); break;
        case 3: launch_g3<RP, 3, TW>(a, units, stage, s); break;
        case 4: launch_g3<RP, 4, TW>(a, units, stage, s); break;
        default: throw_invalid("gram build v3: needs 2..4 other modes");
    }
}

// team width at RP = 64: 1 (8 warps per CTA, 255 registers) unless CPHIFI_GRAM3_TW=4 (16 warps, the
// 36 tile pairs split over 4 warps)
int g3_tw64() {
    static const int tw = [] {
        const char* e = std::getenv("CPHIFI_GRAM3_TW");
        return e && std::atoi(e) == 4 ? 4 : 1;
    }();
    return tw;
}

}  // namespace

// 2: all factors fit shared memory; 1: modes 1.. fit (mode 0 through L1); 0: v3 does not apply
int gram3_stage(int64_t rp, int dother, const GramArgs& a) {
    if (!(rp == 16 || rp == 32 || rp == 64) || dother < 2 || dother > 4) return 0;
    if (reinterpret_cast<uintptr_t>(a.fac) % 16) return 0;
    for (int m = 0; m < dother; ++m)
        if (a.fac_off[m] % 2) return 0;
    if (a.fac_total % 2) return 0;
    constexpr size_t cap = 220 * 1024;
    if (sizeof(double) * (size_t)a.fac_total <= cap) return 2;
    // (nothing staged — every factor row through L1 — measured 219 ms at config 4 against 62 for
    // k_gram.cu: not offered)
    if (sizeof(double) * (size_t)(a.fac_total - a.fac_off[1]) <= cap) return 1;
    return 0;
}

int gram3_units_per_sm(int64_t rp) {
    switch (rp) {
        case 16: return G3<16, 1>::TEAMS;
        case 32: return G3<32, 1>::TEAMS;
        default: return g3_tw64() == 4 ? G3<64, 4>::TEAMS : G3<64, 1>::TEAMS;
    }
}

void gram3_build(const GramArgs& a, int units, int stage, cudaStream_t s) {
    if (stage < 1 || stage > 3) throw_invalid("gram build v3: nothing staged");
    switch (a.rp) {
        case 16: launch_g3_do<16, 1>(a, units, stage, s); break;
        case 32: launch_g3_do<32, 1>(a, units, stage, s); break;
        case 64:
            if (g3_tw64() == 4) launch_g3_do<64, 4>(a, units, stage, s);
            else launch_g3_do<64, 1>(a, units, stage, s);
            break;
        default: throw_invalid("gram build v3: padded rank must be 16, 32 or 64");
    }
}

}  // namespace cphifi
