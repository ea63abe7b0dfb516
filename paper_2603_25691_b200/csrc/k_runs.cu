// k_runs.cu — the unaligned operator's q-pass as a run-structured streaming kernel (sm_100a).
//
// The reference computes, per operator application (observations.hpp:174-198 via
// unaligned.hpp:110-111, Zhat materialised by observations.hpp:142-158),
//     Yhat(i,:) = sum_{l: i_k(l)=i} w_l (Xhat(i,:) . z_l) z_l,   z_l = A_1(a_l,:) o A_2(b_l,:) o ...
// (w_l = multiplicity of a coalesced entry, 1 otherwise).  The plan is lexicographic in
// (i_k, a, b, ...), so the entries of a row form RUNS of equal first other index a.  Per run
// (i, a), with u = Xhat(i,:) o A_1(a,:) and t_l = A_2(b_l,:) o ... :
//     x_l = u . t_l,     v = sum_{l in run} w_l x_l t_l,     Yhat(i,:) += A_1(a,:) o v.
//
// Layout and schedule (one CTA per SM, 16 warps, everything else per warp):
//  * the per-observation factors (modes 2.. of the plan) live in shared memory for the whole
//    launch (one bulk copy per CTA); when they do not fit, the plan is cut into parts by row
//    blocks of the last mode (capi.cu build_run_parts) and each part stages its block;
//  * every warp owns a contiguous, equal-count range of plan entries (rows split between warps
//    are finished by the last-arriving warp summing the per-warp slots in warp order: no fp64
//    atomics, bit-reproducible) and walks it run by run using a precomputed run table
//    (run start, first other index);
//  * plan columns stream into a per-warp ring of CH-entry chunks by TMA bulk copies (mbarrier
//    completion), NCH chunks in flight; the A_1 row two runs ahead and the Xhat row of the next
//    row arrive the same way, so the inner loop never waits on L2;
//  * inside a run, 32 / G lane groups of G lanes take B consecutive entries each per step; a lane
//    holds RP / G columns of u, v and the entries' rows (odd lane groups read the two halves of
//    every pair of 2G-column chunks swapped, so the groups of one LDS.128 fill all 32 banks); a
//    dot is summed over its G lanes by a butterfly; each lane group folds its runs' A_1 o v into
//    its own partial row accumulator (registers), summed over the lane groups once per row.
//  All positions inside a warp's range are 32-bit offsets from its 16-byte aligned base.
#include <cstdlib>
#include <type_traits>

#include <climits>

#include "kernels.cuh"
#include "lanegroup.cuh"
#include "tma.cuh"

namespace cphifi {
namespace {

// ring chunks per warp: 4 of 64 entries, or 2 of 128 (the same ring bytes, half the chunk refills)
template <int CH>
__host__ __device__ constexpr int nch_of() { return CH >= 128 ? 2 : 4; }
constexpr int SMEM_CAP = 226 * 1024;  // opt-in maximum minus a little static shared memory

// CTA shape: NW warps (one CTA per SM), ring chunks of CH plan entries (CH x 4 B per column: one
// bulk copy each)
template <int RP, int DO, bool MULT, int NW, int CH>
struct Lay {
    static constexpr int NCOL = DO + (MULT ? 1 : 0);
    static constexpr int NCH = nch_of<CH>();
    static constexpr int NBAR = NCH + 3 + 1;       // ring chunks, A_1 slots, Xhat row
    static constexpr int WBUF = 4 * RP;            // doubles per warp: A_1 x 3, Xhat row
    static constexpr size_t bars = 128 + 8 * (size_t)NW * NBAR;
    static constexpr size_t wbuf = sizeof(double) * (size_t)NW * WBUF;
    static constexpr size_t ring = sizeof(int32_t) * (size_t)NW * NCH * NCOL * CH;
    static size_t bytes(int64_t sf_doubles) { return bars + wbuf + ring + sizeof(double) * (size_t)sf_doubles; }
};

__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

// Column of register pair t (VPL / 2 pairs) of lane gl: the pairs of a 2G-column chunk are
// [2 gl, 2 gl + 1]; odd lane groups take the chunks pairwise swapped (t ^ 1).
template <int G>
__device__ __forceinline__ int col_of(int t, int gl, int odd) {
    return 2 * (t ^ odd) * G + 2 * gl;
}
template <int G, int VPL>
__device__ __forceinline__ void lds_row(double (&v)[VPL], const double* row, int gl, int odd) {
#pragma unroll
    for (int t = 0; t < VPL / 2; ++t) {
        const double2 x = *reinterpret_cast<const double2*>(row + col_of<G>(t, gl, odd));
        v[2 * t] = x.x;
        v[2 * t + 1] = x.y;
    }
}

// VAR (bit mask, measured variants of the inner loop; 0 = the layout above):
//  RV_IDXS  plan indices of a 16-entry window read once per lane (one LDS.32: lanes 0-15 the
//           per-observation index, 16-31 the multiplicity) and handed to the entries by shuffles
//           instead of one broadcast LDS per entry and column (3-way coalesced plans);
//  RV_PRED  the last, partial step of a run loads only the rows of entries inside the run (lane
//           groups past the end skip their loads) instead of re-loading the run's last row;
//  RV_A1REG the run's A_1 row kept in registers from u = Xhat o A_1 to the fold (one row read per run
//           instead of two);
//  RV_XREG  the row's Xhat row kept in registers (read once per row instead of once per run).
//  RV_RHS   the right-hand side B instead of the operator: each entry's weight is its observed value
//           (RunsArgs::vals; summed over duplicates in a coalesced plan) — no dot with Xhat, no
//           reduction over the lane group, no multiplicity.
//  RV_S32   the step loop's shared-memory reads (plan indices, factor rows) through 32-bit shared
//           addresses computed once (ld.shared with explicit addresses) instead of generic pointers
//           the compiler converts (and, at 128 registers, re-derives) every step.
//  RV_CHUNKED the staging test once per stretch of landed entries instead of once per step.
//  RV_FOLDZ the run's A_1 row folded into every entry's row instead of into u and the run's sum: with
//           z' = A_1(a,:) o t the dot is Xhat(i,:) . z' and the row accumulator takes w x z' directly, so a
//           lane keeps the Xhat row (read once per ROW), the A_1 row (once per run) and the row
//           accumulator — the same registers as u, v and the accumulator — and a run reads one row
//           from shared memory instead of three (Xhat, A_1 for u, A_1 for the fold): 32 fewer
//           shared-memory wavefronts per run and warp for RP / G more multiplies per entry and lane.
constexpr int RV_IDXS = 1, RV_PRED = 2, RV_A1REG = 4, RV_XREG = 8, RV_RHS = 32, RV_S32 = 64, RV_CHUNKED = 128,
              RV_FOLDZ = 256;

template <int RP, int DO, bool MULT, int G, int B, bool PIPE, int NW, int CH, int VAR>
__global__ void __launch_bounds__(NW * 32, 1) runs_kernel(const RunsArgs a) {
    using L = Lay<RP, DO, MULT, NW, CH>;
    constexpr int NCH = nch_of<CH>();
    constexpr int RNW = NW, RING = NCH * CH;
    constexpr int VPL = RP / G, NCOL = L::NCOL, NGR = 32 / G, STEP = NGR * B;
    constexpr bool IDXS = (VAR & RV_IDXS) != 0, PRED = (VAR & RV_PRED) != 0, A1REG = (VAR & RV_A1REG) != 0,
                   XREG = (VAR & RV_XREG) != 0, RHS = (VAR & RV_RHS) != 0, S32 = (VAR & RV_S32) != 0,
                   FOLDZ = (VAR & RV_FOLDZ) != 0;
    static_assert(!RHS || (!PIPE && !IDXS), "RV_RHS: the plain step loop");
    static_assert(!FOLDZ || (!RHS && !A1REG && !XREG), "RV_FOLDZ: the operator loop");
    constexpr int WIN = MULT ? 16 : 32;  // RV_IDXS window (entries)
    static_assert(!IDXS || (DO == 2 && STEP <= WIN / 2), "RV_IDXS: 3-way plans, window >= 2 steps");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* cbar = reinterpret_cast<uint64_t*>(smem_raw);  // CTA: staged factors
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int g = lane / G, gl = lane % G;
    // the chunk swap: only when a lane group's LDS.128 covers less than 128 B (G < 8), and it needs
    // >= 2 pairs per lane
    const int odd = (G < 8 && VPL >= 4) ? (g & 1) : 0;
    uint64_t* wbar = reinterpret_cast<uint64_t*>(smem_raw + 128) + wid * L::NBAR;
    double* wb = reinterpret_cast<double*>(smem_raw + L::bars) + (size_t)wid * L::WBUF;
    double* a1s = wb;              // 3 x RP: A_1 rows of runs j, j+1, j+2 (slot j % 3)
    double* xrs = wb + 3 * RP;     // Xhat row of the current row
    int32_t* ring = reinterpret_cast<int32_t*>(smem_raw + L::bars + L::wbuf) + (size_t)wid * NCOL * RING;
    double* sfac = reinterpret_cast<double*>(smem_raw + L::bars + L::wbuf + L::ring);

    // staged per-observation factors: other modes 1 .. DO-1 (packed rows of RP doubles)
    int frows[DO];
#pragma unroll
    for (int m = 0; m < DO; ++m) frows[m] = (int)(((m + 1 < DO ? a.fac_off[m + 1] : a.fac_total) - a.fac_off[m]) / RP);
    if (tid == 0) {
        tma::mbar_init(cbar, 1);
        tma::fence_mbar_init();
        unsigned bytes = 0;
#pragma unroll
        for (int m = 1; m < DO; ++m) bytes += (unsigned)frows[m] * RP * 8;
        tma::mbar_expect_tx(cbar, bytes);
        int so = 0;
#pragma unroll
        for (int m = 1; m < DO; ++m) {
            const int tot = frows[m] * RP * 8;
            for (int b0 = 0; b0 < tot; b0 += 32768)
                tma::bulk_g2s(reinterpret_cast<unsigned char*>(sfac + so) + b0,
                              reinterpret_cast<const unsigned char*>(a.fac + a.fac_off[m]) + b0,
                              (unsigned)min(32768, tot - b0), cbar);
            so += frows[m] * RP;
        }
    }
    const double* fs[DO];  // fs[m]: staged rows of mode m (m >= 1)
    uint32_t fs_s[DO];     // (their shared-memory addresses, RV_S32)
    {
        int so = 0;
        fs[0] = nullptr;
        fs_s[0] = 0;
#pragma unroll
        for (int m = 1; m < DO; ++m) {
            fs[m] = sfac + so;
            fs_s[m] = tma::smem_u32(fs[m]);
            so += frows[m] * RP;
        }
    }
    __syncthreads();  // CTA barrier initialised before any warp waits on it

    const int w = blockIdx.x * RNW + wid;
    if (w >= a.warps) return;
    const int64_t e0 = a.warp_beg[w], e_end64 = a.warp_beg[w + 1];
    if (e0 >= e_end64) return;
    if (lane == 0) {
        for (int b = 0; b < L::NBAR; ++b) tma::mbar_init(wbar + b, 1);
        tma::fence_mbar_init();
    }
    __syncwarp();
    uint64_t* bar_ring = wbar;
    uint64_t* bar_a1 = wbar + NCH;
    uint64_t* bar_x = wbar + NCH + 3;

    // ---- ring of plan chunks: chunk j = relative entries [j CH, (j + 1) CH) ----------------------
    const int64_t cbase = e0 & ~(int64_t)3;  // 16-byte aligned column offsets
    const int rel_end = (int)(e_end64 - cbase);
    const int nchunks = (rel_end + CH - 1) / CH;
    const int32_t* gidx = a.idx + cbase;
    const int32_t* gmul = MULT ? a.mult + cbase : nullptr;
    int issued = 0, landed = 0;
    auto issue_chunk = [&](int j) {  // lane 0
        const int slot = j & (NCH - 1);
        tma::mbar_expect_tx(bar_ring + slot, (unsigned)(NCOL * CH * 4));
#pragma unroll
        for (int m = 0; m < DO; ++m)
            tma::bulk_g2s(ring + m * RING + slot * CH, gidx + (int64_t)m * a.ldq + j * CH, CH * 4, bar_ring + slot);
        if constexpr (MULT) tma::bulk_g2s(ring + DO * RING + slot * CH, gmul + j * CH, CH * 4, bar_ring + slot);
    };
    // chunks below the one holding `rel` are consumed: keep NCH chunks issued from there on, and
    // every chunk up to the one holding `last` landed.  The step loop calls it only when `last`
    // reaches past the landed entries or `rel` enters a chunk whose predecessor can be refilled.
    int land_lim = 0, refill_at = 0;  // entries < land_lim landed; rel >= refill_at frees a slot
    auto stage = [&](int rel, int last) {
        const int jlo = rel / CH;
        if (issued < nchunks && issued < jlo + NCH) {
            __syncwarp();
            const int upto = min(nchunks, jlo + NCH);
            if (lane == 0) {
                tma::fence_proxy_async();
                for (int j = issued; j < upto; ++j) issue_chunk(j);
            }
            issued = upto;
        }
        refill_at = issued < nchunks ? (issued - NCH + 1) * CH : INT_MAX;
        const int jhi = last / CH;
        while (landed <= jhi) {
            tma::mbar_wait(bar_ring + (landed & (NCH - 1)), (unsigned)((landed / NCH) & 1));
            ++landed;
        }
        land_lim = landed * CH;
    };
    // column `col` of the ring is a circular buffer of RING entries: entry rel sits at rel mod RING
    auto ring_at = [&](int rel, int col) -> int32_t { return ring[col * RING + (rel & (RING - 1))]; };
    const uint32_t ring_s = tma::smem_u32(ring);
    auto ring_at32 = [&](int rel, int col) -> int32_t {
        int32_t v;
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(ring_s + 4u * (unsigned)(col * RING + (rel & (RING - 1)))));
        return v;
    };

    // ---- runs, rows ------------------------------------------------------------------------
    int r = 0;  // runs and rows fit 32 bits (plans hold < 2^31 entries)
    const int nruns = (int)a.nruns;
    if (lane == 0) {  // largest r with run_start[r] <= e0
        int lo = 0, hi = nruns - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (a.run_start[mid] <= e0) lo = mid;
            else hi = mid - 1;
        }
        r = lo;
    }
    r = __shfl_sync(0xffffffffu, r, 0);
    const int r0 = r;
    int cur_row = (int)a.warp_rows[2 * w];
    const int first_row = cur_row;
    int row_end = (int)(min(a.row_ptr[cur_row + 1], e_end64) - cbase);
    // relative ends of runs r, r+1 (start of the run after), first other index of run r+2
    auto rel_of = [&](int k) { return (int)(min((int64_t)a.run_start[min(k, nruns)], e_end64) - cbase); };
    int rs1 = rel_of(r + 1), rs2 = rel_of(r + 2);
    int32_t i1_2 = r + 2 < nruns ? a.run_i1[r + 2] : 0;
    const double* fa1 = a.fac + a.fac_off[0];
    int xcnt = 0;  // Xhat-row loads issued (barrier phase)
    if (lane == 0) {
        tma::mbar_expect_tx(bar_x, RP * 8);
        tma::bulk_g2s(xrs, a.xhat_rm + (int64_t)cur_row * RP, RP * 8, bar_x);
        tma::mbar_expect_tx(bar_a1 + 0, RP * 8);
        tma::bulk_g2s(a1s, fa1 + (int64_t)a.run_i1[r] * RP, RP * 8, bar_a1 + 0);
        if (rs1 < rel_end) {
            tma::mbar_expect_tx(bar_a1 + 1, RP * 8);
            tma::bulk_g2s(a1s + RP, fa1 + (int64_t)a.run_i1[r + 1] * RP, RP * 8, bar_a1 + 1);
        }
        for (int j = 0; j < min(nchunks, NCH); ++j) issue_chunk(j);
    }
    issued = min(nchunks, NCH);
    refill_at = issued < nchunks ? CH : INT_MAX;
    tma::mbar_wait(cbar, 0);
    tma::mbar_wait(bar_x, 0);
    xcnt = 1;

    // one step: lane group g takes entries p + g B + b (b < B); FULL: all inside the run
    // a step in two halves so the next step's loads can be issued between them (software
    // pipelining: the loads of step k + 1 overlap the dot reduction and update of step k)
    double u[VPL], v[VPL], racc[VPL];  // racc: this lane's share of its lane group's row accumulator
    double a1r[A1REG ? VPL : 1], xr[XREG ? VPL : 1];
    double rv[B];  // RV_RHS: the step's entries' values
#pragma unroll
    for (int b = 0; b < B; ++b) rv[b] = 0.0;
#pragma unroll
    for (int k = 0; k < VPL; ++k) racc[k] = 0.0;
    if constexpr (XREG) lds_row<G, VPL>(xr, xrs, gl, odd);
    if constexpr (FOLDZ) lds_row<G, VPL>(u, xrs, gl, odd);  // RV_FOLDZ: u = the Xhat row, v = the run's A_1 row
    // RV_IDXS window: entries [wnd, wnd + WIN); lane l holds column 1 of entry wnd + (l % 16) (l < 16)
    // or the multiplicity (l >= 16) — WIN = 32 without multiplicities: column 1 of wnd + l
    int wnd = INT_MIN / 2, widx = 0;
    auto window = [&](int p) {  // before a step at p: [p, p + STEP) inside the window, landed
        if constexpr (IDXS) {
            if (p - wnd > WIN - STEP) {
                wnd = p;
                if (wnd + WIN > land_lim || wnd >= refill_at) stage(wnd, min(wnd + WIN, rel_end) - 1);
                const int e = wnd + (lane % WIN);
                widx = ring_at(e, (MULT && lane >= 16) ? DO : 1);
            }
        } else {
            if (p + STEP > land_lim || p >= refill_at) stage(p, p + STEP - 1);
        }
    };
    auto load = [&](int p, int rend, double (&z)[B][VPL], int (&mu)[B], auto full_tag) {
        constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
        for (int b = 0; b < B; ++b) {
            int ent = p + g * B + b;
            const bool ok = FULL || ent < rend;
            if constexpr (!FULL) ent = min(ent, rend - 1);
            const double* rows[DO];
            if constexpr (RHS) rv[b] = __ldg(a.vals + cbase + ent);
            if constexpr (IDXS) {
                rows[1] = fs[1] + __shfl_sync(0xffffffffu, widx, ent - wnd) * RP;
                if constexpr (MULT) mu[b] = __shfl_sync(0xffffffffu, widx, 16 + ent - wnd);
            } else if constexpr (!S32) {
#pragma unroll
                for (int m = 1; m < DO; ++m) rows[m] = fs[m] + ring_at(ent, m) * RP;
            }
            uint32_t rows_s[DO];
            if constexpr (S32 && !IDXS) {
#pragma unroll
                for (int m = 1; m < DO; ++m) rows_s[m] = fs_s[m] + (uint32_t)ring_at32(ent, m) * (RP * 8);
            }
            if (PRED && !FULL && !ok) {
#pragma unroll
                for (int k = 0; k < VPL; ++k) z[b][k] = 0.0;
                continue;
            }
            // t = A_2(b,:) o A_3(c,:) o ...: one pair of columns at a time (few live registers)
#pragma unroll
            for (int t = 0; t < VPL / 2; ++t) {
                const int c = col_of<G>(t, gl, odd);
                double2 x;
                if constexpr (S32 && !IDXS) {
                    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x.x), "=d"(x.y) : "r"(rows_s[1] + 8u * c));
                } else {
                    x = *reinterpret_cast<const double2*>(rows[1] + c);
                }
#pragma unroll
                for (int m = 2; m < DO; ++m) {
                    double2 f;
                    if constexpr (S32 && !IDXS) {
                        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(f.x), "=d"(f.y) : "r"(rows_s[m] + 8u * c));
                    } else {
                        f = *reinterpret_cast<const double2*>(rows[m] + c);
                    }
                    x.x *= f.x;
                    x.y *= f.y;
                }
                if constexpr (FOLDZ) {
                    x.x *= v[2 * t];
                    x.y *= v[2 * t + 1];
                }
                z[b][2 * t] = x.x;
                z[b][2 * t + 1] = x.y;
            }
            if constexpr (MULT && !IDXS) mu[b] = S32 ? ring_at32(ent, DO) : ring_at(ent, DO);
        }
    };
    auto dots = [&](const double (&z)[B][VPL], double (&d)[B]) {
        if constexpr (RHS) {
#pragma unroll
            for (int b = 0; b < B; ++b) d[b] = rv[b];
            return;
        }
#pragma unroll
        for (int b = 0; b < B; ++b) {
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int k = 0; k < VPL; k += 2) {
                s0 = fma(u[k], z[b][k], s0);
                s1 = fma(u[k + 1], z[b][k + 1], s1);
            }
            d[b] = s0 + s1;
        }
    };
    auto finish = [&](int p, int rend, const double (&z)[B][VPL], const int (&mu)[B], double (&d)[B], auto full_tag) {
        constexpr bool FULL = decltype(full_tag)::value;
        if constexpr (!RHS) group_reduce<B, G>(d, lane);
#pragma unroll
        for (int b = 0; b < B; ++b) {
            double s = d[b];
            if constexpr (MULT && !RHS) s *= (double)mu[b];
            if constexpr (!FULL) s = p + g * B + b < rend ? s : 0.0;
#pragma unroll
            for (int k = 0; k < VPL; ++k) {
                if constexpr (FOLDZ) racc[k] = fma(s, z[b][k], racc[k]);
                else v[k] = fma(s, z[b][k], v[k]);
            }
        }
    };

    int pos = (int)(e0 - cbase);
    while (pos < rel_end) {
        const int jl = (int)(r - r0);  // local run counter: A_1 slot jl % 3, phase jl / 3
        const int rend = rs1;
        tma::mbar_wait(bar_a1 + jl % 3, (unsigned)((jl / 3) & 1));
        // the A_1 row two runs ahead goes into the slot run jl - 1 used
        if (lane == 0 && rs2 < rel_end) {
            const int sl = (jl + 2) % 3;
            tma::fence_proxy_async();  // generic reads of that slot (run jl - 1) precede the async write
            tma::mbar_expect_tx(bar_a1 + sl, RP * 8);
            tma::bulk_g2s(a1s + sl * RP, fa1 + (int64_t)i1_2 * RP, RP * 8, bar_a1 + sl);
        }
        const double* a1 = a1s + (jl % 3) * RP;
        if constexpr (FOLDZ) {
            lds_row<G, VPL>(v, a1, gl, odd);
        } else if constexpr (XREG) {
#pragma unroll
            for (int k = 0; k < VPL; ++k) u[k] = xr[k];
        } else if constexpr (!RHS) {
            lds_row<G, VPL>(u, xrs, gl, odd);  // u = Xhat(i,:) o A_1(a,:), one pair at a time
        }
        if constexpr (A1REG) lds_row<G, VPL>(a1r, a1, gl, odd);
        if constexpr (!FOLDZ) {
#pragma unroll
            for (int t = 0; t < VPL / 2; ++t) {
                double2 x;
                if constexpr (A1REG) x = make_double2(a1r[2 * t], a1r[2 * t + 1]);
                else x = *reinterpret_cast<const double2*>(a1 + col_of<G>(t, gl, odd));
                u[2 * t] *= x.x;
                u[2 * t + 1] *= x.y;
                v[2 * t] = 0.0;
                v[2 * t + 1] = 0.0;
            }
        }
        // the run table one run further (consumed at the next run start)
        const int rs3 = rel_of(r + 3);
        const int32_t i1_3 = r + 3 < nruns ? a.run_i1[r + 3] : 0;

        int p = pos;
        {
            double za[B][VPL], zb[B][VPL], d[B];
            int ma[B], mb[B];
            if constexpr (!PIPE && (VAR & RV_CHUNKED)) {
                // the staging test once per stretch of landed entries, not once per step: every step
                // starting at or before pend is inside the run, landed and before the next refill
                while (p + STEP <= rend) {
                    window(p);
                    const int pend = min(min(rend, land_lim) - STEP, refill_at - 1);
                    for (; p <= pend; p += STEP) {
                        load(p, rend, za, ma, std::true_type{});
                        dots(za, d);
                        finish(p, rend, za, ma, d, std::true_type{});
                    }
                }
            } else if constexpr (!PIPE) {
                for (; p + STEP <= rend; p += STEP) {
                    window(p);
                    load(p, rend, za, ma, std::true_type{});
                    dots(za, d);
                    finish(p, rend, za, ma, d, std::true_type{});
                }
            }
            bool have = PIPE && p + STEP <= rend;
            if (have) {
                window(p);
                load(p, rend, za, ma, std::true_type{});
            }
            while (have) {  // unrolled by two: za / zb alternate as current / next
                dots(za, d);
                int pn = p + STEP;
                bool hn = pn + STEP <= rend;
                if (hn) {
                    window(pn);
                    load(pn, rend, zb, mb, std::true_type{});
                }
                finish(p, rend, za, ma, d, std::true_type{});
                p = pn;
                have = hn;
                if (!have) break;
                dots(zb, d);
                pn = p + STEP;
                hn = pn + STEP <= rend;
                if (hn) {
                    window(pn);
                    load(pn, rend, za, ma, std::true_type{});
                }
                finish(p, rend, zb, mb, d, std::true_type{});
                p = pn;
                have = hn;
            }
            if (p < rend) {  // the last, partial step
                if constexpr (IDXS) window(p);
                else if (rend > land_lim || p >= refill_at) stage(p, rend - 1);
                load(p, rend, za, ma, std::false_type{});
                dots(za, d);
                finish(p, rend, za, ma, d, std::false_type{});
            }
        }
        // run complete: this lane's share of A_1(a,:) o v folded into its row accumulator (lane
        // groups keep separate partial rows; they are summed once per row, at the flush)
        if constexpr (!FOLDZ) {
#pragma unroll
            for (int t = 0; t < VPL / 2; ++t) {
                double2 aa;
                if constexpr (A1REG) aa = make_double2(a1r[2 * t], a1r[2 * t + 1]);
                else aa = *reinterpret_cast<const double2*>(a1 + col_of<G>(t, gl, odd));
                racc[2 * t] = fma(aa.x, v[2 * t], racc[2 * t]);
                racc[2 * t + 1] = fma(aa.y, v[2 * t + 1], racc[2 * t + 1]);
            }
        }
        pos = rend;
        ++r;
        rs1 = rs2;
        rs2 = rs3;
        i1_2 = i1_3;
        if (pos == row_end || pos == rel_end) {  // flush the row accumulator
            // unswizzled column order, then the sum over the lane groups (xor butterfly: every lane
            // ends with the same sum); lane group 0 holds the row, RP / G columns per lane
            if (odd) {
#pragma unroll
                for (int t = 0; t + 1 < VPL / 2; t += 2) {
                    const double x0 = racc[2 * t], x1 = racc[2 * t + 1];
                    racc[2 * t] = racc[2 * t + 2];
                    racc[2 * t + 1] = racc[2 * t + 3];
                    racc[2 * t + 2] = x0;
                    racc[2 * t + 3] = x1;
                }
            }
#pragma unroll
            for (int k = 0; k < VPL; ++k)
#pragma unroll
                for (int off = G; off < 32; off <<= 1) racc[k] += __shfl_xor_sync(0xffffffffu, racc[k], off);
            const int ncta = a.row_nw[cur_row];
            if (ncta <= 1) {
                if (g == 0) {
                    double* dst = a.yhat_rm + (int64_t)cur_row * RP;
#pragma unroll
                    for (int t = 0; t < VPL / 2; ++t) {
                        double2* d2 = reinterpret_cast<double2*>(dst + col_of<G>(t, gl, 0));
                        double2 o = make_double2(racc[2 * t], racc[2 * t + 1]);
                        if (a.accumulate) {
                            const double2 cur = *d2;
                            o.x += cur.x;
                            o.y += cur.y;
                        }
                        *d2 = o;
                    }
                }
            } else {  // a row shared with neighbouring warps: slot, then the last arriver sums
                double* slot = (cur_row == first_row ? a.slot_a : a.slot_b) + (int64_t)w * RP;
                if (g == 0) {
#pragma unroll
                    for (int t = 0; t < VPL / 2; ++t)
                        *reinterpret_cast<double2*>(slot + col_of<G>(t, gl, 0)) = make_double2(racc[2 * t], racc[2 * t + 1]);
                }
                __syncwarp();
                unsigned last = 0;
                if (lane == 0) {
                    __threadfence();
                    last = atom_add_acqrel(a.rowcnt + cur_row, 1u) == (unsigned)ncta - 1;
                    if (last) a.rowcnt[cur_row] = 0;
                }
                last = __shfl_sync(0xffffffffu, last, 0);
                if (last) {
                    const int u0 = a.row_first_w[cur_row];
                    for (int c = lane; c < RP; c += 32) {
                        double s = a.warp_rows[2 * u0] == cur_row ? __ldcg(a.slot_a + (int64_t)u0 * RP + c)
                                                                   : __ldcg(a.slot_b + (int64_t)u0 * RP + c);
                        for (int uu = u0 + 1; uu < u0 + ncta; ++uu) s += __ldcg(a.slot_a + (int64_t)uu * RP + c);
                        double* dst = a.yhat_rm + (int64_t)cur_row * RP + c;
                        *dst = a.accumulate ? *dst + s : s;
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < VPL; ++k) racc[k] = 0.0;
            if (pos < rel_end) {  // next row with entries, its Xhat row
                int64_t re;
                do {
                    ++cur_row;
                    re = a.row_ptr[cur_row + 1];
                } while (re - cbase <= pos);
                row_end = (int)(min(re, e_end64) - cbase);
                __syncwarp();
                if (lane == 0) {
                    tma::fence_proxy_async();
                    tma::mbar_expect_tx(bar_x, RP * 8);
                    tma::bulk_g2s(xrs, a.xhat_rm + (int64_t)cur_row * RP, RP * 8, bar_x);
                }
                tma::mbar_wait(bar_x, (unsigned)(xcnt & 1));
                ++xcnt;
                if constexpr (XREG) lds_row<G, VPL>(xr, xrs, gl, odd);
                if constexpr (FOLDZ) lds_row<G, VPL>(u, xrs, gl, odd);
            }
        }
        __syncwarp();
    }
}

template <int RP, int DO, bool MULT, int G, int B, bool PIPE, int NW = 16, int CH = 64, int VAR = 0>
void launch4(const RunsArgs& a, int64_t sf, cudaStream_t s) {
    auto kern = runs_kernel<RP, DO, MULT, G, B, PIPE, NW, CH, VAR>;
    const size_t smem = Lay<RP, DO, MULT, NW, CH>::bytes(sf);
    func_attr_once((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_CAP);
    const int grid = (a.warps + NW - 1) / NW;
    kern<<<grid, NW * 32, smem, s>>>(a);
    CPHIFI_CHECK_LAUNCH();
}

// lanes per entry G, entries per lane group per step B, and whether the next step's loads are
// issued before the current step's reduction (PIPE: two steps' rows live in registers), measured
// per padded rank (profiles/prof_stream.py; config 4: 8.3 ms vs 9.4 pipelined with B = 1;
// config 3: 4.2 ms vs 5.3 with G = 8 and 4.7 pipelined): RP = 64: G = 8, B = 2; RP = 32: G = 4,
// B = 2; RP = 16: G = 4, B = 2, none pipelined.  CPHIFI_RUNS_LAYOUT=1 / 2 / 3 select the alternatives.
int runs_layout() {
    static const int layout = [] {
        const char* e = std::getenv("CPHIFI_RUNS_LAYOUT");
        return e ? std::atoi(e) : 0;
    }();
    return layout;
}
// inner-loop variant (RV_* bits; + 16: 12 warps per CTA, up to 168 registers) of the G = 8, B = 2
// layout at RP = 64 (CPHIFI_RUNS_VAR)
// The default inner loop: 32-bit shared addresses + loads of in-run entries only in the partial
// step (RV_S32 | RV_PRED; config 4: run kernel 4.01 -> 3.87 ms per application, either alone no
// faster) + the staging test once per landed stretch (RV_CHUNKED: -> 3.66 ms) —
// profiles/round2/runs_variants_config4.txt.  CPHIFI_RUNS_VAR selects another (0: the plain loop).
constexpr int RV_DEFAULT = RV_S32 | RV_PRED | RV_CHUNKED;
// ... and, for coalesced 3-way plans at RP = 64 (config 4: ~32-entry runs per part), the A_1 row folded
// into the entries' rows (RV_FOLDZ, all-entry loads in the partial step): run kernel 3.62 -> 3.53 ms,
// application 174.4 -> 180.5 matvecs/s; no spills at 128 registers (the former default spilled 40 B).
// CPHIFI_RUNS_VAR=194 selects the former default.
constexpr int RV_DEFAULT_FOLDZ = RV_S32 | RV_CHUNKED | RV_FOLDZ;
constexpr int DEF_CH = 128;  // with 2 chunks in flight (nch_of): config 4 3.66 -> 3.62 ms
int runs_var() {
    static const int var = [] {
        const char* e = std::getenv("CPHIFI_RUNS_VAR");
        return e ? std::atoi(e) : RV_DEFAULT;
    }();
    return var;
}
bool runs_var_chosen() {
    static const bool set = std::getenv("CPHIFI_RUNS_VAR") != nullptr;
    return set;
}

template <int RP, int DO, bool MULT>
void launch_var(const RunsArgs& a, int64_t sf, cudaStream_t s) {
    if constexpr (RP == 64 && DO == 2 && MULT) {
        if (!runs_var_chosen()) {
            launch4<RP, DO, MULT, 8, 2, false, 16, DEF_CH, RV_DEFAULT_FOLDZ>(a, sf, s);
            return;
        }
        switch (runs_var()) {
            case 1: launch4<RP, DO, MULT, 8, 2, false, 16, 64, 1>(a, sf, s); return;
            case 2: launch4<RP, DO, MULT, 8, 2, false, 16, 64, 2>(a, sf, s); return;
            case 3: launch4<RP, DO, MULT, 8, 2, false, 16, 64, 3>(a, sf, s); return;
            case 4: launch4<RP, DO, MULT, 8, 2, false, 16, 64, 4>(a, sf, s); return;
            case 7: launch4<RP, DO, MULT, 8, 2, false, 16, 64, 7>(a, sf, s); return;
            case 20: launch4<RP, DO, MULT, 8, 2, false, 12, 64, 4>(a, sf, s); return;
            case 23: launch4<RP, DO, MULT, 8, 2, false, 12, 64, 7>(a, sf, s); return;
            case 28: launch4<RP, DO, MULT, 8, 2, false, 12, 64, 12>(a, sf, s); return;
            case 31: launch4<RP, DO, MULT, 8, 2, false, 12, 64, 15>(a, sf, s); return;
            case 80: launch4<RP, DO, MULT, 8, 2, true, 12, 64, 0>(a, sf, s); return;
            case 81: launch4<RP, DO, MULT, 8, 2, true, 8, 64, 0>(a, sf, s); return;
            case 82: launch4<RP, DO, MULT, 8, 4, false, 8, 64, 0>(a, sf, s); return;
            case 83: launch4<RP, DO, MULT, 8, 3, false, 12, 64, 0>(a, sf, s); return;
            case 84: launch4<RP, DO, MULT, 8, 4, false, 12, 64, 0>(a, sf, s); return;
            case 0: launch4<RP, DO, MULT, 8, 2, false, 16, 64, 0>(a, sf, s); return;
            case 64: launch4<RP, DO, MULT, 8, 2, false, 16, 64, RV_S32>(a, sf, s); return;
            case 70: launch4<RP, DO, MULT, 8, 2, false, 16, 64, RV_S32 | RV_PRED | RV_A1REG>(a, sf, s); return;
            case 74: launch4<RP, DO, MULT, 8, 2, false, 16, 64, RV_S32 | RV_PRED | RV_XREG>(a, sf, s); return;
            case 86: launch4<RP, DO, MULT, 8, 2, false, 12, 64, RV_S32 | RV_PRED | RV_A1REG | RV_XREG>(a, sf, s); return;
            case 66: launch4<RP, DO, MULT, 8, 2, false, 16, 64, RV_S32 | RV_PRED>(a, sf, s); return;
            case 1194: launch4<RP, DO, MULT, 8, 2, false, 16, 64, RV_DEFAULT>(a, sf, s); return;  // 4 x 64
            // the default inner loop with one entry per lane group and step (2 x 128 ring; 119
            // registers, no spills): 3.91 vs 3.62 ms at config 4.  (G = 4 with B = 1 / 2 and G = 8
            // with B = 3 spill 204-664 B at 128 registers.)
            case 4099: launch4<RP, DO, MULT, 8, 1, false, 16, DEF_CH, RV_DEFAULT>(a, sf, s); return;
            case 450: launch4<RP, DO, MULT, 8, 2, false, 16, DEF_CH, RV_DEFAULT | RV_FOLDZ>(a, sf, s); return;
            case 451: launch4<RP, DO, MULT, 8, 3, false, 16, DEF_CH, RV_DEFAULT | RV_FOLDZ>(a, sf, s); return;
            case 452: launch4<RP, DO, MULT, 8, 1, false, 16, DEF_CH, RV_DEFAULT | RV_FOLDZ>(a, sf, s); return;
            case 453: launch4<RP, DO, MULT, 8, 2, false, 16, DEF_CH, RV_DEFAULT_FOLDZ>(a, sf, s); return;
            case 454: launch4<RP, DO, MULT, 8, 1, true, 16, DEF_CH, RV_S32 | RV_FOLDZ>(a, sf, s); return;
            case 460: launch4<RP, DO, MULT, 8, 2, false, 16, 64, RV_IDXS | RV_FOLDZ>(a, sf, s); return;
            case 456: launch4<RP, DO, MULT, 16, 4, false, 20, 32, RV_FOLDZ>(a, sf, s); return;
            case 457: launch4<RP, DO, MULT, 16, 2, false, 24, 32, RV_FOLDZ>(a, sf, s); return;
            case 458: launch4<RP, DO, MULT, 16, 4, false, 24, 32, RV_FOLDZ>(a, sf, s); return;
            case 459: launch4<RP, DO, MULT, 16, 2, false, 20, 32, RV_FOLDZ>(a, sf, s); return;
            case 455: launch4<RP, DO, MULT, 8, 2, true, 16, DEF_CH, RV_S32 | RV_FOLDZ>(a, sf, s); return;
            default: break;
        }
    }
    if (runs_var() == 0) launch4<RP, DO, MULT, 8, 2, false, 16, 64, 0>(a, sf, s);
    else launch4<RP, DO, MULT, 8, 2, false, 16, DEF_CH, RV_DEFAULT>(a, sf, s);
}

template <int RP, int DO, bool MULT>
void launch3(const RunsArgs& a, int64_t sf, cudaStream_t s) {
    if (a.vals) {  // the right-hand side B, on the default layout
        if constexpr (RP == 64) launch4<RP, DO, MULT, 8, 2, false, 16, 64, RV_RHS>(a, sf, s);
        else launch4<RP, DO, MULT, 4, 2, false, 16, 64, RV_RHS>(a, sf, s);
        return;
    }
    const int lay = runs_layout();
    if constexpr (RP == 64) {
        if (lay == 1) launch4<RP, DO, MULT, 8, 1, true>(a, sf, s);
        else if (lay == 3) launch4<RP, DO, MULT, 16, 4, false, 20, 32>(a, sf, s);
        else launch_var<RP, DO, MULT>(a, sf, s);
    } else if constexpr (RP == 32) {
        if (lay == 1) launch4<RP, DO, MULT, 8, 2, false>(a, sf, s);
        else if (lay == 2) launch4<RP, DO, MULT, 4, 1, true>(a, sf, s);
        else if (runs_var() == 0) launch4<RP, DO, MULT, 4, 2, false>(a, sf, s);
        else if (runs_var_chosen() && runs_var() == 448) launch4<RP, DO, MULT, 4, 2, false, 16, DEF_CH, RV_DEFAULT_FOLDZ>(a, sf, s);
        else launch4<RP, DO, MULT, 4, 2, false, 16, DEF_CH, RV_DEFAULT>(a, sf, s);
    } else {
        if (runs_var() == 0) launch4<RP, DO, MULT, 4, 2, false>(a, sf, s);
        else launch4<RP, DO, MULT, 4, 2, false, 16, DEF_CH, RV_DEFAULT>(a, sf, s);
    }
}

template <int RP, int DO>
void launch2(const RunsArgs& a, int64_t sf, cudaStream_t s) {
    if (a.mult) launch3<RP, DO, true>(a, sf, s);
    else launch3<RP, DO, false>(a, sf, s);
}

template <int RP>
void launch1(const RunsArgs& a, int64_t sf, cudaStream_t s) {
    switch (a.dother) {
        case 2: launch2<RP, 2>(a, sf, s); break;
        case 3: launch2<RP, 3>(a, sf, s); break;
        case 4: launch2<RP, 4>(a, sf, s); break;
        default: throw_invalid("runs scatter-gather: needs 2..4 other modes");
    }
}

}  // namespace

bool runs_supported(int64_t rp, int dother) { return (rp == 16 || rp == 32 || rp == 64) && dother >= 2 && dother <= 4; }

// the CTA shape the launch picks for padded rank rp (layout 3: 24 warps, 32-entry chunks at RP 64)
// (layout 3 trades registers for warps: G = 16 lanes per entry, 20 warps, 32-entry chunks — measured
// 4.79 ms against 4.01 for the 16-warp G = 8 layout at config 4; 24 warps with B = 4 / 2: 5.76 / 5.08)
static int shape_nw(int64_t rp) {
    if (rp == 64 && runs_layout() == 3) return 20;
    if (rp != 64 || runs_layout() != 0) return 16;
    const int v = runs_var();
    if (v == 81 || v == 82) return 8;
    if (v == 456 || v == 459) return 20;
    if (v == 457 || v == 458) return 24;
    return (v & 16) || v == 80 || v == 83 || v == 84 || v == 86 ? 12 : 16;
}
static int shape_ch(int64_t rp) {
    if (rp == 64 && runs_layout() == 3) return 32;
    if (runs_layout() != 0) return 64;
    const int v = runs_var();
    if (v >= 456 && v <= 459) return 32;
    return (v == RV_DEFAULT || v >= 4096 || (v >= 448 && v <= 455)) ? DEF_CH : 64;
}

size_t runs_smem_bytes(int64_t rp, int dother, bool mult, int64_t sf_doubles) {
    const size_t ncol = (size_t)dother + (mult ? 1 : 0), nw = (size_t)shape_nw(rp), ch = (size_t)shape_ch(rp);
    const size_t nch = ch >= 128 ? 2 : 4;
    return 128 + 8 * nw * (nch + 4) + sizeof(double) * nw * 4 * rp + sizeof(int32_t) * nw * nch * ncol * ch +
           sizeof(double) * (size_t)sf_doubles;
}

size_t runs_smem_cap() { return SMEM_CAP; }
int runs_warps_per_sm(int64_t rp) { return shape_nw(rp); }
int runs_chunk(int64_t rp) { return shape_ch(rp); }

void runs_scatter_gather(const RunsArgs& a, int64_t sf_doubles, cudaStream_t s) {
    if (runs_smem_bytes(a.rp, a.dother, a.mult != nullptr, sf_doubles) > SMEM_CAP)
        throw_invalid("runs scatter-gather: staged factors exceed shared memory");
    switch (a.rp) {
        case 16: launch1<16>(a, sf_doubles, s); break;
        case 32: launch1<32>(a, sf_doubles, s); break;
        case 64: launch1<64>(a, sf_doubles, s); break;
        default: throw_invalid("runs scatter-gather: padded rank must be 16, 32 or 64");
    }
}

}  // namespace cphifi
