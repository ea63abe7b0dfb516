// k_xruns.cu — the q-pass of 3-way coalesced plans with steps that cross run boundaries (sm_100a).
//
// Same sum as k_runs.cu (observations.hpp:174-198 via unaligned.hpp:110-111): per run (i, a) of
// the lexicographic plan, u = Xhat(i,:) o A_1(a,:), x_l = u . A_2(b_l,:), v = sum_l w_l x_l A_2(b_l,:),
// Yhat(i,:) += A_1(a,:) o v.  In k_runs.cu the whole warp walks one run at a time: with the ~28-entry
// runs of config 4's factor-block parts that costs a run start (A_1 row, u), a fold and a partial last
// step per run — 45 % of the kernel's instructions (ncu source view, profiles/round2).  Here:
//  * every run of the part's plan is padded to an even length with a zero-multiplicity entry
//    (pad_runs_even, called by capi.cu build_run_parts), and every warp range starts at an even position, so the two entries a
//    lane group takes per step always belong to one run;
//  * a step covers 8 consecutive entries of the row whatever runs they belong to: each of the 4 lane
//    groups keeps its OWN run state (u, v) and switches run when its pair enters a new one — fold
//    A_1(a_old,:) o v into its row accumulator, u = Xhat o A_1(a_new,:), v = 0 — so runs cost a
//    switch per lane group instead of a warp-wide run start, and no step is partial inside a row;
//  * run starts are flagged in bit 30 of the multiplicity column; a lane group's run is the warp's
//    running run count plus a popcount of the flags before its pair (the index window: lanes 0-15
//    hold the b index, 16-31 the flagged multiplicity of 16 entries, handed out by shuffles);
//  * A_1 rows arrive by TMA in a per-warp ring of NS slots indexed by run number, issued up to
//    NS - 1 runs past the oldest run a lane group still holds (the folds read the old slots before
//    the ring moves on).
// Rows stay warp-wide: a step never crosses a row end, and at a row end the lane groups' partial
// rows are summed and written exactly as in k_runs.cu (split rows by the last-arriving warp, in warp
// order: deterministic).  Equal to k_runs.cu up to the rounding of the per-lane-group sums.
//
// MEASURED SLOWER, opt-in (CPHIFI_XRUNS=1): config 4, ncu one launch 2.41 ms against 2.03 ms for
// k_runs.cu (application 6.93 vs 6.18 ms).  It removes the per-run work as intended, but 42 % of the
// steps carry a lane-group switch (~84 instructions: fold, u, the slot ring), the index window and
// flag bookkeeping add ~30 instructions per step, and the two step paths cost register moves at 128
// registers: 1.53e9 instructions per launch against 1.14e9 (profiles/round2/runs_variants_config4.txt).
#include <climits>

#include <cub/cub.cuh>

#include "kernels.cuh"
#include "lanegroup.cuh"
#include "tma.cuh"

namespace cphifi {
namespace {

constexpr int XNCH = 4;                // ring chunks per warp
constexpr int XNS = 6;                 // A_1 row slots per warp
constexpr int XSMEM_CAP = 226 * 1024;
constexpr unsigned XFLAG = 1u << 30;   // run start, in the multiplicity column

template <int RP, int NW, int CH>
struct XLay {
    static constexpr int NBAR = XNCH + XNS + 1;  // ring chunks, A_1 slots, Xhat row
    static constexpr int WBUF = (XNS + 1) * RP;  // doubles per warp
    static constexpr size_t bars = (128 + 8 * (size_t)NW * NBAR + 127) / 128 * 128;
    static constexpr size_t wbuf = sizeof(double) * (size_t)NW * WBUF;
    static constexpr size_t ring = sizeof(int32_t) * (size_t)NW * XNCH * 2 * CH;
    static size_t bytes(int64_t sf) { return bars + wbuf + ring + sizeof(double) * (size_t)sf; }
};

__device__ __forceinline__ unsigned xatom_add_acqrel(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

template <int VPL>
__device__ __forceinline__ void lds_cols(double (&v)[VPL], const double* row, int gl) {
#pragma unroll
    for (int t = 0; t < VPL / 2; ++t) {
        const double2 x = *reinterpret_cast<const double2*>(row + 16 * t + 2 * gl);
        v[2 * t] = x.x;
        v[2 * t + 1] = x.y;
    }
}

template <int RP, int NW, int CH>
__global__ void __launch_bounds__(NW * 32, 1) xruns_kernel(const RunsArgs a) {
    using L = XLay<RP, NW, CH>;
    constexpr int G = 8, B = 2, VPL = RP / G, STEP = 8, RING = XNCH * CH, NS = XNS;
    static_assert(RP == 64, "xruns: 8 lanes x 8 columns per entry");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* cbar = reinterpret_cast<uint64_t*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int g = lane / G, gl = lane % G;
    uint64_t* wbar = reinterpret_cast<uint64_t*>(smem_raw + 128) + wid * L::NBAR;
    double* a1s = reinterpret_cast<double*>(smem_raw + L::bars) + (size_t)wid * L::WBUF;  // NS slots
    double* xrs = a1s + NS * RP;
    int32_t* ring = reinterpret_cast<int32_t*>(smem_raw + L::bars + L::wbuf) + (size_t)wid * 2 * RING;
    double* sfac = reinterpret_cast<double*>(smem_raw + L::bars + L::wbuf + L::ring);

    // the part's block of A_2 rows, staged once per CTA
    const int frows = (int)((a.fac_total - a.fac_off[1]) / RP);
    if (tid == 0) {
        tma::mbar_init(cbar, 1);
        tma::fence_mbar_init();
        const unsigned tot = (unsigned)frows * RP * 8;
        tma::mbar_expect_tx(cbar, tot);
        for (unsigned b0 = 0; b0 < tot; b0 += 32768)
            tma::bulk_g2s(reinterpret_cast<unsigned char*>(sfac) + b0,
                          reinterpret_cast<const unsigned char*>(a.fac + a.fac_off[1]) + b0, min(32768u, tot - b0), cbar);
    }
    __syncthreads();

    const int w = blockIdx.x * NW + wid;
    if (w >= a.warps) return;
    const int64_t e0 = a.warp_beg[w], e_end64 = a.warp_beg[w + 1];
    if (e0 >= e_end64) return;
    if (lane == 0) {
        for (int b = 0; b < L::NBAR; ++b) tma::mbar_init(wbar + b, 1);
        tma::fence_mbar_init();
    }
    __syncwarp();
    uint64_t* bar_ring = wbar;
    uint64_t* bar_a1 = wbar + XNCH;
    uint64_t* bar_x = wbar + XNCH + NS;

    // ---- ring of plan chunks (as k_runs.cu): columns b (rebased) and flagged multiplicity ----------
    const int64_t cbase = e0 & ~(int64_t)3;
    const int rel_end = (int)(e_end64 - cbase);
    const int nchunks = (rel_end + CH - 1) / CH;
    const int32_t* gb = a.idx + (int64_t)1 * a.ldq + cbase;
    const int32_t* gm = a.mult + cbase;
    int issued = 0, landed = 0, land_lim = 0, refill_at = 0;
    auto issue_chunk = [&](int j) {  // lane 0
        const int slot = j & (XNCH - 1);
        tma::mbar_expect_tx(bar_ring + slot, (unsigned)(2 * CH * 4));
        tma::bulk_g2s(ring + slot * CH, gb + j * CH, CH * 4, bar_ring + slot);
        tma::bulk_g2s(ring + RING + slot * CH, gm + j * CH, CH * 4, bar_ring + slot);
    };
    auto stage = [&](int rel, int last) {
        const int jlo = rel / CH;
        if (issued < nchunks && issued < jlo + XNCH) {
            __syncwarp();
            const int upto = min(nchunks, jlo + XNCH);
            if (lane == 0) {
                tma::fence_proxy_async();
                for (int j = issued; j < upto; ++j) issue_chunk(j);
            }
            issued = upto;
        }
        refill_at = issued < nchunks ? (issued - XNCH + 1) * CH : INT_MAX;
        const int jhi = last / CH;
        while (landed <= jhi) {
            tma::mbar_wait(bar_ring + (landed & (XNCH - 1)), (unsigned)((landed / XNCH) & 1));
            ++landed;
        }
        land_lim = landed * CH;
    };

    // ---- run table: the warp's first run, A_1 rows of upcoming runs by TMA -----------------------
    const int nruns = (int)a.nruns;
    int r0 = 0;
    if (lane == 0) {
        int lo = 0, hi = nruns - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (a.run_start[mid] <= e0) lo = mid;
            else hi = mid - 1;
        }
        r0 = lo;
    }
    r0 = __shfl_sync(0xffffffffu, r0, 0);
    const double* fa1 = a.fac + a.fac_off[0];
    // lane L holds run_i1 / run_start of run rbat + L
    int rbat = r0;
    int32_t ri1 = r0 + lane < nruns ? a.run_i1[r0 + lane] : 0;
    int32_t rsb = r0 + lane < nruns ? a.run_start[r0 + lane] : INT_MAX;
    int issued_r = r0;  // next run whose A_1 row is to be issued
    bool runs_done = false;
    auto issue_runs = [&](int lim) {  // warp-uniform: runs issued_r .. lim that start inside the range
        while (!runs_done && issued_r <= lim) {
            if (issued_r >= rbat + 32) {
                rbat += 32;
                ri1 = rbat + lane < nruns ? a.run_i1[rbat + lane] : 0;
                rsb = rbat + lane < nruns ? a.run_start[rbat + lane] : INT_MAX;
            }
            const int32_t rs = __shfl_sync(0xffffffffu, rsb, issued_r - rbat);
            const int32_t ai = __shfl_sync(0xffffffffu, ri1, issued_r - rbat);
            if (issued_r >= nruns || (int64_t)rs >= e_end64) {
                runs_done = true;
                break;
            }
            if (lane == 0) {
                const int sl = (issued_r - r0) % NS;  // slot / phase counted from the warp's first run
                tma::mbar_expect_tx(bar_a1 + sl, RP * 8);
                tma::bulk_g2s(a1s + sl * RP, fa1 + (int64_t)ai * RP, RP * 8, bar_a1 + sl);
            }
            ++issued_r;
        }
    };

    // ---- rows ----------------------------------------------------------------------------------
    int cur_row = (int)a.warp_rows[2 * w];
    const int first_row = cur_row;
    int row_end = (int)(min(a.row_ptr[cur_row + 1], e_end64) - cbase);
    int xcnt = 0;
    if (lane == 0) {
        tma::mbar_expect_tx(bar_x, RP * 8);
        tma::bulk_g2s(xrs, a.xhat_rm + (int64_t)cur_row * RP, RP * 8, bar_x);
        for (int j = 0; j < min(nchunks, XNCH); ++j) issue_chunk(j);
    }
    issued = min(nchunks, XNCH);
    refill_at = issued < nchunks ? CH : INT_MAX;
    __syncwarp();
    issue_runs(r0 + NS - 1);
    tma::mbar_wait(cbar, 0);
    tma::mbar_wait(bar_x, 0);
    xcnt = 1;

    double u[VPL], v[VPL], racc[VPL];
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
        racc[k] = 0.0;
        v[k] = 0.0;
        u[k] = 0.0;
    }
    int rg = -1;       // this lane group's run (-1: none since the last row end)
    int rcur = r0 - 1; // run of the entry before the current step (set by the first window)
    bool first_win = true;

    // index window: entries [wnd, wnd + 16); lane l < 16: b index of wnd + l, l >= 16: flagged
    // multiplicity of wnd + l - 16; fmask bit k: entry wnd + k starts a run
    int wnd = INT_MIN / 2, widx = 0;
    unsigned fmask = 0;
    auto window = [&](int p) {
        if (p - wnd > 16 - STEP) {
            wnd = p;
            if (wnd + 16 > land_lim || wnd >= refill_at) stage(wnd, min(wnd + 16, rel_end) - 1);
            widx = ring[(lane >= 16 ? RING : 0) + ((wnd + (lane & 15)) & (RING - 1))];
            fmask = __ballot_sync(0xffffffffu, lane >= 16 && (widx & XFLAG)) >> 16;
            if (first_win) {  // the warp's first entry: run r0 whether or not it starts it
                fmask &= ~1u;
                first_win = false;
                rcur = r0;
            }
        }
    };
    // lane group g's pair: entries p + 2g, p + 2g + 1 (m: valid entries of the step)
    auto step = [&](int p, bool full, int m) {
        double z[B][VPL], d[B];
        int mu[B];
#pragma unroll
        for (int b = 0; b < B; ++b) {
            const int k = p - wnd + 2 * g + b;  // < 16
            const int bi = __shfl_sync(0xffffffffu, widx, k);
            mu[b] = __shfl_sync(0xffffffffu, widx, 16 + k) & (int)(XFLAG - 1);
            if (!full && 2 * g + b >= m) {
#pragma unroll
                for (int c = 0; c < VPL; ++c) z[b][c] = 0.0;
                continue;
            }
            lds_cols<VPL>(z[b], sfac + bi * RP, gl);
        }
#pragma unroll
        for (int b = 0; b < B; ++b) {
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int c = 0; c < VPL; c += 2) {
                s0 = fma(u[c], z[b][c], s0);
                s1 = fma(u[c + 1], z[b][c + 1], s1);
            }
            d[b] = s0 + s1;
        }
        group_reduce<B, G>(d, lane);
#pragma unroll
        for (int b = 0; b < B; ++b) {
            double s = d[b] * (double)mu[b];
            if (!full) s = 2 * g + b < m ? s : 0.0;
#pragma unroll
            for (int c = 0; c < VPL; ++c) v[c] = fma(s, z[b][c], v[c]);
        }
    };
    auto fold = [&]() {  // racc += A_1(run rg) o v, v = 0
        if (rg >= 0) {
            const double* a1 = a1s + ((rg - r0) % NS) * RP;
#pragma unroll
            for (int t = 0; t < VPL / 2; ++t) {
                const double2 aa = *reinterpret_cast<const double2*>(a1 + 16 * t + 2 * gl);
                racc[2 * t] = fma(aa.x, v[2 * t], racc[2 * t]);
                racc[2 * t + 1] = fma(aa.y, v[2 * t + 1], racc[2 * t + 1]);
            }
        }
#pragma unroll
        for (int k = 0; k < VPL; ++k) v[k] = 0.0;
    };

    int pos = (int)(e0 - cbase);
    while (pos < rel_end) {
        // ---- the steps of the current row: [pos, row_end) ----
        int p = pos;
        while (p < row_end) {
            window(p);
            const int o = p - wnd;
            const int m = min(STEP, row_end - p);  // valid entries of this step (even)
            const unsigned fl = (fmask >> o) & ((1u << m) - 1u);
            const int myr = rcur + __popc(fl & ((2u << (2 * g)) - 1u));  // run of my pair
            const bool valid = 2 * g < m;
            const bool sw = valid && myr != rg;
            if (__any_sync(0xffffffffu, sw)) {  // run switches: the lane groups entering a new run
                // (branch-free inside this warp-uniform block: every lane reads a live slot and keeps
                // its registers unless it switches)
                {  // fold: racc += A_1(old run) o v, v = 0 (the old run's slot is still live)
                    const bool f = sw && rg >= 0;
                    const double* a1o = a1s + ((f ? rg - r0 : 0) % NS) * RP;
#pragma unroll
                    for (int t = 0; t < VPL / 2; ++t) {
                        const double2 aa = *reinterpret_cast<const double2*>(a1o + 16 * t + 2 * gl);
                        racc[2 * t] = fma(f ? aa.x : 0.0, v[2 * t], racc[2 * t]);
                        racc[2 * t + 1] = fma(f ? aa.y : 0.0, v[2 * t + 1], racc[2 * t + 1]);
                        v[2 * t] = sw ? 0.0 : v[2 * t];
                        v[2 * t + 1] = sw ? 0.0 : v[2 * t + 1];
                    }
                }
                // the oldest run any lane group holds after this step's switches: slots of older runs
                // are free; refilled in batches (>= 2 runs) up to NS - 1 runs past it (a step's
                // switches reach at most 3 runs past it)
                const int nrun = sw ? myr : rg;
                const int low = (int)__reduce_min_sync(0xffffffffu, (unsigned)(nrun >= 0 ? nrun : INT_MAX));
                if (!runs_done && issued_r <= low + 3) {
                    __syncwarp();
                    if (lane == 0) tma::fence_proxy_async();  // the folds' reads precede the refills
                    issue_runs(low + NS - 1);
                }
                const int sl = ((nrun >= 0 ? nrun : low) - r0) % NS;
                if (sw) tma::mbar_wait(bar_a1 + sl, (unsigned)(((myr - r0) / NS) & 1));
                const double* a1 = a1s + sl * RP;
#pragma unroll
                for (int t = 0; t < VPL / 2; ++t) {
                    const double2 xx = *reinterpret_cast<const double2*>(xrs + 16 * t + 2 * gl);
                    const double2 aa = *reinterpret_cast<const double2*>(a1 + 16 * t + 2 * gl);
                    u[2 * t] = sw ? xx.x * aa.x : u[2 * t];
                    u[2 * t + 1] = sw ? xx.y * aa.y : u[2 * t + 1];
                }
                rg = nrun;
            }
            if (m == STEP) step(p, true, STEP);  // (one masked call site measured slower: 2.61 vs 2.41 ms)
            else step(p, false, m);
            rcur += __popc(fl);
            p += m;
        }
        pos = row_end;
        // ---- row end: the lane groups' folds, then their partial rows summed and written ----
        fold();
        rg = -1;
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
                    double2* d2 = reinterpret_cast<double2*>(dst + 16 * t + 2 * gl);
                    double2 ov = make_double2(racc[2 * t], racc[2 * t + 1]);
                    if (a.accumulate) {
                        const double2 cur = *d2;
                        ov.x += cur.x;
                        ov.y += cur.y;
                    }
                    *d2 = ov;
                }
            }
        } else {  // a row shared with neighbouring warps: slot, then the last arriver sums in warp order
            double* slot = (cur_row == first_row ? a.slot_a : a.slot_b) + (int64_t)w * RP;
            if (g == 0) {
#pragma unroll
                for (int t = 0; t < VPL / 2; ++t)
                    *reinterpret_cast<double2*>(slot + 16 * t + 2 * gl) = make_double2(racc[2 * t], racc[2 * t + 1]);
            }
            __syncwarp();
            unsigned last = 0;
            if (lane == 0) {
                __threadfence();
                last = xatom_add_acqrel(a.rowcnt + cur_row, 1u) == (unsigned)ncta - 1;
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
        }
        __syncwarp();
    }
}

// ---- plan padding: every run of a part to an even length -------------------------------------
// run r of the unpadded part: entries [rs[r], rs[r+1]); dummies before it: off[r] (exclusive scan
// of the odd lengths).  One thread per run copies its entries (b, multiplicity | run-start flag,
// row) and appends a zero-multiplicity copy of its last entry when its length is odd.
__global__ void pad_runs_kernel(const int32_t* __restrict__ rs, const int32_t* __restrict__ off, int64_t nr,
                                const int32_t* __restrict__ ia, const int32_t* __restrict__ ib,
                                const int32_t* __restrict__ mult, const int32_t* __restrict__ rows, int32_t* oa,
                                int32_t* ob, int32_t* om, int32_t* orow) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nr) return;
    const int32_t b0 = rs[r], b1 = rs[r + 1];
    const int64_t o = (int64_t)b0 + off[r];
    for (int32_t e = b0; e < b1; ++e) {
        const int64_t d = o + (e - b0);
        oa[d] = ia[e];
        ob[d] = ib[e];
        om[d] = mult[e] | (e == b0 ? (int32_t)XFLAG : 0);
        orow[d] = rows[e];
    }
    if ((b1 - b0) & 1) {
        const int64_t d = o + (b1 - b0);
        oa[d] = ia[b1 - 1];
        ob[d] = ib[b1 - 1];
        om[d] = 0;
        orow[d] = rows[b1 - 1];
    }
}
__global__ void odd_len_kernel(const int32_t* __restrict__ rs, int64_t nr, int32_t* odd) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < nr) odd[r] = (rs[r + 1] - rs[r]) & 1;
}

}  // namespace

bool xruns_supported(int64_t rp, int dother, bool mult) { return rp == 64 && dother == 2 && mult; }

size_t xruns_smem_bytes(int64_t rp, int64_t sf_doubles) {
    if (rp != 64) return SIZE_MAX;
    return XLay<64, 16, 64>::bytes(sf_doubles);
}
int xruns_warps_per_sm() { return 16; }

void xruns_scatter_gather(const RunsArgs& a, int64_t sf_doubles, cudaStream_t s) {
    if (!xruns_supported(a.rp, a.dother, a.mult != nullptr)) throw_invalid("xruns: 3-way coalesced plans at padded rank 64");
    const size_t smem = xruns_smem_bytes(a.rp, sf_doubles);
    if (smem > XSMEM_CAP) throw_invalid("xruns: staged factors exceed shared memory");
    auto kern = xruns_kernel<64, 16, 64>;
    func_attr_once((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, XSMEM_CAP);
    const int grid = (a.warps + 15) / 16;
    kern<<<grid, 16 * 32, smem, s>>>(a);
    CPHIFI_CHECK_LAUNCH();
}

int64_t pad_runs_even(const int32_t* run_start, int64_t nr, const int32_t* ia, const int32_t* ib, const int32_t* mult,
                      const int32_t* rows, int32_t* oa, int32_t* ob, int32_t* om, int32_t* orow, int64_t q,
                      cudaStream_t s) {
    if (nr == 0) return q;
    DevBuf<int32_t> odd(nr), off(nr);
    odd_len_kernel<<<(unsigned)((nr + 255) / 256), 256, 0, s>>>(run_start, nr, odd.get());
    CPHIFI_CHECK_LAUNCH();
    size_t bytes = 0;
    CPHIFI_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, odd.get(), off.get(), nr, s));
    DevBuf<unsigned char> tmp(bytes);
    CPHIFI_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, odd.get(), off.get(), nr, s));
    pad_runs_kernel<<<(unsigned)((nr + 255) / 256), 256, 0, s>>>(run_start, off.get(), nr, ia, ib, mult, rows, oa, ob,
                                                                 om, orow);
    CPHIFI_CHECK_LAUNCH();
    int32_t last_off = 0, last_odd = 0;
    CPHIFI_CUDA(cudaMemcpyAsync(&last_off, off.get() + nr - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CPHIFI_CUDA(cudaMemcpyAsync(&last_odd, odd.get() + nr - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CPHIFI_CUDA(cudaStreamSynchronize(s));
    return q + last_off + last_odd;
}

}  // namespace cphifi
