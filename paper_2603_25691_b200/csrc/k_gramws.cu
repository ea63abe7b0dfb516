// k_gramws.cu — the row-Gram build G_i = sum_{l in row i} w_l z_l z_l' with producer / consumer
// warp specialisation (sm_100a).
//
// The identity and its use are in k_gram.cu.  The previous builds alternate, inside every CTA, a
// gather phase (Khatri-Rao rows z of a batch of observations, factor rows fetched through L1 / L2)
// and a DMMA phase around __syncthreads, and rely on a second CTA per SM to overlap the two; with
// the factors gathered from L2 (config 4: 2 x 512 B per entry, 250 GB per build) the gathers
// dominated.  Here, one CTA per SM:
//  * the per-observation factors (modes 2.. of the plan) are staged in shared memory once (the run
//    kernel's factor-block parts when they do not fit: config 4 builds G in two passes, one per
//    half of A_3); the first other mode — constant along the plan's runs — is read through L1;
//  * NPW producer warps, each building every NPW-th batch's z rows into its own shared-memory buffer,
//    run ahead of the consumer warps' DMMA (m8n8k4, fp64) of batch k: a full / empty mbarrier pair
//    per buffer, no CTA-wide barrier in the steady state;
//  * consumer warps own 2 x 2 blocks of 8 x 8 tiles of G's upper triangle (RP = 64: 10 warps; RP =
//    32 / 16: 3 / 1 blocks x KS warps splitting each batch's k-steps, summed in ks order at the row
//    flush); the weight w_l multiplies the A fragment (no second, weighted copy of z);
//  * rows split between CTAs are finished by the last CTA summing per-CTA slots in CTA order;
//    with several parts the launches add into G (zeroed first): deterministic.
// Both roles walk the same batch sequence (batches never cross a row), so no per-batch metadata
// is exchanged.
// Status: opt-in (CPHIFI_GRAM_WS=1; capi.cu gram_build_parts): measured slower than k_gram.cu's
// single-pass builds at configs 3 / 4 (26.9 / 71.6 ms vs 24.6 / 61.8 ms; ncu at config 3: tensor
// pipe 32 %, long-scoreboard stalls on the producers' global loads) — kept, tested, for the record.
#include "kernels.cuh"
#include "tma.cuh"

namespace cphifi {
namespace {

constexpr int WGB = 32;    // observations per batch
constexpr int NBUF = 4;    // z buffers
constexpr int NPW = 4;     // producer warps

template <int RP>
struct Ws {
    static constexpr int NT = RP / 8, NB = NT / 2, NBLK = NB * (NB + 1) / 2;
    static constexpr int KS = RP >= 64 ? 1 : (RP >= 32 ? 3 : 8);
    static constexpr int NCW = NBLK * KS;               // consumer warps
    static constexpr int T = 32 * (NCW + NPW);
    static constexpr int ZP = RP + 4;                   // z row pitch (conflict-free fragments)
    static constexpr size_t zbytes = sizeof(double) * NBUF * (WGB * ZP + WGB);
    static constexpr size_t redbytes = KS > 1 ? sizeof(double) * KS * RP * RP : 0;
    static constexpr size_t bars = 128;  // 2 NBUF + 1 mbarriers and a flag, padded: z rows stay 16-byte aligned
    static size_t bytes(int64_t sf) { return bars + zbytes + redbytes + sizeof(double) * (size_t)sf; }
};

__device__ __forceinline__ unsigned atom_add_acqrel_w(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ void consumer_sync(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

template <int RP, int DO>
__global__ void __launch_bounds__(Ws<RP>::T, 1) gram_ws_kernel(const GramArgs a) {
    using W = Ws<RP>;
    constexpr int ZP = W::ZP, KS = W::KS, NB = W::NB, NCW = W::NCW;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* empty = full + NBUF;
    uint64_t* cbar = empty + NBUF;
    int* s_last = reinterpret_cast<int*>(cbar + 1);
    double* zs = reinterpret_cast<double*>(smem_raw + W::bars);  // NBUF x WGB x ZP
    double* sw = zs + NBUF * WGB * ZP;                            // NBUF x WGB
    double* red = sw + NBUF * WGB;                                // KS x RP x RP
    double* sfac = red + (KS > 1 ? KS * RP * RP : 0);             // modes 1 .. DO-1
    const int c = blockIdx.x;
    const int64_t ca = a.cta_beg[c], cb = a.cta_beg[c + 1];
    if (ca >= cb) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int64_t frows[DO > 1 ? DO : 2];
#pragma unroll
    for (int m = 0; m < DO; ++m) frows[m] = ((m + 1 < DO ? a.fac_off[m + 1] : a.fac_total) - a.fac_off[m]) / RP;
    if (tid == 0) {
        for (int b = 0; b < NBUF; ++b) {
            tma::mbar_init(full + b, 32);        // every lane of the buffer's producer warp arrives
            tma::mbar_init(empty + b, NCW * 32); // every consumer thread arrives after its reads
        }
        tma::mbar_init(cbar, 1);
        tma::fence_mbar_init();
        if constexpr (DO > 1) {
            unsigned bytes = 0;
            for (int m = 1; m < DO; ++m) bytes += (unsigned)(frows[m] * RP * 8);
            tma::mbar_expect_tx(cbar, bytes);
            int64_t so = 0;
            for (int m = 1; m < DO; ++m) {
                const int64_t tot = frows[m] * RP * 8;
                for (int64_t b0 = 0; b0 < tot; b0 += 32768)
                    tma::bulk_g2s(reinterpret_cast<unsigned char*>(sfac + so) + b0,
                                  reinterpret_cast<const unsigned char*>(a.fac + a.fac_off[m]) + b0,
                                  (unsigned)min((int64_t)32768, tot - b0), cbar);
                so += frows[m] * RP;
            }
        } else {
            tma::mbar_arrive(cbar);
        }
    }
    __syncthreads();

    // the batch walk shared by both roles: batch = [pos, pos + cnt) inside row `row`
    const int64_t first_row = a.cta_rows[2 * c];

    if (warp >= NCW) {  // ---------------------------------------------------------- producers
        // producer warp pw builds the batches k = pw (mod NPW) into buffer pw (NBUF = NPW): NPW
        // batches in flight.  Lane t loads entry t's indices and weight (coalesced), then the warp
        // builds the z rows PPR column pairs per row, EPI rows per pass, with the row's indices
        // broadcast by shuffles: every factor-row read is a contiguous segment (conflict-free).
        static_assert(NBUF == NPW, "one buffer per producer warp");
        constexpr int PPR = RP / 2, EPI = 32 / PPR;
        const int pw = warp - NCW, sub = lane / PPR, j = 2 * (lane % PPR);
        const double* f0 = a.fac + a.fac_off[0];
        const double* fs[DO > 1 ? DO : 2];
        {
            int64_t so = 0;
            for (int m = 1; m < DO; ++m) {
                fs[m] = sfac + so;
                so += frows[m] * RP;
            }
        }
        tma::mbar_wait(cbar, 0);
        int64_t pos = ca, row = first_row, row_end = a.row_ptr[row + 1];
        for (int k = 0; pos < cb; ++k) {
            while (pos >= row_end) {
                do {
                    ++row;
                    row_end = a.row_ptr[row + 1];
                } while (row_end <= pos);
            }
            const int cnt = (int)min((int64_t)WGB, min(cb, row_end) - pos);
            if (k % NPW == pw) {
                const int b = pw;
                if (k >= NBUF) tma::mbar_wait(empty + b, (unsigned)((k / NBUF - 1) & 1));
                // the plan columns 2 x NPW batches ahead into L2 (the index loads below then hit L2
                // instead of waiting on DRAM: ~1 us per batch otherwise)
                if (lane <= DO) {
                    const int64_t ahead = pos + 2 * NPW * WGB;
                    const int32_t* col = lane < DO ? a.idx + (int64_t)lane * a.q : a.mult;
                    if (col && ahead < cb)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(col + ahead));
                }
                int ix[DO];
                double wl = 0.0;
                if (lane < cnt) {
#pragma unroll
                    for (int m = 0; m < DO; ++m) ix[m] = __ldg(a.idx + (int64_t)m * a.q + pos + lane);
                    wl = a.mult ? (double)(__ldg(a.mult + pos + lane) & RUN_MULT_MASK) : 1.0;
                } else {
#pragma unroll
                    for (int m = 0; m < DO; ++m) ix[m] = 0;
                }
                double* z = zs + b * WGB * ZP;
                sw[b * WGB + lane] = wl;  // WGB == 32: one weight per lane (0 beyond cnt)
#pragma unroll 4
                for (int t0 = 0; t0 < WGB; t0 += EPI) {
                    const int t = t0 + sub;
                    int it[DO];
#pragma unroll
                    for (int m = 0; m < DO; ++m) it[m] = __shfl_sync(0xffffffffu, ix[m], t);
                    double2 v = __ldg(reinterpret_cast<const double2*>(f0 + (int64_t)it[0] * RP + j));
#pragma unroll
                    for (int m = 1; m < DO; ++m) {
                        const double2 f = *reinterpret_cast<const double2*>(fs[m] + (int64_t)it[m] * RP + j);
                        v.x *= f.x;
                        v.y *= f.y;
                    }
                    if (t >= cnt) v = make_double2(0.0, 0.0);
                    *reinterpret_cast<double2*>(z + t * ZP + j) = v;
                }
                tma::mbar_arrive(full + b);
            }
            pos += cnt;
        }
        return;
    }

    // ------------------------------------------------------------------------------ consumers
    const int g = lane >> 2, kq = lane & 3;
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
    const int ctid = tid;  // consumers are threads [0, NCW * 32)
    auto finish_row = [&](int64_t rr) {
        const int ncta = a.row_ncta[rr];
        double* dst = ncta == 1 ? a.g + rr * RP * RP
                    : rr == first_row ? a.slot_a + (int64_t)c * RP * RP
                                      : a.slot_b + (int64_t)c * RP * RP;
        const bool acc_g = a.accumulate && ncta == 1;  // slots are always written fresh
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
                            const double v = acc[x][y][h];
                            dst[ii * RP + jj] = acc_g ? dst[ii * RP + jj] + v : v;
                            if (ti != tj) dst[jj * RP + ii] = acc_g ? dst[jj * RP + ii] + v : v;
                        }
                    }
                }
        } else {
            consumer_sync(NCW * 32);
#pragma unroll
            for (int x = 0; x < 2; ++x)
#pragma unroll
                for (int y = 0; y < 2; ++y)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int ii = (2 * bi + x) * 8 + g, jj = (2 * bj + y) * 8 + 2 * kq + h;
                        red[(ks * RP + ii) * RP + jj] = acc[x][y][h];
                    }
            consumer_sync(NCW * 32);
            for (int e = ctid; e < RP * RP; e += NCW * 32) {  // upper triangle: the k-splits in order
                const int ii = e / RP, jj = e % RP;
                if (ii / 8 > jj / 8) continue;
                double sv = 0.0;
#pragma unroll
                for (int k2 = 0; k2 < KS; ++k2) sv += red[(k2 * RP + ii) * RP + jj];
                if (ii / 8 < jj / 8 || ii <= jj) {
                    dst[ii * RP + jj] = acc_g ? dst[ii * RP + jj] + sv : sv;
                    if (ii != jj) dst[jj * RP + ii] = acc_g ? dst[jj * RP + ii] + sv : sv;
                }
            }
        }
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
            for (int y = 0; y < 2; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
        if (ncta > 1) {  // the last CTA of a split row sums the slots in CTA order
            consumer_sync(NCW * 32);
            if (ctid == 0) {
                __threadfence();
                *s_last = atom_add_acqrel_w(a.rowcnt + rr, 1u) == (unsigned)ncta - 1;
                if (*s_last) a.rowcnt[rr] = 0;
            }
            consumer_sync(NCW * 32);
            if (*s_last) {
                const int u0 = a.row_first_cta[rr];
                const bool starts = a.row_ptr[rr] == a.cta_beg[u0];
                for (int e = ctid; e < RP * RP; e += NCW * 32) {
                    double sv = starts ? __ldcg(a.slot_a + (int64_t)u0 * RP * RP + e)
                                       : __ldcg(a.slot_b + (int64_t)u0 * RP * RP + e);
                    for (int u = u0 + 1; u < u0 + ncta; ++u) sv += __ldcg(a.slot_a + (int64_t)u * RP * RP + e);
                    double* gd = a.g + rr * RP * RP + e;
                    *gd = a.accumulate ? *gd + sv : sv;
                }
            }
            consumer_sync(NCW * 32);  // s_last read by every consumer before the next row reuses it
        }
    };
    int64_t pos = ca, row = first_row, row_end = a.row_ptr[row + 1];
    for (int k = 0; pos < cb; ++k) {
        while (pos >= row_end) {
            finish_row(row);
            do {
                ++row;
                row_end = a.row_ptr[row + 1];
            } while (row_end <= pos);
        }
        const int cnt = (int)min((int64_t)WGB, min(cb, row_end) - pos);
        const int b = k % NBUF;
        tma::mbar_wait(full + b, (unsigned)((k / NBUF) & 1));
        const double* z = zs + b * WGB * ZP;
        const double* w = sw + b * WGB;
#pragma unroll
        for (int k0 = 4 * ks; k0 < WGB; k0 += 4 * KS) {
            const int t = k0 + kq;
            const double wt = w[t];  // 0 beyond cnt: padded observations contribute exactly zero
            double av[2], bv[2];
#pragma unroll
            for (int x = 0; x < 2; ++x) av[x] = z[t * ZP + (2 * bi + x) * 8 + g] * wt;  // A(i, t) = w_t z_t(i)
#pragma unroll
            for (int y = 0; y < 2; ++y) bv[y] = z[t * ZP + (2 * bj + y) * 8 + g];       // B(t, j) = z_t(j)
#pragma unroll
            for (int x = 0; x < 2; ++x)
#pragma unroll
                for (int y = 0; y < 2; ++y) dmma(acc[x][y], av[x], bv[y]);
        }
        tma::mbar_arrive(empty + b);
        pos += cnt;
    }
    finish_row(row);
}

template <int RP, int DO>
void launch_ws(const GramArgs& a, int grid, int64_t sf, cudaStream_t s) {
    using W = Ws<RP>;
    auto kern = gram_ws_kernel<RP, DO>;
    const size_t smem = W::bytes(sf);
    func_attr_once((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, W::T, smem, s>>>(a);
    CPHIFI_CHECK_LAUNCH();
}

template <int RP>
void launch_ws_rp(const GramArgs& a, int grid, int64_t sf, cudaStream_t s) {
    switch (a.dother) {
        case 2: launch_ws<RP, 2>(a, grid, sf, s); break;
        case 3: launch_ws<RP, 3>(a, grid, sf, s); break;
        case 4: launch_ws<RP, 4>(a, grid, sf, s); break;
        default: throw_invalid("gram build (warp-specialised): needs 2..4 other modes");
    }
}

}  // namespace

bool gram_ws_supported(int64_t rp, int dother) { return (rp == 16 || rp == 32 || rp == 64) && dother >= 2 && dother <= 4; }

size_t gram_ws_smem_bytes(int64_t rp, int64_t sf) {
    switch (rp) {
        case 16: return Ws<16>::bytes(sf);
        case 32: return Ws<32>::bytes(sf);
        default: return Ws<64>::bytes(sf);
    }
}

void gram_build_ws(const GramArgs& a, int grid, int64_t sf, cudaStream_t s) {
    switch (a.rp) {
        case 16: launch_ws_rp<16>(a, grid, sf, s); break;
        case 32: launch_ws_rp<32>(a, grid, sf, s); break;
        case 64: launch_ws_rp<64>(a, grid, sf, s); break;
        default: throw_invalid("gram build (warp-specialised): padded rank must be 16, 32 or 64");
    }
}

}  // namespace cphifi
