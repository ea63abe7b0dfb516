// capi.cu — the C-ABI (include/cphifi_b200.h): host orchestration of the sm_100a kernels.
//
// Each entry point restates one reference function (cited per function, paths relative to
// proj/include/cphifi/) on device-resident plans.  C++ exceptions never cross the ABI:
// `guard` maps them to status codes and a thread-local message.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>

#include "kernels.cuh"

using namespace cphifi;

#include <set>
#include <tuple>

namespace cphifi {
static thread_local std::string g_last_error;
void set_last_error(const std::string& m) { g_last_error = m; }

void func_attr_once(const void* f, cudaFuncAttribute attr, int value) {
    static std::mutex m;
    static std::set<std::tuple<const void*, int, int, int>> done;
    int dev = 0;
    CPHIFI_CUDA(cudaGetDevice(&dev));
    const auto key = std::make_tuple(f, (int)attr, value, dev);
    std::lock_guard<std::mutex> lk(m);
    if (done.count(key)) return;
    CPHIFI_CUDA(cudaFuncSetAttribute(f, attr, value));
    done.insert(key);
}
}  // namespace cphifi

namespace {

template <class F>
int guard(F&& f) {
    try {
        f();
        return CPHIFI_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        set_last_error("out of host memory");
        return CPHIFI_RUNTIME_ERROR;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return CPHIFI_RUNTIME_ERROR;
    } catch (...) {
        set_last_error("unknown error");
        return CPHIFI_RUNTIME_ERROR;
    }
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) CPHIFI_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// Plan columns carry OBS_PAD slack elements: the streaming kernels' TMA bulk copies round staged
// columns to 16-byte boundaries (k_stream.cu) or copy whole CH-entry chunks from a 16-byte aligned
// base (k_runs.cu / k_xruns.cu, CH <= 128: up to CH + 2 elements past the last one — 64 was the
// slack of the former 64-entry chunks, and a part ending in the last 256 bytes of its allocation
// faulted now and then).
constexpr int64_t OBS_PAD = 256;

// a kernel's eigenvalues below -PSD_TOL * max(|mu|_max, 1) make it indefinite (not a rounding artefact)
constexpr double PSD_TOL = 1e-10;

void need(const void* p, const char* what) {
    if (!p) throw_invalid(std::string(what) + ": null argument");
}

void h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes) CPHIFI_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
}
void d2h_sync(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes) CPHIFI_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
    CPHIFI_CUDA(cudaStreamSynchronize(s));
}

// More than one rank: NCCL over NVLink, or the one-GPU virtual communicator (test hook).
bool ctx_multi(cphifi_ctx ctx) { return ctx->nranks > 1 && (ctx->comm || ctx->vcomm); }

// Sum of every rank's `send` into `recv` on every rank (in place allowed), ordered on the context
// stream.  NCCL: ncclAllReduce.  Virtual communicator: see cphifi_vcomm_s (common.cuh).
thread_local cudaEvent_t g_dense_event = nullptr;  // cphifi_unaligned_matvec_timed's mid-phase-B event
thread_local bool g_dense_recorded = false;
thread_local bool g_count_only = false;  // cphifi_unaligned_matvec_launches: capture this library's kernels only

void allreduce_sum(cphifi_ctx ctx, const double* send, double* recv, size_t count) {
    if (!ctx_multi(ctx) || !count || g_count_only) {
        if (send != recv && count)
            CPHIFI_CUDA(cudaMemcpyAsync(recv, send, sizeof(double) * count, cudaMemcpyDeviceToDevice, ctx->stream));
        return;
    }
    if (ctx->comm) {
        CPHIFI_NCCL(ncclAllReduce(send, recv, count, ncclDouble, ncclSum, ctx->comm, ctx->stream));
        return;
    }
    cphifi_vcomm_s* vc = ctx->vcomm;
    const int me = ctx->rank, nr = vc->nranks;
    if (ctx->vc_scratch.n < count) ctx->vc_scratch.alloc(count);
    vc->send[me] = send;
    CPHIFI_CUDA(cudaEventRecord(vc->ready[me], ctx->stream));
    vc->barrier();  // every rank's send buffer and ready event are published
    for (int k = 0; k < nr; ++k) CPHIFI_CUDA(cudaStreamWaitEvent(ctx->stream, vc->ready[k], 0));
    rank_order_sum(vc->send.data(), nr, ctx->vc_scratch.get(), count, ctx->num_sms, ctx->stream);
    CPHIFI_CUDA(cudaEventRecord(vc->done[me], ctx->stream));
    vc->barrier();  // every rank has enqueued its reads of the send buffers
    for (int k = 0; k < nr; ++k) CPHIFI_CUDA(cudaStreamWaitEvent(ctx->stream, vc->done[k], 0));
    CPHIFI_CUDA(cudaMemcpyAsync(recv, ctx->vc_scratch.get(), sizeof(double) * count, cudaMemcpyDeviceToDevice,
                                ctx->stream));
}

void allreduce(cphifi_ctx ctx, double* buf, size_t count) { allreduce_sum(ctx, buf, buf, count); }

int read_flag(cphifi_ctx ctx, int* dflag) {
    int h = 0;
    d2h_sync(&h, dflag, sizeof(int), ctx->stream);
    return h;
}

// sym_eig (kernel.hpp:40-49) on a device matrix: symmetry check, syevd, clamp at 0.
// Returns the smallest and largest eigenvalue before the clamp (syevd: ascending order).
std::pair<double, double> device_sym_eig(cphifi_ctx ctx, const double* a, int64_t n, double* u_out, double* d_out) {
    DevBuf<double> chk(2);
    max_asym(a, n, chk.get(), ctx->stream);
    double h[2];
    d2h_sync(h, chk.get(), sizeof h, ctx->stream);
    if (h[0] > 1e-12 * std::max(h[1], 1.0)) throw_invalid("sym_eig: matrix is not symmetric");
    CPHIFI_CUDA(cudaMemcpyAsync(u_out, a, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, ctx->stream));
    int lwork = 0;
    CPHIFI_SOLVER(cusolverDnDsyevd_bufferSize(ctx->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER,
                                              (int)n, u_out, (int)n, d_out, &lwork));
    DevBuf<double> work(std::max(lwork, 1));
    DevBuf<int> info(1);
    CPHIFI_SOLVER(cusolverDnDsyevd(ctx->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)n, u_out,
                                   (int)n, d_out, work.get(), lwork, info.get()));
    int hinfo = 0;
    d2h_sync(&hinfo, info.get(), sizeof(int), ctx->stream);
    if (hinfo != 0) throw_runtime("sym_eig: eigendecomposition failed");
    double ext[2] = {0.0, 0.0};
    d2h_sync(&ext[0], d_out, sizeof(double), ctx->stream);
    d2h_sync(&ext[1], d_out + n - 1, sizeof(double), ctx->stream);
    clamp_nonneg(d_out, n, ctx->stream);
    return {ext[0], ext[1]};
}

void mode_eig_once(cphifi_mode m) {
    std::call_once(m->once, [m] {
        std::lock_guard<std::mutex> lk(m->mu_lock);
        if (m->have_eig) return;  // installed via cphifi_mode_set_eig
        DeviceGuard dg(m->ctx->device);
        m->u.alloc(m->n * m->n);
        m->mu.alloc(m->n);
        const auto ext = device_sym_eig(m->ctx, m->kernel.get(), m->n, m->u.get(), m->mu.get());
        m->psd = ext.first >= -PSD_TOL * std::max(std::fabs(ext.second), 1.0);
        m->have_eig = true;
        m->eig_count = 1;
    });
}

// U' for the sandwich's second phase (k_sandwich.cu), built once per installed eigenbasis
const double* mode_ut(cphifi_mode m) {
    std::lock_guard<std::mutex> lk(m->mu_lock);
    if (!m->have_ut) {
        m->ut.alloc(m->n * m->n);
        transpose_sq(m->u.get(), m->n, m->ut.get(), m->ctx->stream);
        m->have_ut = true;
    }
    return m->ut.get();
}

// U diag(mu) for the eigenbasis PCG (K X = U diag(mu) U' X with the clamped spectrum)
const double* mode_um(cphifi_mode m) {
    std::lock_guard<std::mutex> lk(m->mu_lock);
    if (!m->have_um) {
        m->um.alloc(m->n * m->n);
        scale_cols(m->u.get(), m->n, m->mu.get(), m->um.get(), m->ctx->stream);
        m->have_um = true;
    }
    return m->um.get();
}

// Number of leading eigenvalues that are exactly 0 after the clamp (syevd returns them ascending,
// so the clamped negatives come first), rounded down to a multiple of 8 so the offset GEMM
// operands stay 16-byte aligned.  The eigenbasis operator skips those rows / columns of U: their
// mu_i = 0 multiplies them out of K X, and their rows of y~ reduce to rho x~.  One host read per
// installed eigenbasis.
int64_t mode_nzero(cphifi_mode m) {
    std::lock_guard<std::mutex> lk(m->mu_lock);
    if (m->nzero < 0) {
        std::vector<double> h((size_t)m->n);
        d2h_sync(h.data(), m->mu.get(), sizeof(double) * m->n, m->ctx->stream);
        int64_t z = 0;
        while (z < m->n && h[(size_t)z] == 0.0) ++z;
        m->nzero = z & ~int64_t(7);
    }
    return m->nzero;
}

const double* mode_umt(cphifi_mode m) {
    const double* ut = mode_ut(m);
    std::lock_guard<std::mutex> lk(m->mu_lock);
    if (!m->have_umt) {
        m->umt.alloc(m->n * m->n);
        scale_rows(ut, m->n, m->mu.get(), m->umt.get(), m->ctx->stream);
        m->have_umt = true;
    }
    return m->umt.get();
}

// Per-thread pinned, device-mapped status word for kernels that report a data error (zero
// decoupled denominator): no allocation and no extra synchronisation per call; the caller reads
// it after the synchronisation it performs anyway.
int* thread_flag() {
    static thread_local int* f = nullptr;
    if (!f) CPHIFI_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&f), sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable));
    return f;
}

// GEMM helpers (column-major unless stated)
void gemm_nn(cphifi_ctx ctx, int64_t m, int64_t n, int64_t k, const double* a, int64_t lda, const double* b,
             int64_t ldb, double* c, int64_t ldc) {
    GemmArgs g;
    g.m = m; g.n = n; g.k = k;
    g.a = a; g.a_rs = 1; g.a_cs = lda;
    g.b = b; g.b_rs = 1; g.b_cs = ldb;
    g.c = c; g.c_rs = 1; g.c_cs = ldc;
    gemm(g, ctx->num_sms, ctx->stream);
}

cphifi_mode new_mode(cphifi_ctx ctx, int64_t n, double lambda) {
    auto* m = new cphifi_mode_s;
    m->ctx = ctx;
    m->n = n;
    m->lambda = lambda;
    m->kernel.alloc(n * n);
    return m;
}

// ---- row-aligned CTA partition of the sorted observations (the fused kernel's schedule) --
// Greedy packing of WHOLE rows into CTAs of at most L observations; a row longer than L is cut
// into ceil(len / L) near-equal pieces (the only split rows).  L starts at ceil(q / cmax) and
// grows until the plan fits the co-resident CTA budget cmax.  The launch is padded with empty
// CTAs up to `cmin` so that the dense row phases still spread over the whole chip.
struct PartitionPlan {
    int ctas = 0;
    int64_t max_span = 0;                 // max rows touched by one CTA
    std::vector<int64_t> beg;             // ctas + 1
    std::vector<int64_t> rows;            // 2 * ctas: first / last row per CTA
    std::vector<int32_t> row_first_cta;   // n
    std::vector<int32_t> row_ncta;        // n
};

// equal > 0: exactly `equal` CTAs of equal observation count (rows split wherever a boundary
// falls; the kernel finishes split rows through its slots), else the row-aligned plan below.
// `given` (non-empty, nondecreasing, from 0 to q): those CTA boundaries as they are.
void plan_partition(const std::vector<int64_t>& rp, int cmax, int cmin, PartitionPlan& pl, int equal = 0,
                    const std::vector<int64_t>* given = nullptr) {
    const int64_t n = (int64_t)rp.size() - 1, q = rp[n];
    std::vector<int64_t> starts;
    if (given) {
        starts = *given;
        starts.erase(std::unique(starts.begin(), starts.end()), starts.end());
        if (starts.size() < 2) starts.assign({0, q});
        equal = 1;  // no row-aligned search below
    } else if (equal > 0) {  // (empty CTAs dropped: the CTAs sharing a split row must be consecutive)
        for (int c = 0; c <= equal; ++c) starts.push_back(q * c / equal);
        starts.erase(std::unique(starts.begin(), starts.end()), starts.end());
        if (starts.size() < 2) starts.assign({0, q});
    }
    auto build = [&](int64_t L) {
        starts.assign(1, 0);
        int64_t load = 0;
        for (int64_t i = 0; i < n; ++i) {
            const int64_t len = rp[i + 1] - rp[i];
            if (len == 0) continue;
            if (len > L) {
                if (load > 0) starts.push_back(rp[i]);
                const int64_t pieces = (len + L - 1) / L;
                for (int64_t pc = 1; pc < pieces; ++pc) starts.push_back(rp[i] + len * pc / pieces);
                starts.push_back(rp[i + 1]);
                load = 0;
            } else {
                if (load > 0 && load + len > L) {
                    starts.push_back(rp[i]);
                    load = 0;
                }
                load += len;
            }
        }
        starts.push_back(q);
        starts.erase(std::unique(starts.begin(), starts.end()), starts.end());  // drop empty CTAs
        if (starts.size() < 2) starts.assign({0, q});
    };
    int64_t L = std::max<int64_t>(1, (q + cmax - 1) / std::max(cmax, 1));
    for (; equal <= 0;) {
        build(L);
        if ((int64_t)starts.size() - 1 <= cmax) break;
        L = L + L / 8 + 1;
    }
    while ((int64_t)starts.size() - 1 < cmin) starts.push_back(q);  // empty padding CTAs
    pl.ctas = (int)starts.size() - 1;
    pl.beg = starts;
    pl.rows.assign(2 * (size_t)pl.ctas, 0);
    pl.row_first_cta.assign(n, -1);
    pl.row_ncta.assign(n, 0);
    pl.max_span = 0;
    auto row_of = [&](int64_t pos) {  // largest i with rp[i] <= pos
        return (int64_t)(std::upper_bound(rp.begin(), rp.end(), pos) - rp.begin()) - 1;
    };
    for (int c = 0; c < pl.ctas; ++c) {
        const int64_t a = starts[c], b = starts[c + 1];
        if (a >= b) continue;
        const int64_t r0 = row_of(a), r1 = row_of(b - 1);
        pl.rows[2 * c] = r0;
        pl.rows[2 * c + 1] = r1;
        pl.max_span = std::max(pl.max_span, r1 - r0 + 1);
        for (int64_t i = r0; i <= r1; ++i) {
            if (rp[i + 1] == rp[i]) continue;
            if (pl.row_first_cta[i] < 0) pl.row_first_cta[i] = c;
            ++pl.row_ncta[i];
        }
    }
    for (auto& v : pl.row_first_cta) v = std::max(v, 0);
}

// ---- unaligned pieces ------------------------------------------------------------------
bool is_multi(cphifi_unaligned p) { return ctx_multi(p->obs->ctx); }

// The complete (all-rank) Yhat: the local one on one GPU, the NCCL sum otherwise.
double* yhat_result(cphifi_unaligned p) { return is_multi(p) ? p->yhat_sum.get() : p->yhat_rm.get(); }

// Out-of-place sum of the ranks' partial Yhat (the local buffer keeps its zero rows).
void allreduce_yhat(cphifi_unaligned p) {
    cphifi_ctx ctx = p->obs->ctx;
    if (is_multi(p)) allreduce_sum(ctx, p->yhat_rm.get(), p->yhat_sum.get(), (size_t)p->n * p->rp);
}

FusedArgs fused_args(cphifi_unaligned p, unsigned phases) {
    cphifi_obs o = p->obs;
    FusedArgs a;
    a.n = p->n;
    a.r = p->r;
    a.rp = p->rp;
    a.q = o->ldq;
    a.dother = o->d - 1;
    a.phases = phases;
    a.row_ptr = o->row_ptr.get();
    a.idx = o->idx_o.get();
    a.fac = p->fac.get();
    for (int m = 0; m < o->d - 1; ++m) a.fac_off[m] = p->fac_off[m];
    a.fac_total = (int64_t)p->fac.n;
    a.mult = o->coalesced ? o->mult.get() : nullptr;
    a.kmat = p->mode ? p->mode->kernel.get() : nullptr;
    a.xhat_rm = p->xhat_rm.get();
    a.yhat_rm = p->yhat_rm.get();
    a.slot_a = p->slot_a.get();
    a.slot_b = p->slot_b.get();
    a.cta_rows = p->cta_rows.get();
    a.cta_beg = p->cta_beg.get();
    a.row_first_cta = p->row_first_cta.get();
    a.row_ncta = p->row_ncta.get();
    a.lambda = p->mode ? p->mode->lambda : 0.0;
    a.rho = p->rho;
    a.barrier = p->barrier.get();
    a.rowcnt = p->rowcnt.get();
    a.prefetch = p->prefetch ? 1 : 0;
    a.yhat_c2 = yhat_result(p);
    return a;
}

void launch_fused(cphifi_unaligned p, const FusedArgs& a) {
    fused_matvec(a, p->grid, p->smem, p->smem_factors, p->obs->ctx->stream);
}

// Phase B alone (large plans, the RHS build, test hooks): k_stream.cu when planned, else the
// fused kernel restricted to PH_B.
bool build_run_parts(cphifi_unaligned p, int64_t sf_all, QpassPlan& Q);
void ensure_runs(cphifi_unaligned p);

// The run kernel's parts and split-row slots, on the first use (never inside a graph capture: every
// capture site applies the operator once before capturing, and the solve calls this in its setup).
void ensure_runs(cphifi_unaligned p) {
    if (!p->runs_pending) return;
    p->runs_pending = false;
    const auto t0 = std::chrono::steady_clock::now();
    cphifi_obs o = p->obs;
    // the plan's q-pass plan for this padded rank, shared by every subproblem on the plan; the key
    // also carries the tuning knobs the build reads
    std::string key = std::to_string(p->rp) + "/" + std::to_string(p->runs_sf);
    for (const char* v : {"CPHIFI_DENSE_MIN", "CPHIFI_DENSE_MAX_GB", "CPHIFI_RUNS_RUNCOST", "CPHIFI_RUNS_LAYOUT",
                          "CPHIFI_RUNS_VAR", "CPHIFI_XRUNS"}) {
        const char* e = std::getenv(v);
        key += std::string("/") + (e ? e : "-");
    }
    bool built = false;
    {
        std::lock_guard<std::mutex> lk(o->qp_mu);
        std::shared_ptr<QpassPlan>& slot = o->qp_cache[key];
        if (!slot) {
            auto Q = std::make_shared<QpassPlan>();
            if (!build_run_parts(p, p->runs_sf, *Q)) *Q = QpassPlan();
            for (const auto& sp : Q->parts) Q->max_warps = std::max(Q->max_warps, sp.warps);
            for (const auto& sp : Q->dense_parts) Q->max_warps = std::max(Q->max_warps, sp.warps);
            slot = Q;
            built = true;
        }
        p->qp = slot;
    }
    const QpassPlan& Q = *p->qp;
    if (!Q.parts.empty()) {  // this subproblem's scratch
        p->runs_slot_a.alloc((size_t)Q.max_warps * p->rp);
        p->runs_slot_b.alloc((size_t)Q.max_warps * p->rp);
    }
    if (Q.dense_nd > 0) {
        p->dense_partial.alloc((size_t)Q.dense_nd * (Q.dense_n1p / dense_rows_block_a()) * p->rp);
        p->dense_cnt.alloc(Q.dense_nd);
        CPHIFI_CUDA(cudaMemsetAsync(p->dense_cnt.get(), 0, sizeof(unsigned) * Q.dense_nd, o->ctx->stream));
    }
    if (std::getenv("CPHIFI_SOLVE_TIMING"))  // developer: host time of the build (or the cache hit)
        std::fprintf(stderr, "cphifi: q-pass plan %s in %.3f ms\n", built ? "built" : "shared",
                     1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
}

// The right-hand side B = sampled_mttkrp(observed values) (observations.hpp:186-188) through the run
// kernel over every part of the q-pass plan (the run kernel's parts, then the dense rows' parts:
// every entry once, weights = the entries' values, summed over duplicates in a coalesced plan), added
// into a zeroed Yhat in part order.  False when the plan has no parts or a part lacks its values.
bool rhs_over_parts(cphifi_unaligned p, FusedArgs a) {
    if (std::getenv("CPHIFI_RHS_PARTS") && std::atoi(std::getenv("CPHIFI_RHS_PARTS")) == 0) return false;
    ensure_runs(p);
    if (!p->qp || p->qp->parts.empty()) return false;
    const QpassPlan& Q = *p->qp;
    std::vector<const StreamPart*> all;
    for (const auto& sp : Q.parts) all.push_back(&sp);
    for (const auto& sp : Q.dense_parts) all.push_back(&sp);
    for (const StreamPart* sp : all)
        if (sp->q > 0 && (!sp->vals || sp->padded || sp->warps == 0)) return false;
    cudaStream_t s = p->obs->ctx->stream;
    const int dl = p->obs->d - 2;
    CPHIFI_CUDA(cudaMemsetAsync(a.yhat_rm, 0, sizeof(double) * p->n * p->rp, s));
    for (const StreamPart* spp : all) {
        const StreamPart& sp = *spp;
        if (sp.q == 0) continue;
        RunsArgs b;
        b.rp = p->rp;
        b.ldq = sp.ldq;
        b.dother = p->obs->d - 1;
        b.idx = sp.idx;
        b.mult = sp.mult;
        b.vals = sp.vals;
        b.fac = a.fac;
        for (int m = 0; m < b.dother; ++m) b.fac_off[m] = a.fac_off[m];
        b.fac_off[dl] = a.fac_off[dl] + sp.row_lo * p->rp;
        b.fac_total = b.fac_off[dl] + sp.rows * p->rp;
        b.row_ptr = sp.row_ptr;
        b.run_start = sp.run_start.get();
        b.run_i1 = sp.run_i1.get();
        b.nruns = sp.nruns;
        b.warps = sp.warps;
        b.warp_beg = sp.warp_beg.get();
        b.warp_rows = sp.warp_rows.get();
        b.row_first_w = sp.row_first_w.get();
        b.row_nw = sp.row_nw.get();
        b.xhat_rm = a.xhat_rm;
        b.yhat_rm = a.yhat_rm;
        b.slot_a = p->runs_slot_a.get();
        b.slot_b = p->runs_slot_b.get();
        b.rowcnt = a.rowcnt;
        b.accumulate = 1;
        runs_scatter_gather(b, sp.sf, s);
    }
    return true;
}

// The q-pass of the dense rows (k_dense_rows.cu): written into Yhat, not accumulated.
void launch_dense_rows(cphifi_unaligned p, const FusedArgs& a, cudaStream_t s) {
    const QpassPlan& Q = *p->qp;
    DenseRowsArgs dr;
    dr.rp = p->rp;
    dr.n1 = Q.dense_n1;
    dr.n2 = Q.dense_n2;
    dr.n1p = Q.dense_n1p;
    dr.n2p = Q.dense_n2p;
    dr.nd = Q.dense_nd;
    dr.rows = Q.dense_rows.get();
    dr.w = Q.dense_w.get();
    dr.a1 = a.fac + a.fac_off[0];
    dr.a2 = a.fac + a.fac_off[1];
    dr.xhat_rm = a.xhat_rm;
    dr.yhat_rm = a.yhat_rm;
    dr.partial = p->dense_partial.get();
    dr.cnt = p->dense_cnt.get();
    dense_rows_qpass(dr, p->obs->ctx->num_sms, s);
}

// the plan's second stream (and its fork / join events), created on first use
void ensure_side_stream(cphifi_unaligned p) {
    if (p->side) return;
    CPHIFI_CUDA(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking));
    CPHIFI_CUDA(cudaEventCreateWithFlags(&p->side_fork, cudaEventDisableTiming));
    CPHIFI_CUDA(cudaEventCreateWithFlags(&p->side_join, cudaEventDisableTiming));
}

// The operator's q-pass (not the RHS build) runs the run kernel over the plan's parts when they
// exist: with more than one part, Yhat is zeroed and every part adds into it, Yhat(i) =
// (0 + part 0) + part 1 + ... in part order.
void launch_phase_b(cphifi_unaligned p, FusedArgs a) {
    a.phases = PH_B;
    if (!a.weights) ensure_runs(p);
    if (p->qp && !p->qp->parts.empty() && !a.weights) {
        const QpassPlan& Q = *p->qp;
        cudaStream_t s = p->obs->ctx->stream;
        const int dl = p->obs->d - 2;  // the blocked (last) other mode's column / packed factor
        const bool acc = Q.parts.size() > 1;
        if (acc) CPHIFI_CUDA(cudaMemsetAsync(a.yhat_rm, 0, sizeof(double) * p->n * p->rp, s));
        // the dense rows (no entries in any part: written, not accumulated) on the plan's second
        // stream, concurrent with the parts — their CTAs fill the SMs the run kernel's last warps
        // leave idle.  Sequential under cphifi_unaligned_matvec_timed (per-kernel device times) and
        // with CPHIFI_DENSE_CONCURRENT=0.
        bool conc = Q.dense_nd > 0 && !g_dense_event;
        if (const char* e = std::getenv("CPHIFI_DENSE_CONCURRENT")) conc = conc && std::atoi(e) != 0;
        int fork_at = 0;  // (developer: CPHIFI_DENSE_FORK_AT = the part the dense launch is issued after)
        if (const char* e = std::getenv("CPHIFI_DENSE_FORK_AT")) fork_at = std::atoi(e);
        if (conc) {
            ensure_side_stream(p);
            CPHIFI_CUDA(cudaEventRecord(p->side_fork, s));
            CPHIFI_CUDA(cudaStreamWaitEvent(p->side, p->side_fork, 0));
        }
        int part_i = 0;
        for (const StreamPart& sp : Q.parts) {
            if (conc && part_i++ == fork_at) {
                launch_dense_rows(p, a, p->side);
                CPHIFI_CUDA(cudaEventRecord(p->side_join, p->side));
            }
            if (sp.q == 0) continue;
            RunsArgs b;
            b.rp = p->rp;
            b.ldq = sp.ldq;
            b.dother = p->obs->d - 1;
            b.idx = sp.idx;
            b.mult = sp.mult;
            b.fac = a.fac;
            for (int m = 0; m < b.dother; ++m) b.fac_off[m] = a.fac_off[m];
            b.fac_off[dl] = a.fac_off[dl] + sp.row_lo * p->rp;
            b.fac_total = b.fac_off[dl] + sp.rows * p->rp;
            b.row_ptr = sp.row_ptr;
            b.run_start = sp.run_start.get();
            b.run_i1 = sp.run_i1.get();
            b.nruns = sp.nruns;
            b.warps = sp.warps;
            b.warp_beg = sp.warp_beg.get();
            b.warp_rows = sp.warp_rows.get();
            b.row_first_w = sp.row_first_w.get();
            b.row_nw = sp.row_nw.get();
            b.xhat_rm = a.xhat_rm;
            b.yhat_rm = a.yhat_rm;
            b.slot_a = p->runs_slot_a.get();
            b.slot_b = p->runs_slot_b.get();
            b.rowcnt = a.rowcnt;
            b.accumulate = acc ? 1 : 0;
            if (sp.padded) xruns_scatter_gather(b, sp.sf, s);
            else runs_scatter_gather(b, sp.sf, s);
        }
        if (g_dense_event) {  // cphifi_unaligned_matvec_timed: the run kernel / dense rows split
            CPHIFI_CUDA(cudaEventRecord(g_dense_event, s));
            g_dense_recorded = true;
        }
        if (conc && part_i <= fork_at) {  // (fork point past the last part)
            launch_dense_rows(p, a, p->side);
            CPHIFI_CUDA(cudaEventRecord(p->side_join, p->side));
        }
        if (conc) CPHIFI_CUDA(cudaStreamWaitEvent(s, p->side_join, 0));
        else if (Q.dense_nd > 0) launch_dense_rows(p, a, s);
        return;
    }
    if (p->stream) stream_scatter_gather(a, p->grid, p->stream_sf, p->obs->ctx->stream);
    else launch_fused(p, a);
}

// The run kernel's parts (StreamPart, common.cuh; k_runs.cu).  When the per-observation factors
// fit shared memory next to the kernel's per-warp buffers, one part aliases the plan.  Otherwise
// the last other mode's factor is cut into H row blocks that do fit, and the plan is stably
// partitioned by block (radix sort on the block id: plan order kept inside each part); each part
// stages its block (config 4: A_3's 512 rows as 2 x 256, 128 KB each) instead of gathering rows
// through L1 / L2 — 125 GB of L2 traffic per application, above the L2's bandwidth for 10 ms.
// Then, per part: the run table and the equal-count warp ranges.  Returns false (no parts) when no
// block size fits.
void finish_part(cphifi_unaligned p, StreamPart& sp, const int32_t* rows, int64_t nw) {
    cphifi_ctx ctx = p->obs->ctx;
    cudaStream_t s = ctx->stream;
    const int64_t q = sp.q;
    if (q > 0) {
        DevBuf<int32_t> rs_tmp(q + 1);
        const int64_t nr = build_run_starts(rows, sp.idx, q, rs_tmp.get(), s);
        sp.nruns = nr;
        sp.run_start.alloc(nr + 1);
        CPHIFI_CUDA(cudaMemcpyAsync(sp.run_start.get(), rs_tmp.get(), sizeof(int32_t) * nr, cudaMemcpyDeviceToDevice, s));
        const int32_t qq = (int32_t)q;
        h2d(sp.run_start.get() + nr, &qq, sizeof(int32_t), s);
        sp.run_i1.alloc(std::max<int64_t>(nr, 1));
        gather_i32(sp.idx, sp.run_start.get(), 0, nr, sp.run_i1.get(), s);
    }
    if (!sp.padded) sp.draws = q;  // (a padded part's draws are counted before its flags are set)
    if (sp.mult && q > 0 && !sp.padded) {
        DevBuf<unsigned long long> sum(1);
        CPHIFI_CUDA(cudaMemsetAsync(sum.get(), 0, sizeof(unsigned long long), s));
        sum_i32(sp.mult, q, sum.get(), s);
        unsigned long long h = 0;
        d2h_sync(&h, sum.get(), sizeof(h), s);
        sp.draws = (int64_t)h;
    }
    std::vector<int64_t> rp_host(p->n + 1);
    d2h_sync(rp_host.data(), sp.row_ptr, sizeof(int64_t) * (p->n + 1), s);
    // warp ranges of equal COST, cost = entries + C x runs started: a warp's time grows with its
    // runs as well as its entries (per-run work: the A_1 row, u, the partial last step), so an
    // equal-count split leaves the warps in sparse rows (short runs) far behind the others
    double cpr = 12.0;
    if (const char* e = std::getenv("CPHIFI_RUNS_RUNCOST")) cpr = std::atof(e);
    std::vector<int64_t> starts;
    if (q > 0 && cpr > 0.0) {
        std::vector<int32_t> rs(sp.nruns + 1);
        d2h_sync(rs.data(), sp.run_start.get(), sizeof(int32_t) * (sp.nruns + 1), s);
        const double total = (double)q + cpr * (double)sp.nruns;
        starts.push_back(0);
        int64_t j = 0;  // run holding the current target
        for (int64_t wi = 1; wi < nw; ++wi) {
            const double tgt = total * (double)wi / (double)nw;
            while (j + 1 < sp.nruns && (double)rs[j + 1] + cpr * (double)(j + 1) <= tgt) ++j;
            const double c0 = (double)rs[j] + cpr * (double)j;  // cost at run j's start
            int64_t e = rs[j] + (int64_t)std::max(0.0, tgt - c0 - cpr);
            e = std::min<int64_t>(std::max<int64_t>(e, rs[j]), rs[j + 1]);
            if (sp.padded) e &= ~(int64_t)1;  // pairs of entries never straddle a warp range
            starts.push_back(std::max(e, starts.back()));
        }
        starts.push_back(q);
    }
    PartitionPlan plan;
    plan_partition(rp_host, (int)nw, (int)nw, plan, (int)nw, starts.empty() ? nullptr : &starts);
    sp.warps = plan.ctas;
    sp.warp_beg.alloc(plan.beg.size());
    h2d(sp.warp_beg.get(), plan.beg.data(), sizeof(int64_t) * plan.beg.size(), s);
    sp.warp_rows.alloc(plan.rows.size());
    h2d(sp.warp_rows.get(), plan.rows.data(), sizeof(int64_t) * plan.rows.size(), s);
    sp.row_first_w.alloc(p->n);
    h2d(sp.row_first_w.get(), plan.row_first_cta.data(), sizeof(int32_t) * p->n, s);
    sp.row_nw.alloc(p->n);
    h2d(sp.row_nw.get(), plan.row_ncta.data(), sizeof(int32_t) * p->n, s);
    CPHIFI_CUDA(cudaStreamSynchronize(s));  // host plan vectors go out of scope
}

// Dense rows (k_dense_rows.cu): 3-way plans only; a row goes to the GEMM form when its distinct
// cells cover at least CPHIFI_DENSE_MIN (default 0.3) of its n_1 x n_2 grid — the measured break-even
// of two DMMA GEMMs per row against the run kernel's per-entry cost — and the grids
// of all such rows fit CPHIFI_DENSE_MAX_GB (default 16 GB, int32 per cell).  Picks the rows, builds
// their multiplicity grids and returns the per-row slot table (-1: sparse) on the device, or an empty
// buffer when no row qualifies.
DevBuf<int32_t> build_dense_rows(cphifi_unaligned p, const int32_t* rows_of_entry, QpassPlan& Q) {
    cphifi_obs o = p->obs;
    cphifi_ctx ctx = o->ctx;
    cudaStream_t s = ctx->stream;
    DevBuf<int32_t> slot;
    Q.dense_nd = 0;
    double dmin = 0.3, max_gb = 16.0;
    if (const char* e = std::getenv("CPHIFI_DENSE_MIN")) dmin = std::atof(e);
    if (const char* e = std::getenv("CPHIFI_DENSE_MAX_GB")) max_gb = std::atof(e);
    if (!(dmin > 0.0) || !dense_rows_supported(p->rp, o->d - 1) || !o->lex) return slot;
    int m1 = -1, m2 = -1;  // the other modes, ascending (plan columns 0 and 1)
    for (int m = 0; m < o->d; ++m)
        if (m != o->k) (m1 < 0 ? m1 : m2) = m;
    const int64_t n1 = o->shape[m1], n2 = o->shape[m2];
    const int64_t ba = dense_rows_block_a(), bb = dense_rows_block_b();
    const int64_t n1p = (n1 + ba - 1) / ba * ba, n2p = (n2 + bb - 1) / bb * bb;
    std::vector<int64_t> rph(p->n + 1);
    d2h_sync(rph.data(), o->row_ptr.get(), sizeof(int64_t) * (p->n + 1), s);
    const double cells = (double)n1 * (double)n2;
    std::vector<int32_t> drows, slot_h(p->n, -1);
    const int64_t cap = (int64_t)(max_gb * 1e9 / (4.0 * (double)n1p * (double)n2p));
    for (int64_t i = 0; i < p->n && (int64_t)drows.size() < cap; ++i)
        if ((double)(rph[i + 1] - rph[i]) >= dmin * cells) {
            slot_h[i] = (int32_t)drows.size();
            drows.push_back((int32_t)i);
        }
    if (drows.empty()) return slot;
    const int nd = (int)drows.size();
    Q.dense_nd = nd;
    Q.dense_n1 = n1;
    Q.dense_n2 = n2;
    Q.dense_n1p = n1p;
    Q.dense_n2p = n2p;
    Q.dense_rows.alloc(nd);
    h2d(Q.dense_rows.get(), drows.data(), sizeof(int32_t) * nd, s);
    slot.alloc(p->n);
    h2d(slot.get(), slot_h.data(), sizeof(int32_t) * p->n, s);
    Q.dense_w.alloc((size_t)nd * n1p * n2p);
    CPHIFI_CUDA(cudaMemsetAsync(Q.dense_w.get(), 0, sizeof(int32_t) * (size_t)nd * n1p * n2p, s));
    dense_grid_build(o->idx_o.get(), o->ldq, o->coalesced ? o->mult.get() : nullptr, rows_of_entry, slot.get(),
                     o->q_local, n1p, n2p, Q.dense_w.get(), s);
    CPHIFI_CUDA(cudaStreamSynchronize(s));  // host vectors go out of scope
    return slot;
}

bool build_run_parts(cphifi_unaligned p, int64_t sf_all, QpassPlan& Q) {
    cphifi_obs o = p->obs;
    cphifi_ctx ctx = o->ctx;
    cudaStream_t s = ctx->stream;
    const int d = o->d, k = o->k, dl = d - 2;  // dl: column of the blocked mode in idx_o
    const bool mult = o->coalesced;
    const int64_t nw = (int64_t)ctx->num_sms * runs_warps_per_sm(p->rp);
    int lm = -1;  // the blocked mode itself (last mode != k)
    for (int m = d - 1; m >= 0 && lm < 0; --m)
        if (m != k) lm = m;
    const int64_t nl = o->shape[lm], rp = p->rp, q = o->q_local;
    DevBuf<int32_t> rows(std::max<int64_t>(q, 1));
    row_of_entries(o->row_ptr.get(), p->n, q, rows.get(), s);
    const DevBuf<int32_t> dslot = build_dense_rows(p, rows.get(), Q);
    const bool dense = Q.dense_nd > 0;
    const bool fits = runs_smem_bytes(rp, d - 1, mult, sf_all) <= runs_smem_cap();
    if (fits && !dense) {  // one part: the plan itself
        std::vector<StreamPart> parts(1);
        StreamPart& sp = parts[0];
        sp.q = q;
        sp.q_real = q;
        sp.ldq = o->ldq;
        sp.rows = nl;
        sp.idx = o->idx_o.get();
        sp.mult = mult ? o->mult.get() : nullptr;
        sp.vals = o->values.n ? o->values.get() : nullptr;
        sp.row_ptr = o->row_ptr.get();
        sp.sf = sf_all;
        finish_part(p, sp, rows.get(), nw);
        Q.parts = std::move(parts);
        return true;
    }
    const int64_t rest = sf_all - nl * rp;  // staged doubles of the other per-observation modes
    int64_t br = fits ? nl : 0;
    for (int64_t b = nl; b >= 8 && br == 0; b -= 8)
        if (runs_smem_bytes(rp, d - 1, mult, rest + b * rp) <= runs_smem_cap()) br = b;
    if (br < 8 && !fits) {
        Q.dense_nd = 0;  // no parts: the stream kernel takes the whole plan
        return false;
    }
    const int H = (int)((nl + br - 1) / br);
    br = (nl + H - 1) / H;  // balanced blocks
    // opt-in (CPHIFI_XRUNS=1; measured slower at config 4, k_xruns.cu): the cross-run kernel for 3-way
    // coalesced plans whose blocks fit its buffers, over parts padded to even run lengths
    bool xruns = mult && xruns_supported(rp, d - 1, mult) && xruns_smem_bytes(rp, rest + br * rp) <= runs_smem_cap() &&
                 xruns_warps_per_sm() == runs_warps_per_sm(rp);
    {
        const char* e = std::getenv("CPHIFI_XRUNS");
        xruns = xruns && e && std::atoi(e) != 0;
    }
    // part key = block of the last other mode; the dense rows' entries get key H (dropped)
    DevBuf<int32_t> key(std::max<int64_t>(q, 1)), key_s(std::max<int64_t>(q, 1)), perm_in(std::max<int64_t>(q, 1)),
        perm(std::max<int64_t>(q, 1)), rows_h(std::max<int64_t>(q, 1));
    block_key(o->idx_o.get() + (int64_t)dl * o->ldq, q, (int32_t)br, key.get(), s);
    // the dense rows' entries go to buckets H + block (their own parts, for the row-Gram build)
    if (dense) dense_key(rows.get(), dslot.get(), q, (int32_t)H, key.get(), s);
    const int nb = dense ? 2 * H : H;
    iota32(perm_in.get(), q, s);
    int bits = 1;
    while ((1 << bits) < nb) ++bits;
    if (q > 0) {
        const size_t tb = radix_sort_pairs_bytes(q, bits);
        DevBuf<unsigned char> tmp(tb);
        radix_sort_pairs(tmp.get(), tb, key.get(), key_s.get(), perm_in.get(), perm.get(), q, bits, s);
    }
    DevBuf<int64_t> bnd(nb + 1);
    csr_from_sorted(key_s.get(), q, nb, bnd.get(), s);  // bnd[b] = first entry of bucket b
    std::vector<int64_t> hb(nb + 1);
    d2h_sync(hb.data(), bnd.get(), sizeof(int64_t) * (nb + 1), s);
    auto make_part = [&](StreamPart& sp, int b, bool runs) {
        const int h = b % H;
        const int64_t lo = hb[b], cnt = hb[b + 1] - hb[b];
        sp.q = cnt;
        sp.q_real = cnt;
        sp.ldq = (cnt + 3) / 4 * 4;
        sp.row_lo = h * br;
        sp.rows = std::min(br, nl - sp.row_lo);
        sp.sf = rest + sp.rows * rp;
        sp.idx_own.alloc((int64_t)(d - 1) * sp.ldq + OBS_PAD);
        for (int m = 0; m < d - 1; ++m)
            gather_i32(o->idx_o.get() + (int64_t)m * o->ldq, perm.get(), lo, cnt, sp.idx_own.get() + (int64_t)m * sp.ldq,
                       s);
        add_i32(sp.idx_own.get() + (int64_t)dl * sp.ldq, cnt, (int32_t)(-sp.row_lo), s);
        sp.idx = sp.idx_own.get();
        if (mult) {
            sp.mult_own.alloc(cnt + OBS_PAD);
            gather_i32(o->mult.get(), perm.get(), lo, cnt, sp.mult_own.get(), s);
            sp.mult = sp.mult_own.get();
        }
        gather_i32(rows.get(), perm.get(), lo, cnt, rows_h.get(), s);
        if (o->values.n && !(runs && xruns) && cnt > 0) {  // the observed values, for B over the parts
            sp.vals_own.alloc(cnt + OBS_PAD);
            gather_f64(o->values.get(), perm.get(), lo, cnt, sp.vals_own.get(), s);
            sp.vals = sp.vals_own.get();
        }
        if (runs && xruns && cnt > 0) {  // runs padded to even lengths for k_xruns.cu
            DevBuf<int32_t> rs(cnt + 1);
            const int64_t nr = build_run_starts(rows_h.get(), sp.idx_own.get(), cnt, rs.get(), s);
            const int32_t qq = (int32_t)cnt;
            h2d(rs.get() + nr, &qq, sizeof(int32_t), s);
            DevBuf<unsigned long long> sum(1);
            CPHIFI_CUDA(cudaMemsetAsync(sum.get(), 0, sizeof(unsigned long long), s));
            sum_i32(sp.mult, cnt, sum.get(), s);
            unsigned long long hsum = 0;
            d2h_sync(&hsum, sum.get(), sizeof(hsum), s);
            const int64_t qmax = cnt + nr, ldq2 = (qmax + 3) / 4 * 4;
            DevBuf<int32_t> idx2(2 * ldq2 + OBS_PAD), mult2(qmax + OBS_PAD), rows2(qmax);
            const int64_t q2 = pad_runs_even(rs.get(), nr, sp.idx_own.get(), sp.idx_own.get() + sp.ldq, sp.mult,
                                             rows_h.get(), idx2.get(), idx2.get() + ldq2, mult2.get(), rows2.get(),
                                             cnt, s);
            sp.q = q2;
            sp.ldq = ldq2;
            sp.idx_own = std::move(idx2);
            sp.idx = sp.idx_own.get();
            sp.mult_own = std::move(mult2);
            sp.mult = sp.mult_own.get();
            sp.draws = (int64_t)hsum;
            sp.padded = true;
            sp.row_ptr_own.alloc(p->n + 1);
            csr_from_sorted(rows2.get(), q2, p->n, sp.row_ptr_own.get(), s);
            sp.row_ptr = sp.row_ptr_own.get();
            finish_part(p, sp, rows2.get(), nw);
            return;
        }
        sp.row_ptr_own.alloc(p->n + 1);
        csr_from_sorted(rows_h.get(), cnt, p->n, sp.row_ptr_own.get(), s);
        sp.row_ptr = sp.row_ptr_own.get();
        if (runs) finish_part(p, sp, rows_h.get(), nw);
        else CPHIFI_CUDA(cudaStreamSynchronize(s));  // rows_h is reused by the next part
    };
    std::vector<StreamPart> parts(H), dparts(dense ? H : 0);
    for (int h = 0; h < H; ++h) make_part(parts[h], h, true);
    // the dense rows' parts get run tables and warp ranges too: the right-hand side B runs the run
    // kernel over every entry (k_runs.cu, RunsArgs::vals)
    for (int h = 0; h < (dense ? H : 0); ++h) make_part(dparts[h], H + h, true);
    Q.parts = std::move(parts);
    Q.dense_parts = std::move(dparts);
    return true;
}

// The row-Gram build over the q-pass plan's factor-block parts (the run kernel's parts plus the dense
// rows' parts: every entry once), one launch per part adding into G (zeroed by the caller):
//  * default (CPHIFI_GRAM3_PARTS=0: off), 3-way plans whose factors do not fit shared memory (config 4:
//    2 x 256 KB): the register-fragment build (k_gram3.cu) with the part's block staged and mode 0
//    through L1, over an equal-count unit partition of the part (cached on the part);
//  * opt-in (CPHIFI_GRAM_WS=1): the warp-specialised build (k_gramws.cu) — measured slower than the
//    single-pass builds of k_gram.cu: config 4 71.6 vs 61.8 ms, config 3 26.9 vs 24.6 ms (tensor
//    pipe 32 %: the producers' global loads and the handshakes of 32-entry batches).
// False when neither applies (no parts, rank or order out of range, staging too large): the caller
// falls back to the single-pass builds.
bool gram_build_parts(cphifi_unaligned p) {
    bool ws = false;
    if (const char* e = std::getenv("CPHIFI_GRAM_WS")) ws = std::atoi(e) != 0;
    // The register-fragment build over the parts is the default for 3-way plans whose factors do not
    // fit shared memory (config 4: 40.7 ms against 62.1 for k_gram.cu's batched build, with each
    // warp's tile pairs a compile-time set and single-warp teams; the q-pass plan it walks is shared with the stream
    // operator and cached on the observation plan).  CPHIFI_GRAM3_PARTS=0 turns it off; =3 selects
    // the run-hoisted form (72.6 ms: the fold per run end and a second masked pass per straddled
    // k-step, measured slower).
    bool v3 = !ws && p->obs->d == 3;
    int v3stage = 1;
    if (const char* e = std::getenv("CPHIFI_GRAM3_PARTS")) {
        v3 = v3 && std::atoi(e) != 0;
        if (std::atoi(e) == 3) v3stage = 3;
    }
    cphifi_obs o = p->obs;
    if (ws && !gram_ws_supported(p->rp, o->d - 1)) return false;
    if (!ws && !v3) return false;
    if (v3) {  // only where the whole-plan staging of k_gram3.cu does not fit
        GramArgs probe;
        probe.rp = p->rp;
        probe.dother = o->d - 1;
        probe.fac = p->fac.get();
        for (int m = 0; m < o->d - 1; ++m) probe.fac_off[m] = p->fac_off[m];
        probe.fac_total = (int64_t)p->fac.n;
        // whole-plan staging fits: ensure_gram's single launch instead
        if (gram3_stage(p->rp, o->d - 1, probe) == 2) return false;
        if (!(p->rp == 16 || p->rp == 32 || p->rp == 64) || reinterpret_cast<uintptr_t>(p->fac.get()) % 16) return false;
        for (int m = 0; m < o->d - 1; ++m)
            if (p->fac_off[m] % 2) return false;
    }
    ensure_runs(p);
    if (!p->qp || p->qp->parts.empty()) return false;
    QpassPlan& Q = *p->qp;
    if (ws && Q.dense_nd > 0) return false;  // (the warp-specialised path: run-kernel parts only)
    std::vector<StreamPart*> all;
    for (auto& sp : Q.parts) all.push_back(&sp);
    for (auto& sp : Q.dense_parts) all.push_back(&sp);
    for (const StreamPart* sp : all) {
        if (ws && gram_ws_smem_bytes(p->rp, sp->sf) > runs_smem_cap()) return false;
        if (v3 && sizeof(double) * (size_t)sp->sf > 220 * 1024) return false;
    }
    cphifi_ctx ctx = o->ctx;
    cudaStream_t s = ctx->stream;
    const int dl = o->d - 2;
    const size_t rp2 = (size_t)p->rp * p->rp;
    const int units = v3 ? ctx->num_sms * gram3_units_per_sm(p->rp) : ctx->num_sms;
    DevBuf<unsigned> rowcnt(p->n);
    CPHIFI_CUDA(cudaMemsetAsync(rowcnt.get(), 0, sizeof(unsigned) * p->n, s));
    DevBuf<double> slot_a((size_t)units * rp2), slot_b((size_t)units * rp2);
    const bool timing = std::getenv("CPHIFI_GRAM_TIMING") != nullptr;  // developer: device time of the build
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timing) {
        CPHIFI_CUDA(cudaEventCreate(&e0));
        CPHIFI_CUDA(cudaEventCreate(&e1));
        CPHIFI_CUDA(cudaEventRecord(e0, s));
    }
    // opt-in (CPHIFI_GRAM_CONCURRENT=1): the dense rows' parts (rows disjoint from the run-kernel
    // parts': G rows and row counters disjoint) on the plan's second stream with their own unit
    // slots, concurrent with the sparse parts — each stream keeps its parts in part order, so every
    // G_i sums in the same order (bit-identical).  Measured slower at config 4 (53.5 against 41.8 ms,
    // profiles/round2c/gram_concurrent.txt): every part's unit partition is planned as exactly one
    // wave of the whole GPU, and two builds sharing the SMs turn each into two uneven waves.
    bool conc = false;
    if (const char* e = std::getenv("CPHIFI_GRAM_CONCURRENT")) conc = !timing && !Q.dense_parts.empty() && !Q.parts.empty() && std::atoi(e) != 0;
    DevBuf<double> slot_a2, slot_b2;
    for (StreamPart* sp : all) {  // every part's unit partition first (host round trips), then the launches
        if (sp->q == 0) continue;
        {  // the part's unit partition, built once and kept with the (shared) plan
            std::lock_guard<std::mutex> lk(o->qp_mu);
            if (sp->g_units != units) {
                std::vector<int64_t> rp_host(p->n + 1);
                d2h_sync(rp_host.data(), sp->row_ptr, sizeof(int64_t) * (p->n + 1), s);
                PartitionPlan plan;
                if (v3) plan_partition(rp_host, units, units, plan, units);
                else plan_partition(rp_host, units, units, plan);
                sp->g_beg.alloc(plan.beg.size());
                sp->g_rows.alloc(plan.rows.size());
                sp->g_rfc.alloc(p->n);
                sp->g_rnc.alloc(p->n);
                h2d(sp->g_beg.get(), plan.beg.data(), sizeof(int64_t) * plan.beg.size(), s);
                h2d(sp->g_rows.get(), plan.rows.data(), sizeof(int64_t) * plan.rows.size(), s);
                h2d(sp->g_rfc.get(), plan.row_first_cta.data(), sizeof(int32_t) * p->n, s);
                h2d(sp->g_rnc.get(), plan.row_ncta.data(), sizeof(int32_t) * p->n, s);
                CPHIFI_CUDA(cudaStreamSynchronize(s));  // host vectors released
                sp->g_units = units;  // (the launch takes the partition's own count, g_beg.n - 1)
            }
        }
    }
    for (StreamPart* sp : all) {
        if (sp->q == 0) continue;
        GramArgs g;
        g.n = p->n;
        g.rp = p->rp;
        g.q = sp->ldq;
        g.dother = o->d - 1;
        g.row_ptr = sp->row_ptr;
        g.idx = sp->idx;
        g.fac = p->fac.get();
        for (int m = 0; m < o->d - 1; ++m) g.fac_off[m] = p->fac_off[m];
        g.fac_off[dl] = p->fac_off[dl] + sp->row_lo * p->rp;
        g.fac_total = g.fac_off[dl] + sp->rows * p->rp;
        g.mult = sp->mult;
        g.cta_beg = sp->g_beg.get();
        g.cta_rows = sp->g_rows.get();
        g.row_first_cta = sp->g_rfc.get();
        g.row_ncta = sp->g_rnc.get();
        g.rowcnt = rowcnt.get();
        g.slot_a = slot_a.get();
        g.slot_b = slot_b.get();
        g.g = p->gram.get();
        g.accumulate = 1;  // G was zeroed: every part adds, in part order
        cudaStream_t ls = s;
        if (conc && sp >= &Q.dense_parts.front() && sp <= &Q.dense_parts.back()) {
            if (!slot_a2.n) {  // first dense part: fork the side stream off the main one
                slot_a2.alloc((size_t)units * rp2);
                slot_b2.alloc((size_t)units * rp2);
                ensure_side_stream(p);
                CPHIFI_CUDA(cudaEventRecord(p->side_fork, s));
                CPHIFI_CUDA(cudaStreamWaitEvent(p->side, p->side_fork, 0));
            }
            g.slot_a = slot_a2.get();
            g.slot_b = slot_b2.get();
            ls = p->side;
        }
        cudaEvent_t p0 = nullptr, p1 = nullptr;
        if (timing) {
            CPHIFI_CUDA(cudaEventCreate(&p0));
            CPHIFI_CUDA(cudaEventCreate(&p1));
            CPHIFI_CUDA(cudaEventRecord(p0, s));
        }
        if (v3) gram3_build(g, (int)(sp->g_beg.n - 1), v3stage, ls);
        else gram_build_ws(g, (int)(sp->g_beg.n - 1), sp->sf, ls);
        if (timing) {
            CPHIFI_CUDA(cudaEventRecord(p1, s));
            CPHIFI_CUDA(cudaEventSynchronize(p1));
            float ms = 0.f;
            CPHIFI_CUDA(cudaEventElapsedTime(&ms, p0, p1));
            std::fprintf(stderr, "cphifi: gram build part (%lld entries) %.3f ms\n", (long long)sp->q, ms);
            cudaEventDestroy(p0);
            cudaEventDestroy(p1);
        }
    }
    if (slot_a2.n) {  // join
        CPHIFI_CUDA(cudaEventRecord(p->side_join, p->side));
        CPHIFI_CUDA(cudaStreamWaitEvent(s, p->side_join, 0));
    }
    CPHIFI_CUDA(cudaStreamSynchronize(s));  // the slots / counters are released on return
    if (timing) {
        CPHIFI_CUDA(cudaEventRecord(e1, s));
        CPHIFI_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        CPHIFI_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        std::fprintf(stderr, "cphifi: gram build (%s, %zu parts) %.3f ms on device\n", v3 ? "v3 over parts" : "warp-specialised",
                     all.size(), ms);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
    return true;
}

// Row-Gram operator: build G_i = sum_l z_l z_l' once (k_gram.cu), on first use.
void ensure_gram(cphifi_unaligned p) {
    if (p->gram.n) return;
    if (p->rp > 64) throw_invalid("gram operator: padded rank above 64 is not supported");
    cphifi_obs o = p->obs;
    cphifi_ctx ctx = o->ctx;
    cudaStream_t s = ctx->stream;
    const size_t rp2 = (size_t)p->rp * p->rp;
    p->gram.alloc((size_t)p->n * rp2);
    CPHIFI_CUDA(cudaMemsetAsync(p->gram.get(), 0, sizeof(double) * p->n * rp2, s));
    if (gram_build_parts(p)) return;
    // The build's own row-aligned partition, sized from the chosen kernel's occupancy (each CTA
    // alternates a gather phase and a DMMA phase around barriers, so several per SM overlap them).  Measured (profiles/prof_gram_grid.sh): config 3 (v1) 27.4 ms at 4 CTAs/SM
    // -> 24.7 at 8; config 4 (v2, 2 resident) 68.3 at 4 -> 61.8 at 2 (no partial second wave).
    GramArgs probe;
    probe.rp = p->rp;
    probe.dother = o->d - 1;
    probe.fac = p->fac.get();
    for (int m = 0; m < o->d - 1; ++m) probe.fac_off[m] = p->fac_off[m];
    probe.fac_total = (int64_t)p->fac.n;
    // the register-fragment build (k_gram3.cu) over an equal-count partition of gram3_units_per_sm
    // units per SM; else the single-pass builds of k_gram.cu over their row-aligned partition
    const int stage3 = gram3_stage(p->rp, o->d - 1, probe);
    bool v3 = stage3 == 2;  // (stage 1 — modes 1.. staged — needs factor-block parts)
    if (const char* e = std::getenv("CPHIFI_GRAM3")) v3 = v3 && std::atoi(e) != 0;
    int per_sm = v3 ? gram3_units_per_sm(p->rp) : gram_build_occupancy(probe);
    if (const char* e = std::getenv("CPHIFI_GRAM_CTAS_PER_SM")) per_sm = std::max(1, std::atoi(e));
    const int cmax = per_sm * ctx->num_sms;
    PartitionPlan plan;
    {
        std::vector<int64_t> rp_host(p->n + 1);
        d2h_sync(rp_host.data(), o->row_ptr.get(), sizeof(int64_t) * (p->n + 1), s);
        if (v3) plan_partition(rp_host, cmax, cmax, plan, cmax);
        else plan_partition(rp_host, cmax, std::min(cmax, ctx->num_sms), plan);
    }
    const int grid = plan.ctas;
    DevBuf<int64_t> cta_beg(plan.beg.size()), cta_rows(plan.rows.size());
    DevBuf<int32_t> rfc(p->n), rnc(p->n);
    DevBuf<unsigned> rowcnt(p->n);
    h2d(cta_beg.get(), plan.beg.data(), sizeof(int64_t) * plan.beg.size(), s);
    h2d(cta_rows.get(), plan.rows.data(), sizeof(int64_t) * plan.rows.size(), s);
    h2d(rfc.get(), plan.row_first_cta.data(), sizeof(int32_t) * p->n, s);
    h2d(rnc.get(), plan.row_ncta.data(), sizeof(int32_t) * p->n, s);
    CPHIFI_CUDA(cudaMemsetAsync(rowcnt.get(), 0, sizeof(unsigned) * p->n, s));
    DevBuf<double> slot_a((size_t)grid * rp2), slot_b((size_t)grid * rp2);
    GramArgs g;
    g.n = p->n;
    g.rp = p->rp;
    g.q = o->ldq;
    g.dother = o->d - 1;
    g.row_ptr = o->row_ptr.get();
    g.idx = o->idx_o.get();
    g.fac = p->fac.get();
    for (int m = 0; m < o->d - 1; ++m) g.fac_off[m] = p->fac_off[m];
    g.fac_total = (int64_t)p->fac.n;
    g.mult = o->coalesced ? o->mult.get() : nullptr;
    g.cta_beg = cta_beg.get();
    g.cta_rows = cta_rows.get();
    g.row_first_cta = rfc.get();
    g.row_ncta = rnc.get();
    g.rowcnt = rowcnt.get();
    g.slot_a = slot_a.get();
    g.slot_b = slot_b.get();
    g.g = p->gram.get();
    const bool timing = std::getenv("CPHIFI_GRAM_TIMING") != nullptr;  // developer: device time of the build
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timing) {
        CPHIFI_CUDA(cudaEventCreate(&e0));
        CPHIFI_CUDA(cudaEventCreate(&e1));
        CPHIFI_CUDA(cudaEventRecord(e0, s));
    }
    if (o->q_local > 0) {
        if (v3) gram3_build(g, grid, stage3, s);
        else gram_build(g, grid, s);
    }
    if (timing) CPHIFI_CUDA(cudaEventRecord(e1, s));
    CPHIFI_CUDA(cudaStreamSynchronize(s));  // the plan buffers are released on return
    if (timing) {
        float ms = 0.f;
        CPHIFI_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        std::fprintf(stderr, "cphifi: gram build %.3f ms on device (grid %d)\n", ms, grid);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
}

// CPHIFI_OP_AUTO: the row-Gram form pays off when the rows carry on average >= 2 rp observations
// (each application then costs O(n rp^2) instead of O(q d rp)) and G fits comfortably; small n
// keeps the single fused launch.  Plans start with this choice (cphifi_unaligned_create).
int auto_operator(cphifi_unaligned p) {
    if (!p->mode || p->small_n) return CPHIFI_OP_STREAM;
    const double g_bytes = 8.0 * (double)p->n * (double)p->rp * (double)p->rp;
    return (p->rp <= 64 && p->obs->q_local >= 2 * p->rp * p->n && g_bytes <= 8e9) ? CPHIFI_OP_GRAM : CPHIFI_OP_STREAM;
}

// Phase sets of the operator launches (see kernels.cuh).  part 0 = the (first) launch,
// part 1 = the launch after the NCCL all-reduce (multi-GPU, small n).
unsigned matvec_phases(cphifi_unaligned p, bool multi, int part) {
    const unsigned ax = p->local_x ? PH_AL : PH_A;
    if (!p->small_n) return PH_B;
    if (!multi) return ax | PH_B | PH_C2;
    return part == 0 ? (ax | PH_B) : ((p->local_x ? PH_AL : 0u) | PH_C2);
}

// Xhat = K X -> column-major copy (lambda term) + row-major padded copy (kernel input)
void xhat_gemm(cphifi_unaligned p, const double* x) {
    cphifi_ctx ctx = p->obs->ctx;
    GemmArgs g;
    g.m = p->n; g.n = p->r; g.k = p->n;
    g.a = p->mode->kernel.get(); g.a_rs = 1; g.a_cs = p->n;
    g.b = x; g.b_rs = 1; g.b_cs = p->n;
    g.c = p->xhat_cm.get(); g.c_rs = 1; g.c_cs = p->n;
    g.c2 = p->xhat_rm.get(); g.ld2 = p->rp;
    gemm(g, ctx->num_sms, ctx->stream);
}

// y = (K Yhat + lambda Xhat) + rho x
void y_gemm(cphifi_unaligned p, const double* x, double* y) {
    cphifi_ctx ctx = p->obs->ctx;
    GemmArgs g;
    g.m = p->n; g.n = p->r; g.k = p->n;
    g.a = p->mode->kernel.get(); g.a_rs = 1; g.a_cs = p->n;
    g.b = yhat_result(p); g.b_rs = p->rp; g.b_cs = 1;
    g.c = y; g.c_rs = 1; g.c_cs = p->n;
    g.epi = EPI_AXPY2;
    g.e1 = p->xhat_cm.get(); g.e2 = x; g.ld_e = p->n;
    g.beta1 = p->mode->lambda; g.beta2 = p->rho;
    gemm(g, ctx->num_sms, ctx->stream);
}

// Row-sharded operator (large n, sharded observations; stream and row-Gram operators): the shards are contiguous
// in the plan order, so rank s's observations touch only the rows [own_lo, hull_hi) — it needs only
// those rows of Xhat = K X and its partial Yhat is zero elsewhere.  Both dense contractions shrink
// to the rank's rows: Xhat[rows,:] = K[rows,:] X, then, with lambda K X folded into the operand,
//     y_s = K[:, rows] (Yhat_s[rows,:] + lambda X[owned rows,:])  (+ rho x on shard 0),
// and ONE n x r all-reduce of y_s replaces the Yhat all-reduce: sum_s y_s =
// K (Yhat + lambda X) + rho x.  Without it the two n x n x r GEMMs are replicated on every rank
// (config 4: 0.18 of the 0.9 ms an 8-way shard takes).  CPHIFI_ROW_SHARDED=0 restores the replicated form.
bool row_sharded(cphifi_unaligned p) {
    cphifi_obs o = p->obs;
    if (o->shards <= 1 || p->small_n) return false;
    if (ctx_multi(o->ctx) && o->ctx->nranks != o->shards) return false;
    const char* e = std::getenv("CPHIFI_ROW_SHARDED");
    return !(e && std::atoi(e) == 0);
}

void xhat_gemm_rows(cphifi_unaligned p, const double* x) {
    cphifi_ctx ctx = p->obs->ctx;
    const int64_t lo = p->obs->own_lo, hi = p->obs->hull_hi;
    GemmArgs g;
    g.m = hi - lo; g.n = p->r; g.k = p->n;
    g.a = p->mode->kernel.get() + lo; g.a_rs = 1; g.a_cs = p->n;
    g.b = x; g.b_rs = 1; g.b_cs = p->n;
    g.c = p->xhat_cm.get() + lo; g.c_rs = 1; g.c_cs = p->n;
    g.c2 = p->xhat_rm.get() + lo * p->rp; g.ld2 = p->rp;
    gemm(g, ctx->num_sms, ctx->stream);
}

void y_gemm_rows(cphifi_unaligned p, const double* x, double* y) {
    cphifi_obs o = p->obs;
    cphifi_ctx ctx = o->ctx;
    const int64_t lo = o->own_lo, hi = o->hull_hi, n = p->n;
    if (!p->yhat_sum.n) p->yhat_sum.alloc(n * p->rp);
    if (!p->y_part.n) p->y_part.alloc(n * p->r);
    shard_operand(p->yhat_rm.get(), x, n, p->r, p->rp, lo, hi, o->own_lo, o->own_hi, p->mode->lambda,
                  p->yhat_sum.get(), ctx->stream);
    GemmArgs g;
    g.m = n; g.n = p->r; g.k = hi - lo;
    g.a = p->mode->kernel.get() + lo * n; g.a_rs = 1; g.a_cs = n;
    g.b = p->yhat_sum.get() + lo * p->rp; g.b_rs = p->rp; g.b_cs = 1;
    g.c = p->y_part.get(); g.c_rs = 1; g.c_cs = n;
    if (o->shard == 0) {  // rho x once
        g.epi = EPI_AXPY2;
        g.e1 = x; g.e2 = x; g.ld_e = n;
        g.beta1 = 0.0; g.beta2 = p->rho;
    }
    if (g.k > 0) {
        gemm(g, ctx->num_sms, ctx->stream);
    } else {  // a shard without rows: its share is rho x (shard 0) or nothing
        CPHIFI_CUDA(cudaMemsetAsync(p->y_part.get(), 0, sizeof(double) * n * p->r, ctx->stream));
        if (o->shard == 0) axpby(p->y_part.get(), x, p->rho, p->y_part.get(), 0.0, n * p->r, ctx->stream);
    }
    allreduce_sum(ctx, p->y_part.get(), y, (size_t)n * p->r);
}

// y = vec(K Yhat + lambda Xhat) + rho x with Xhat = K X  (unaligned.hpp:101-115).
// Small n on one GPU: ONE cooperative launch.  Otherwise DMMA GEMMs around the fused
// scatter-gather, with the NCCL all-reduce of Yhat between them on multi-GPU.
void need_mode(cphifi_unaligned p) {
    if (!p->mode) throw_invalid("unaligned: a finite-mode subproblem (no kernel) has no operator");
}

void matvec_dev(cphifi_unaligned p, const double* x, double* y) {
    need_mode(p);
    cphifi_ctx ctx = p->obs->ctx;
    const bool multi = ctx_multi(ctx);
    if (p->op == 1) ensure_gram(p);
    const double* gr = p->op == 1 ? p->gram.get() : nullptr;
    if (p->small_n) {
        FusedArgs a = fused_args(p, matvec_phases(p, multi, 0));
        a.x = x;
        a.y = y;
        a.gram = gr;
        launch_fused(p, a);
        if (multi) {
            allreduce_yhat(p);
            a.phases = matvec_phases(p, multi, 1);
            launch_fused(p, a);
        }
        return;
    }
    if (row_sharded(p)) {
        xhat_gemm_rows(p, x);
        if (gr) gram_apply(gr, p->xhat_rm.get(), p->obs->row_ptr.get(), p->n, p->rp, p->yhat_rm.get(), ctx->stream);
        else launch_phase_b(p, fused_args(p, PH_B));
        y_gemm_rows(p, x, y);
        return;
    }
    xhat_gemm(p, x);
    if (gr) gram_apply(gr, p->xhat_rm.get(), p->obs->row_ptr.get(), p->n, p->rp, p->yhat_rm.get(), ctx->stream);
    else launch_phase_b(p, fused_args(p, PH_B));
    allreduce_yhat(p);
    y_gemm(p, x, y);
}

// build_preconditioner (unaligned.hpp:120-134): eig(K) (cached), eig(V), D
void ensure_precond(cphifi_unaligned p) {
    need_mode(p);
    mode_eig_once(p->mode);
    cphifi_ctx ctx = p->obs->ctx;
    const int64_t n = p->n, r = p->r;
    if (!p->have_veig) {
        p->uv.alloc(r * r);
        p->sv.alloc(r);
        device_sym_eig(ctx, p->v.get(), r, p->uv.get(), p->sv.get());
        p->have_veig = true;
    }
    if (!p->dmat.n) {
        p->dmat.alloc(n * r);
        ++p->veig_gen;  // a new D buffer: graphs captured with the old one are stale
        DevBuf<int> flag(1);
        CPHIFI_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), ctx->stream));
        precond_diag(p->mode->mu.get(), p->sv.get(), n, r, p->obs->density, p->mode->lambda, p->rho,
                     p->dmat.get(), flag.get(), ctx->stream);
        if (read_flag(ctx, flag.get())) {
            p->dmat.release();
            throw_runtime("build_preconditioner: nonpositive denominator");
        }
    }
}

// M^-1 x = U_K ((U_K' X U_V) .* D) U_V'   (unaligned.hpp:135-139), left-to-right
void precond_dev(cphifi_unaligned p, const double* x, double* y) {
    cphifi_ctx ctx = p->obs->ctx;
    const int64_t n = p->n, r = p->r;
    const double* uk = p->mode->u.get();
    if (sandwich_supported(n, r)) {
        const int64_t need_d = sandwich_scratch_doubles(n, r);
        if (p->t1.n < (size_t)need_d) {
            p->t1.alloc(need_d);
            CPHIFI_CUDA(cudaMemsetAsync(p->t1.get(), 0, sizeof(double) * need_d, ctx->stream));  // counters
        }
        SandArgs a;
        a.n = n; a.r = r;
        a.u = uk; a.ut = mode_ut(p->mode);
        a.x = x; a.ldx = n;
        a.uv = p->uv.get();
        a.op = SW_MUL; a.dmat = p->dmat.get();
        a.core_out = p->t1.get();
        a.y = y; a.ldy = n;
        sandwich(a, ctx->num_sms, ctx->stream);
        return;
    }
    GemmArgs g;
    g.m = n; g.n = r; g.k = n;                    // t1 = U_K' X
    g.a = uk; g.a_rs = n; g.a_cs = 1;
    g.b = x; g.b_rs = 1; g.b_cs = n;
    g.c = p->t1.get(); g.c_rs = 1; g.c_cs = n;
    gemm(g, ctx->num_sms, ctx->stream);
    GemmArgs h;
    h.m = n; h.n = r; h.k = r;                    // t2 = (t1 U_V) .* D
    h.a = p->t1.get(); h.a_rs = 1; h.a_cs = n;
    h.b = p->uv.get(); h.b_rs = 1; h.b_cs = r;
    h.c = p->t2.get(); h.c_rs = 1; h.c_cs = n;
    h.epi = EPI_HADAMARD; h.e1 = p->dmat.get(); h.ld_e = n;
    gemm(h, ctx->num_sms, ctx->stream);
    gemm_nn(ctx, n, r, n, uk, n, p->t2.get(), n, p->t1.get(), n);  // t1 = U_K t2
    GemmArgs o;
    o.m = n; o.n = r; o.k = r;                    // y = t1 U_V'
    o.a = p->t1.get(); o.a_rs = 1; o.a_cs = n;
    o.b = p->uv.get(); o.b_rs = r; o.b_cs = 1;
    o.c = y; o.c_rs = 1; o.c_cs = n;
    gemm(o, ctx->num_sms, ctx->stream);
}

// ---- the PCG in the eigenbasis of K (large n) ---------------------------------------------
// With K = U diag(mu) U' (the clamped spectrum the preconditioner already uses) and the PCG run on
// x~ = (I x U') x, an orthogonal change of variables (same inner products, same iterates in exact
// arithmetic):  A~ x~ = mu o (U' Yhat) + lambda mu o x~ + rho x~  with  Xhat = U diag(mu) x~,  and
// the preconditioner becomes  M~^-1 r~ = ((r~ U_V) o D) U_V'  — no n x n product.  Two n x n x r
// GEMMs per iteration instead of four (K X, K Yhat, U'R, U Z).  K differs from its clamped
// reconstruction by the clamped negative eigenvalues (rounding-level for the configs' kernels).
// Only for a kernel that is positive semidefinite up to rounding (mode->psd, decided when the
// eigendecomposition is computed or installed): there the clamped reconstruction differs from K at
// rounding level.  A markedly indefinite K (a caller-supplied matrix) keeps the original basis, so
// the operator is the reference's own, K included, and p'Ap <= 0 is detected as the reference does
// (solvers.hpp:65-68).
bool pcg_eigbasis(cphifi_unaligned p) {
    bool on = true;
    if (const char* e = std::getenv("CPHIFI_PCG_EIGBASIS")) on = std::atoi(e) != 0;
    return on && p->mode && p->mode->psd;
}

// leading rows / columns of the eigenbasis that the large-n operator skips (mode_nzero; 0 when off)
int64_t rot_null_rows(cphifi_unaligned p) {
    int64_t z = 0;
    if (const char* e = std::getenv("CPHIFI_PCG_SKIPZERO"); !e || std::atoi(e) != 0) z = mode_nzero(p->mode);
    return z >= p->n ? 0 : z;
}

// null_rows = false: the caller supplies rows i < z of y~ (= rho x~) itself (the fused PCG step)
// parts / nparts non-null: the output GEMM's split-K partials are left unreduced for the fused PCG
// step (EPI_PARTIALS; *parts = nullptr when that GEMM does not take the tensor-map path)
// The eigenbasis operator on a row-sharded plan (see row_sharded): rank s contracts only its rows of
// U diag(mu) and U' — Xhat[rows,:] = (U diag(mu))[rows, z:] x~[z:], its q-pass or row-Gram apply,
// y~_s = mu o (U[rows, z:]' Yhat_s[rows,:]) — the ridge terms (lambda mu + rho) x~ are diagonal in the
// eigenbasis and added on shard 0 alone, and ONE all-reduce of the n x r partials replaces the
// Yhat all-reduce.  Every rank ends with the same bits (the all-reduce's result).
bool row_sharded_rot(cphifi_unaligned p) {
    cphifi_obs o = p->obs;
    if (o->shards <= 1 || p->small_n) return false;
    if (ctx_multi(o->ctx) && o->ctx->nranks != o->shards) return false;
    const char* e = std::getenv("CPHIFI_ROW_SHARDED");
    return !(e && std::atoi(e) == 0);
}

void matvec_rot_rows(cphifi_unaligned p, const double* xt, double* yt, int64_t z, bool null_rows) {
    cphifi_obs o = p->obs;
    cphifi_ctx ctx = o->ctx;
    const int64_t n = p->n, r = p->r;
    int64_t lo = o->own_lo, hi = o->hull_hi;
    if (hi <= lo) {  // a shard without rows: contract 8 rows of zeros
        lo = std::max<int64_t>(0, std::min(lo, n - 8)) / 8 * 8;
        hi = std::min(n, lo + 8);
    }
    if (!p->y_part.n) p->y_part.alloc(n * r);
    GemmArgs g;  // Xhat[rows,:] -> row-major padded copy for the gather
    g.m = hi - lo; g.n = r; g.k = n - z;
    g.a = mode_um(p->mode) + z * n + lo; g.a_rs = 1; g.a_cs = n;
    g.b = xt + z; g.b_rs = 1; g.b_cs = n;
    g.c2 = p->xhat_rm.get() + lo * p->rp; g.ld2 = p->rp;
    gemm(g, ctx->num_sms, ctx->stream);
    if (p->op == 1) gram_apply(p->gram.get(), p->xhat_rm.get(), o->row_ptr.get(), n, p->rp, p->yhat_rm.get(), ctx->stream);
    else launch_phase_b(p, fused_args(p, PH_B));
    GemmArgs h;  // y~_s = mu o (U[rows, z:]' Yhat_s[rows,:]) (+ (lambda mu + rho) x~ on shard 0), rows i >= z
    h.m = n - z; h.n = r; h.k = hi - lo;
    h.a = mode_ut(p->mode) + z + lo * n; h.a_rs = 1; h.a_cs = n;
    h.b = p->yhat_rm.get() + lo * p->rp; h.b_rs = p->rp; h.b_cs = 1;
    h.c = p->y_part.get() + z; h.c_rs = 1; h.c_cs = n;
    h.epi = EPI_ROWSCALE; h.e_row = p->mode->mu.get() + z; h.ld_e = n;
    if (o->shard == 0) {
        h.e1 = xt + z;
        h.beta1 = p->mode->lambda; h.beta2 = p->rho;
    }
    gemm(h, ctx->num_sms, ctx->stream);
    if (z > 0) scale_row_block(p->y_part.get(), xt, z, n, r, 0.0, ctx->stream);  // rows i < z of the partial: zero
    allreduce_sum(ctx, p->y_part.get(), yt, (size_t)n * r);
    if (z > 0 && null_rows) scale_row_block(yt, xt, z, n, r, p->rho, ctx->stream);  // y~ = rho x~  (rows i < z)
}

void matvec_rot(cphifi_unaligned p, const double* xt, double* yt, bool null_rows = true,
                const double** parts = nullptr, int* nparts = nullptr) {
    need_mode(p);
    cphifi_ctx ctx = p->obs->ctx;
    const int64_t n = p->n, r = p->r;
    if (p->small_n) {  // the fused kernel with the eigenbasis columns and epilogue
        const bool multi = is_multi(p);
        const double* gr = p->op == 1 ? p->gram.get() : nullptr;
        FusedArgs a = fused_args(p, matvec_phases(p, multi, 0));
        a.kmat = mode_umt(p->mode);
        a.kmat_c2 = p->mode->u.get();
        a.mu_rot = p->mode->mu.get();
        a.x = xt;
        a.y = yt;
        a.gram = gr;
        launch_fused(p, a);
        if (multi) {
            allreduce_yhat(p);
            a.phases = matvec_phases(p, multi, 1);
            launch_fused(p, a);
        }
        return;
    }
    // rows / columns of the clamped null space (mu_i = 0) drop out of both GEMMs (mode_nzero)
    const int64_t z = rot_null_rows(p);
    if (!parts && row_sharded_rot(p)) {
        matvec_rot_rows(p, xt, yt, z, null_rows);
        return;
    }
    GemmArgs g;  // Xhat = U diag(mu) x~  -> row-major padded copy for the gather
    g.m = n; g.n = r; g.k = n - z;
    g.a = mode_um(p->mode) + z * n; g.a_rs = 1; g.a_cs = n;
    g.b = xt + z; g.b_rs = 1; g.b_cs = n;
    g.c2 = p->xhat_rm.get(); g.ld2 = p->rp;
    const double* gr = p->op == 1 ? p->gram.get() : nullptr;
    bool fuse_gram = gr && p->rp <= 64 && gemm_tma_ok(g);  // split-K reduction + row-Gram apply in one launch
    if (const char* e = std::getenv("CPHIFI_GRAM_EPI")) fuse_gram = fuse_gram && std::atoi(e) != 0;
    if (fuse_gram) {
        g.epi = EPI_GRAM; g.c2 = nullptr;
        g.gram = gr; g.row_ptr = p->obs->row_ptr.get(); g.rp = p->rp; g.yhat = p->yhat_rm.get();
    }
    gemm(g, ctx->num_sms, ctx->stream);
    if (fuse_gram) {
    } else if (gr) {
        gram_apply(gr, p->xhat_rm.get(), p->obs->row_ptr.get(), n, p->rp, p->yhat_rm.get(), ctx->stream);
    } else {
        launch_phase_b(p, fused_args(p, PH_B));
    }
    allreduce_yhat(p);
    GemmArgs h;  // y~ = mu o (U' Yhat + lambda x~) + rho x~   (rows i >= z)
    h.m = n - z; h.n = r; h.k = n;
    h.a = mode_ut(p->mode) + z; h.a_rs = 1; h.a_cs = n;
    h.b = yhat_result(p); h.b_rs = p->rp; h.b_cs = 1;
    h.c = yt + z; h.c_rs = 1; h.c_cs = n;
    h.epi = EPI_ROWSCALE; h.e_row = p->mode->mu.get() + z; h.e1 = xt + z; h.ld_e = n;
    h.beta1 = p->mode->lambda; h.beta2 = p->rho;
    if (parts) {
        *parts = nullptr;
        // opt-in (CPHIFI_PCG_AP_PARTS=1): measured slower at config 4 (12.25 vs 12.07 ms: the step's
        // partial-sum loads cost more than the reduce_epi launch they replace)
        bool on = false;
        if (const char* e = std::getenv("CPHIFI_PCG_AP_PARTS"))
            on = std::atoi(e) != 0 && gemm_tma_ok(h) && gemm_splitk_depth(h, ctx->num_sms) <= 4;  // step unrolls <= 4
        if (on) {
            h.epi = EPI_PARTIALS;
            h.parts_out = parts;
            h.p_out = nparts;
        }
    }
    gemm(h, ctx->num_sms, ctx->stream);
    if (z > 0 && null_rows) scale_row_block(yt, xt, z, n, r, p->rho, ctx->stream);  // y~ = rho x~  (rows i < z)
}

void precond_rot(cphifi_unaligned p, const double* rt, double* zt) {
    cphifi_ctx ctx = p->obs->ctx;
    const int64_t n = p->n, r = p->r;
    if (r <= 64) {  // one launch: r x r work per row
        precond_rot_small(rt, p->uv.get(), p->dmat.get(), n, r, zt, ctx->stream);
        return;
    }
    GemmArgs h;  // t2 = (r~ U_V) .* D
    h.m = n; h.n = r; h.k = r;
    h.a = rt; h.a_rs = 1; h.a_cs = n;
    h.b = p->uv.get(); h.b_rs = 1; h.b_cs = r;
    h.c = p->t2.get(); h.c_rs = 1; h.c_cs = n;
    h.epi = EPI_HADAMARD; h.e1 = p->dmat.get(); h.ld_e = n;
    gemm(h, ctx->num_sms, ctx->stream);
    GemmArgs o;  // z~ = t2 U_V'
    o.m = n; o.n = r; o.k = r;
    o.a = p->t2.get(); o.a_rs = 1; o.a_cs = n;
    o.b = p->uv.get(); o.b_rs = r; o.b_cs = 1;
    o.c = zt; o.c_rs = 1; o.c_cs = n;
    gemm(o, ctx->num_sms, ctx->stream);
}

// y = op(U) x (column-major n x r), op = U' (transpose) or U, optionally rows scaled by mu
void rotate(cphifi_unaligned p, bool transpose, bool scale_mu, const double* x, double* y) {
    cphifi_ctx ctx = p->obs->ctx;
    const int64_t n = p->n, r = p->r;
    GemmArgs g;
    g.m = n; g.n = r; g.k = n;
    g.a = transpose ? mode_ut(p->mode) : p->mode->u.get(); g.a_rs = 1; g.a_cs = n;
    g.b = x; g.b_rs = 1; g.b_cs = n;
    g.c = y; g.c_rs = 1; g.c_cs = n;
    if (scale_mu) {
        g.epi = EPI_ROWSCALE;
        g.e_row = p->mode->mu.get();
    }
    gemm(g, ctx->num_sms, ctx->stream);
}

// solve_aligned_decoupled core on device buffers (aligned.hpp:41-54)
// Enqueues only: the zero-denominator status lands in the returned mapped word, which the caller
// checks (decoupled_check) after its own synchronisation.
int* decoupled_dev(cphifi_mode mode, int64_t r, const double* b, const double* uv, const double* sv, double* w,
                   DevBuf<double>& t1, DevBuf<double>& core) {
    cphifi_ctx ctx = mode->ctx;
    const int64_t n = mode->n;
    int* flag = thread_flag();
    *flag = 0;
    if (sandwich_supported(n, r)) {
        const int64_t need_d = sandwich_scratch_doubles(n, r);
        if (core.n < (size_t)need_d) {
            core.alloc(need_d);
            CPHIFI_CUDA(cudaMemsetAsync(core.get(), 0, sizeof(double) * need_d, ctx->stream));  // counters
        }
        SandArgs a;
        a.n = n; a.r = r;
        a.u = mode->u.get(); a.ut = mode_ut(mode);
        a.x = b; a.ldx = n;
        a.uv = uv;
        a.op = SW_DIV; a.e_row = mode->mu.get(); a.e_col = sv; a.beta = mode->lambda; a.flag = flag;
        a.core_out = core.get();
        a.y = w; a.ldy = n;
        sandwich(a, ctx->num_sms, ctx->stream);
        return flag;
    }
    if (t1.n < (size_t)(n * r)) t1.alloc(n * r);
    if (core.n < (size_t)(n * r)) core.alloc(n * r);
    GemmArgs g;
    g.m = n; g.n = r; g.k = n;                    // t1 = U_K' B
    g.a = mode->u.get(); g.a_rs = n; g.a_cs = 1;
    g.b = b; g.b_rs = 1; g.b_cs = n;
    g.c = t1.get(); g.c_rs = 1; g.c_cs = n;
    gemm(g, ctx->num_sms, ctx->stream);
    GemmArgs h;
    h.m = n; h.n = r; h.k = r;                    // core = (t1 U_V) ./ (sigma_j mu_i + lambda)
    h.a = t1.get(); h.a_rs = 1; h.a_cs = n;
    h.b = uv; h.b_rs = 1; h.b_cs = r;
    h.c = core.get(); h.c_rs = 1; h.c_cs = n;
    h.epi = EPI_SCALE_DIV; h.e_row = mode->mu.get(); h.e_col = sv; h.beta1 = mode->lambda;
    h.flag = flag;
    gemm(h, ctx->num_sms, ctx->stream);
    gemm_nn(ctx, n, r, n, mode->u.get(), n, core.get(), n, t1.get(), n);  // U_K core
    GemmArgs o;
    o.m = n; o.n = r; o.k = r;                    // W = (.) U_V'
    o.a = t1.get(); o.a_rs = 1; o.a_cs = n;
    o.b = uv; o.b_rs = r; o.b_cs = 1;
    o.c = w; o.c_rs = 1; o.c_cs = n;
    gemm(o, ctx->num_sms, ctx->stream);
    return flag;
}

// after the caller's synchronisation (W is discarded on error, aligned.hpp:48-50)
void decoupled_check(const int* flag) {
    if (*reinterpret_cast<const volatile int*>(flag))
        throw_runtime("solve_aligned_decoupled: zero eigenvalue pair; use lambda > 0");
}

void upload_factors_cm(cphifi_ctx ctx, int d, const int64_t* shape, int k, int64_t r, const double* const* factors,
                       DevBuf<double>& buf, std::vector<const double*>& ptrs) {
    int64_t tot = 0;
    for (int m = 0; m < d; ++m)
        if (m != k) tot += shape[m] * r;
    buf.alloc(std::max<int64_t>(tot, 1));
    ptrs.assign(d, nullptr);
    int64_t off = 0;
    for (int m = 0; m < d; ++m) {
        if (m == k) continue;
        need(factors[m], "factor");
        h2d(buf.get() + off, factors[m], sizeof(double) * shape[m] * r, ctx->stream);
        ptrs[m] = buf.get() + off;
        off += shape[m] * r;
    }
}

// The device-resident PCG loop needs a single GPU (no NCCL inside the graph body); opt out with
// CPHIFI_PCG_GRAPH=0.  A failed capture or instantiation falls back to the host loop for good.
// Default: the graph unless the iteration is long enough that the host round trip is cheaper than
// the WHILE body's per-iteration cost — measured on B200 (profiles/prof_pcg_ab.sh): config 4
// (n r = 262144) 15.0 ms graph vs 13.0 ms host loop; config 3 (n r = 65536) 0.58 vs 0.64 ms.
bool pcg_graph_ok(cphifi_unaligned p) {
    if (p->pcg_graph_failed || is_multi(p)) return false;
    if (const char* e = std::getenv("CPHIFI_PCG_GRAPH")) return std::atoi(e) != 0;
    return p->n * p->r <= 131072;
}

// Capture `body` (one PCG iteration) into the body graph of a WHILE conditional node and
// instantiate it, once per plan and operator form.  The captured pointers are the plan's
// persistent PCG vectors, so later solves reuse the executable graph.
// The captured graphs hold device pointers of the mode's eigendecomposition (U, U', U diag(mu), mu)
// and of the plan's preconditioner (U_V, D): installing new ones must force a recapture.
uint64_t eig_generation(cphifi_unaligned p) { return ((p->mode ? p->mode->eig_gen : 0) << 32) ^ p->veig_gen; }

template <class F>
bool ensure_pcg_graph(cphifi_unaligned p, bool rot, F&& body) {
    const int64_t zkey = rot && p->mode ? p->mode->nzero : -1;
    const uint64_t gen = eig_generation(p);
    if (p->pcg_exec && p->pcg_graph_op == p->op && p->pcg_graph_rot == (int)rot && p->pcg_graph_z == zkey &&
        p->pcg_graph_gen == gen)
        return true;
    if (p->pcg_exec) cudaGraphExecDestroy(p->pcg_exec);
    if (p->pcg_graph) cudaGraphDestroy(p->pcg_graph);
    p->pcg_exec = nullptr;
    p->pcg_graph = nullptr;
    cudaStream_t s = p->obs->ctx->stream;
    CPHIFI_CUDA(cudaStreamSynchronize(s));
    cudaGraph_t g = nullptr;
    bool capturing = false;
    try {
        CPHIFI_CUDA(cudaGraphCreate(&g, 0));
        cudaGraphConditionalHandle h;
        CPHIFI_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        CPHIFI_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
        cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
        CPHIFI_CUDA(cudaStreamBeginCaptureToGraph(s, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
        capturing = true;
        body(h);
        capturing = false;
        CPHIFI_CUDA(cudaStreamEndCapture(s, &bodyg));
        cudaGraphExec_t ex = nullptr;
        CPHIFI_CUDA(cudaGraphInstantiate(&ex, g, 0));
        p->pcg_graph = g;
        p->pcg_exec = ex;
        p->pcg_graph_op = p->op;
        p->pcg_graph_rot = (int)rot;
        p->pcg_graph_z = zkey;
        p->pcg_graph_gen = gen;
        return true;
    } catch (const Error& e) {
        if (capturing) {
            cudaGraph_t junk = nullptr;
            cudaStreamEndCapture(s, &junk);
        }
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        p->pcg_graph_failed = true;
        if (std::getenv("CPHIFI_DEBUG")) std::fprintf(stderr, "cphifi: PCG graph disabled: %s\n", e.what());
        return false;
    }
}

// Whole-solve graph: segment A (captured) -> WHILE node (body captured) -> segment B (captured).
// Built once per plan, operator form and basis; the captured pointers are the plan's persistent
// PCG vectors.  Returns false (and disables itself for the plan) when capture fails.
template <class FA, class FW, class FB>
bool ensure_pcg_full_graph(cphifi_unaligned p, bool rot, FA&& seg_a, FW&& body, FB&& seg_b) {
    const int64_t zkey = rot && p->mode ? p->mode->nzero : -1;
    const uint64_t gen = eig_generation(p);
    if (p->pcgf_exec && p->pcgf_op == p->op && p->pcgf_rot == (int)rot && p->pcgf_z == zkey && p->pcgf_gen == gen)
        return true;
    if (p->pcgf_exec) cudaGraphExecDestroy(p->pcgf_exec);
    if (p->pcgf_graph) cudaGraphDestroy(p->pcgf_graph);
    p->pcgf_exec = nullptr;
    p->pcgf_graph = nullptr;
    cudaStream_t s = p->obs->ctx->stream;
    CPHIFI_CUDA(cudaStreamSynchronize(s));
    cudaGraph_t g = nullptr;
    bool capturing = false;
    try {
        CPHIFI_CUDA(cudaGraphCreate(&g, 0));
        cudaGraphConditionalHandle h;
        CPHIFI_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
        CPHIFI_CUDA(cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
        capturing = true;
        seg_a(h);
        capturing = false;
        CPHIFI_CUDA(cudaStreamEndCapture(s, &g));
        // leaves of segment A
        size_t nn = 0;
        CPHIFI_CUDA(cudaGraphGetNodes(g, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn), leaves;
        CPHIFI_CUDA(cudaGraphGetNodes(g, nodes.data(), &nn));
        for (auto nd : nodes) {
            size_t ndep = 0;
            CPHIFI_CUDA(cudaGraphNodeGetDependentNodes(nd, nullptr, &ndep));
            if (ndep == 0) leaves.push_back(nd);
        }
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t wnode;
        CPHIFI_CUDA(cudaGraphAddNode(&wnode, g, leaves.data(), leaves.size(), &cp));
        cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
        CPHIFI_CUDA(cudaStreamBeginCaptureToGraph(s, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
        capturing = true;
        body(h);
        capturing = false;
        CPHIFI_CUDA(cudaStreamEndCapture(s, &bodyg));
        CPHIFI_CUDA(cudaStreamBeginCaptureToGraph(s, g, &wnode, nullptr, 1, cudaStreamCaptureModeRelaxed));
        capturing = true;
        seg_b();
        capturing = false;
        CPHIFI_CUDA(cudaStreamEndCapture(s, &g));
        cudaGraphExec_t ex = nullptr;
        CPHIFI_CUDA(cudaGraphInstantiate(&ex, g, 0));
        p->pcgf_graph = g;
        p->pcgf_exec = ex;
        p->pcgf_op = p->op;
        p->pcgf_rot = (int)rot;
        p->pcgf_z = zkey;
        p->pcgf_gen = gen;
        return true;
    } catch (const Error& e) {
        if (capturing) {
            cudaGraph_t junk = nullptr;
            cudaStreamEndCapture(s, &junk);
        }
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        p->pcg_graph_failed = true;
        if (std::getenv("CPHIFI_DEBUG")) std::fprintf(stderr, "cphifi: PCG solve graph disabled: %s\n", e.what());
        return false;
    }
}

}  // namespace

extern "C" {

const char* cphifi_last_error(void) { return g_last_error.c_str(); }
int cphifi_abi_version(void) { return CPHIFI_ABI_VERSION; }

// ---- context -------------------------------------------------------------------------
int cphifi_ctx_create(int device, cphifi_ctx* out) {
    return guard([&] {
        need(out, "cphifi_ctx_create");
        int count = 0;
        CPHIFI_CUDA(cudaGetDeviceCount(&count));
        if (device < 0 || device >= count) throw_invalid("cphifi_ctx_create: device out of range");
        CPHIFI_CUDA(cudaSetDevice(device));
        auto* c = new cphifi_ctx_s;
        c->device = device;
        CPHIFI_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
        CPHIFI_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        CPHIFI_SOLVER(cusolverDnCreate(&c->solver));
        CPHIFI_SOLVER(cusolverDnSetStream(c->solver, c->stream));
        CPHIFI_CUDA(cudaEventCreate(&c->ev0));
        CPHIFI_CUDA(cudaEventCreate(&c->ev1));
        CPHIFI_CUDA(cudaMallocHost(&c->host_scalars, 64 * sizeof(double)));
        *out = c;
    });
}

int cphifi_ctx_destroy(cphifi_ctx ctx) {
    return guard([&] {
        if (!ctx) return;
        DeviceGuard dg(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        if (ctx->comm) ncclCommDestroy(ctx->comm);
        if (ctx->solver) cusolverDnDestroy(ctx->solver);
        if (ctx->ev0) cudaEventDestroy(ctx->ev0);
        if (ctx->ev1) cudaEventDestroy(ctx->ev1);
        if (ctx->host_scalars) cudaFreeHost(ctx->host_scalars);
        if (ctx->stream) cudaStreamDestroy(ctx->stream);
        delete ctx;
    });
}

int cphifi_ctx_synchronize(cphifi_ctx ctx) {
    return guard([&] {
        need(ctx, "ctx");
        CPHIFI_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int cphifi_ctx_stream(cphifi_ctx ctx, void** stream_out) {
    return guard([&] {
        need(ctx, "ctx");
        need(stream_out, "stream_out");
        *stream_out = (void*)ctx->stream;
    });
}

int cphifi_fp64_peak(cphifi_ctx ctx, double* dfma_tflops, double* dmma_tflops) {
    return guard([&] {
        need(ctx, "ctx");
        need(dfma_tflops, "dfma_tflops");
        need(dmma_tflops, "dmma_tflops");
        DeviceGuard dg(ctx->device);
        fp64_peaks(ctx->num_sms, ctx->stream, dfma_tflops, dmma_tflops);
    });
}

int cphifi_comm_unique_id(uint8_t id_out[128]) {
    return guard([&] {
        need(id_out, "id_out");
        ncclUniqueId id;
        CPHIFI_NCCL(ncclGetUniqueId(&id));
        static_assert(sizeof(id) == 128, "ncclUniqueId size");
        std::memcpy(id_out, &id, 128);
    });
}

int cphifi_ctx_init_comm(cphifi_ctx ctx, int nranks, int rank, const uint8_t id[128]) {
    return guard([&] {
        need(ctx, "ctx");
        need(id, "id");
        if (nranks < 1 || rank < 0 || rank >= nranks) throw_invalid("cphifi_ctx_init_comm: bad rank");
        DeviceGuard dg(ctx->device);
        ncclUniqueId uid;
        std::memcpy(&uid, id, 128);
        if (ctx->vcomm) throw_invalid("cphifi_ctx_init_comm: the context uses a virtual communicator");
        if (ctx->comm) ncclCommDestroy(ctx->comm);
        ctx->comm = nullptr;
        CPHIFI_NCCL(ncclCommInitRank(&ctx->comm, nranks, uid, rank));
        ctx->nranks = nranks;
        ctx->rank = rank;
    });
}

int cphifi_vcomm_create(int nranks, cphifi_vcomm* out) {
    return guard([&] {
        need(out, "out");
        if (nranks < 1 || nranks > 8) throw_invalid("cphifi_vcomm_create: 1..8 ranks");
        auto* v = new cphifi_vcomm_s;
        v->nranks = nranks;
        v->send.assign(nranks, nullptr);
        v->ready.assign(nranks, nullptr);
        v->done.assign(nranks, nullptr);
        *out = v;
    });
}

int cphifi_vcomm_destroy(cphifi_vcomm vc) {
    return guard([&] {
        if (!vc) return;
        for (auto e : vc->ready)
            if (e) cudaEventDestroy(e);
        for (auto e : vc->done)
            if (e) cudaEventDestroy(e);
        delete vc;
    });
}

int cphifi_ctx_init_vcomm(cphifi_ctx ctx, cphifi_vcomm vc, int rank) {
    return guard([&] {
        need(ctx, "ctx");
        need(vc, "vc");
        if (rank < 0 || rank >= vc->nranks) throw_invalid("cphifi_ctx_init_vcomm: bad rank");
        if (ctx->comm) throw_invalid("cphifi_ctx_init_vcomm: the context already has an NCCL communicator");
        DeviceGuard dg(ctx->device);
        std::lock_guard<std::mutex> lk(vc->m);
        if (vc->ready[rank]) throw_invalid("cphifi_ctx_init_vcomm: rank already taken");
        CPHIFI_CUDA(cudaEventCreateWithFlags(&vc->ready[rank], cudaEventDisableTiming));
        CPHIFI_CUDA(cudaEventCreateWithFlags(&vc->done[rank], cudaEventDisableTiming));
        ctx->vcomm = vc;
        ctx->nranks = vc->nranks;
        ctx->rank = rank;
    });
}

int cphifi_ctx_world(cphifi_ctx ctx, int* nranks, int* rank) {
    return guard([&] {
        need(ctx, "ctx");
        if (nranks) *nranks = ctx->nranks;
        if (rank) *rank = ctx->rank;
    });
}

// ---- modes (kernel.hpp:17-30, 53-101) -----------------------------------------------
int cphifi_mode_create_gaussian(cphifi_ctx ctx, int64_t n, const double* points, double sigma, double lambda,
                                cphifi_mode* out) {
    return guard([&] {
        need(ctx, "ctx");
        need(out, "out");
        if (n < 1) throw_invalid("RkhsMode: empty design");
        need(points, "points");
        if (sigma <= 0.0) throw_invalid("gaussian_kernel: sigma must be positive");
        if (lambda < 0.0) throw_invalid("RkhsMode: lambda must be nonnegative");
        DeviceGuard dg(ctx->device);
        cphifi_mode m = new_mode(ctx, n, lambda);
        DevBuf<double> pts(n);
        h2d(pts.get(), points, sizeof(double) * n, ctx->stream);
        kernel_matrix(0, pts.get(), n, 1.0 / (2.0 * sigma * sigma), m->kernel.get(), ctx->stream);
        CPHIFI_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = m;
    });
}

int cphifi_mode_create_matern32(cphifi_ctx ctx, int64_t n, const double* points, double lengthscale,
                                double lambda, cphifi_mode* out) {
    return guard([&] {
        need(ctx, "ctx");
        need(out, "out");
        if (n < 1) throw_invalid("RkhsMode: empty design");
        need(points, "points");
        if (lengthscale <= 0.0) throw_invalid("matern32_kernel: lengthscale must be positive");
        if (lambda < 0.0) throw_invalid("RkhsMode: lambda must be nonnegative");
        DeviceGuard dg(ctx->device);
        cphifi_mode m = new_mode(ctx, n, lambda);
        DevBuf<double> pts(n);
        h2d(pts.get(), points, sizeof(double) * n, ctx->stream);
        kernel_matrix(1, pts.get(), n, std::sqrt(3.0) / lengthscale, m->kernel.get(), ctx->stream);
        CPHIFI_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = m;
    });
}

int cphifi_mode_create(cphifi_ctx ctx, int64_t n, const double* kernel, double lambda, cphifi_mode* out) {
    return guard([&] {
        need(ctx, "ctx");
        need(out, "out");
        need(kernel, "kernel");
        if (n < 1) throw_invalid("RkhsMode: empty design");
        if (lambda < 0.0) throw_invalid("RkhsMode: lambda must be nonnegative");
        DeviceGuard dg(ctx->device);
        cphifi_mode m = new_mode(ctx, n, lambda);
        h2d(m->kernel.get(), kernel, sizeof(double) * n * n, ctx->stream);
        CPHIFI_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = m;
    });
}

int cphifi_mode_destroy(cphifi_mode mode) {
    return guard([&] {
        if (!mode) return;
        DeviceGuard dg(mode->ctx->device);
        cudaStreamSynchronize(mode->ctx->stream);
        delete mode;
    });
}

int cphifi_mode_size(cphifi_mode mode, int64_t* n) {
    return guard([&] { need(mode, "mode"); need(n, "n"); *n = mode->n; });
}
int cphifi_mode_lambda(cphifi_mode mode, double* lambda) {
    return guard([&] { need(mode, "mode"); need(lambda, "lambda"); *lambda = mode->lambda; });
}
int cphifi_mode_get_kernel(cphifi_mode mode, double* kernel_out) {
    return guard([&] {
        need(mode, "mode");
        need(kernel_out, "kernel_out");
        DeviceGuard dg(mode->ctx->device);
        d2h_sync(kernel_out, mode->kernel.get(), sizeof(double) * mode->n * mode->n, mode->ctx->stream);
    });
}
int cphifi_mode_eig(cphifi_mode mode) {
    return guard([&] {
        need(mode, "mode");
        mode_eig_once(mode);
    });
}
int cphifi_mode_set_eig(cphifi_mode mode, const double* u, const double* mu) {
    return guard([&] {
        need(mode, "mode");
        need(u, "u");
        need(mu, "mu");
        DeviceGuard dg(mode->ctx->device);
        std::lock_guard<std::mutex> lk(mode->mu_lock);
        const int64_t n = mode->n;
        mode->u.alloc(n * n);
        mode->mu.alloc(n);
        mode->have_ut = false;
        mode->have_um = false;
        mode->have_umt = false;
        mode->nzero = -1;
        h2d(mode->u.get(), u, sizeof(double) * n * n, mode->ctx->stream);
        h2d(mode->mu.get(), mu, sizeof(double) * n, mode->ctx->stream);
        clamp_nonneg(mode->mu.get(), n, mode->ctx->stream);
        CPHIFI_CUDA(cudaStreamSynchronize(mode->ctx->stream));
        double lo = 0.0, hi = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            lo = std::min(lo, mu[i]);
            hi = std::max(hi, std::fabs(mu[i]));
        }
        mode->psd = lo >= -PSD_TOL * std::max(hi, 1.0);
        mode->have_eig = true;
        mode->eig_count = 1;
        ++mode->eig_gen;  // plans recapture their PCG graphs (eig_generation)
    });
}
int cphifi_mode_get_eig(cphifi_mode mode, double* u_out, double* mu_out) {
    return guard([&] {
        need(mode, "mode");
        mode_eig_once(mode);
        DeviceGuard dg(mode->ctx->device);
        if (u_out) d2h_sync(u_out, mode->u.get(), sizeof(double) * mode->n * mode->n, mode->ctx->stream);
        if (mu_out) d2h_sync(mu_out, mode->mu.get(), sizeof(double) * mode->n, mode->ctx->stream);
    });
}
int cphifi_mode_eig_count(cphifi_mode mode, int* count) {
    return guard([&] { need(mode, "mode"); need(count, "count"); *count = mode->eig_count; });
}

// ---- observations (observations.hpp:18-79) --------------------------------------------
namespace {
// The dense-row rule of the q-pass plan (build_dense_rows): a 3-way row whose entries cover at least
// this share of its n_1 x n_2 grid runs as two DMMA GEMMs, at the cost of ~DENSE_ROW_COST_CELLS x
// cells entries on the run kernel (config 4, B200: 2.26 us per dense row against 33.8 ps per sparse
// entry of a 512 x 512 grid).
double dense_min_density() {
    double dmin = 0.3;
    if (const char* e = std::getenv("CPHIFI_DENSE_MIN")) dmin = std::atof(e);
    return dmin;
}
// A dense row costs ~DENSE_ROW_COST_CELLS x cells plan entries of the run kernel, a sparse row its
// entries plus ~RUN_COST_ENTRIES per run (run start, partial last step, fold; two factor-block
// parts at config 4): fitted on the B200 to config 4's shards timed alone (26.8 ps per entry, 0.29 us
// per 512-run row, 2.3 us per dense row of a 512 x 512 grid; profiles/round2d/shard_cuts_config4.json;
// the dense share raised from 0.32 after the run kernel's RV_FOLDZ loop: 8 shards 0.75-0.86 -> 0.79-0.81 ms).
constexpr double DENSE_ROW_COST_CELLS = 0.345;
constexpr double RUN_COST_ENTRIES = 21.0;

bool shard_equal_count(uint32_t flags) {
    if (flags & CPHIFI_OBS_SHARD_EQUAL_COUNT) return true;
    const char* e = std::getenv("CPHIFI_SHARD_EQUAL_COUNT");
    return e && std::atoi(e) != 0;
}

// Cost-balanced shards of the sorted draws (SURVEY §8e shards the observations; equal counts of
// DRAWS leave a skewed plan — config 4's Zipf rows — with all the sparse rows, 63 % of the q-pass
// time, on the last rank: 1.4x at 8 shards).  The cost of row i is its plan entries (distinct cells
// when the plan coalesces, draws otherwise) plus a per-run term, or the dense-row equivalent when
// the q-pass would run it as GEMMs; shard s ends where the cost prefix reaches (s + 1) / S of the
// total, snapped to the nearer row boundary (whole rows keep the single-GPU dense / sparse split
// and never share a Yhat row between ranks) unless that row alone is more than a quarter of a
// shard, which is then cut inside by draw count.  Every rank computes the same cuts from the same
// sorted keys.  rp = row pointers of ALL draws (host); returns the S + 1 monotone cut positions.
std::vector<int64_t> balanced_shard_cuts(const uint64_t* keys, int64_t q, int64_t nk, uint64_t span, int d,
                                         int64_t n_first, bool coalesce, bool by_entries, int shards,
                                         const std::vector<int64_t>& rp, cudaStream_t s) {
    std::vector<unsigned long long> dist;
    if (coalesce) {
        DevBuf<unsigned long long> cnt_d(nk);
        dist.resize(nk);
        row_distinct_counts(keys, q, nk, span, cnt_d.get(), s);
        d2h_sync(dist.data(), cnt_d.get(), sizeof(unsigned long long) * nk, s);
    }
    const double cells = (double)span, dmin = dense_min_density();
    std::vector<double> pre(nk + 1, 0.0);
    for (int64_t i = 0; i < nk; ++i) {
        const double e = coalesce ? (double)dist[i] : (double)(rp[i + 1] - rp[i]);
        double c = e;  // by_entries: the row-Gram build's cost (2 rp^2 flops per plan entry, dense row or not)
        if (!by_entries) {
            c = e + RUN_COST_ENTRIES * std::min(e, (double)n_first);
            if (d == 3 && dmin > 0.0 && e >= dmin * cells) c = DENSE_ROW_COST_CELLS * cells;
        }
        pre[i + 1] = pre[i] + c;
    }
    const double total = pre[nk];
    std::vector<int64_t> cuts(shards + 1, 0);
    cuts[shards] = q;
    for (int t = 1; t < shards; ++t) {
        int64_t pos = q * t / shards;
        if (total > 0.0) {
            const double target = total * (double)t / (double)shards;
            int64_t i = std::upper_bound(pre.begin(), pre.end(), target) - pre.begin() - 1;  // pre[i] <= target
            i = std::min<int64_t>(std::max<int64_t>(i, 0), nk - 1);
            const double ci = pre[i + 1] - pre[i];
            if (ci <= total / (4.0 * shards)) pos = target - pre[i] < pre[i + 1] - target ? rp[i] : rp[i + 1];
            else pos = rp[i] + (int64_t)std::llround((target - pre[i]) / ci * (double)(rp[i + 1] - rp[i]));
        }
        cuts[t] = std::min(q, std::max(cuts[t - 1], pos));
    }
    return cuts;
}

// Row ranges of the shards (multiples of 8 rows, the GEMM operands' alignment): shard s owns rows
// [floor8(first row of s), floor8(first row of s + 1)), a partition of [0, n_k); its observations lie
// in rows [own_lo, hull_hi), hull_hi covering the row it may share with shard s + 1.
void shard_rows(cphifi_obs o, const std::vector<int64_t>& cuts, const std::vector<int64_t>& rp, int shard) {
    const int64_t nk = (int64_t)rp.size() - 1;
    const int S = (int)cuts.size() - 1;
    auto first_row = [&](int t) -> int64_t {  // the row holding draw cuts[t] (the largest i with rp[i] <= cut)
        if (t <= 0) return 0;
        if (t >= S) return nk;
        const int64_t i = (int64_t)(std::upper_bound(rp.begin(), rp.end(), cuts[t]) - rp.begin()) - 1;
        return std::min<int64_t>(std::max<int64_t>(i, 0), nk) / 8 * 8;
    };
    o->shards = S;
    o->shard = shard;
    o->own_lo = first_row(shard);
    o->own_hi = shard + 1 >= S ? nk : first_row(shard + 1);
    o->hull_hi = shard + 1 >= S ? nk : std::min(nk, o->own_hi + 8);
}
}  // namespace

int cphifi_obs_create(cphifi_ctx ctx, int d, const int64_t* shape, int64_t q, const int32_t* idx,
                      const double* values, int k, uint32_t flags, int shard, int shards, cphifi_obs* out) {
    return guard([&] {
        need(ctx, "ctx");
        need(out, "out");
        need(shape, "shape");
        if (d < 2 || d > 6) throw_invalid("ObservationSet: tensor order must be in [2, 6]");
        if (k < 0 || k >= d) throw_invalid("ObservationSet: mode out of range");
        if (q < 0) throw_invalid("ObservationSet: index/value count mismatch");
        if (q > (int64_t)INT32_MAX) throw_invalid("ObservationSet: more than 2^31-1 observations per plan");
        if (shards < 1 || shard < 0 || shard >= shards) throw_invalid("ObservationSet: bad shard");
        double ntot = 1.0;
        for (int m = 0; m < d; ++m) {
            if (shape[m] <= 0) throw_invalid("DenseTensor: nonpositive mode size");
            if (shape[m] > (int64_t)INT32_MAX) throw_invalid("ObservationSet: mode size exceeds int32");
        }
        int64_t ntot_i = 1;
        for (int m = 0; m < d; ++m) ntot_i *= shape[m];
        ntot = (double)ntot_i;
        if (q > 0) {
            need(idx, "idx");
            need(values, "values");
        }
        DeviceGuard dg(ctx->device);
        cudaStream_t s = ctx->stream;
        const bool dev_in = flags & CPHIFI_OBS_DEVICE_INPUT;
        auto* o = new cphifi_obs_s;
        std::unique_ptr<cphifi_obs_s> hold(o);
        o->ctx = ctx;
        o->d = d;
        o->k = k;
        o->shape.assign(shape, shape + d);
        o->q_total = q;
        o->density = (double)q / ntot;
        const int64_t nk = shape[k];

        DevBuf<int32_t> idx_up;
        DevBuf<double> val_up;
        const int32_t* didx = idx;
        const double* dval = values;
        if (!dev_in && q > 0) {
            idx_up.alloc((size_t)d * q);
            val_up.alloc(q);
            h2d(idx_up.get(), idx, sizeof(int32_t) * d * q, s);
            h2d(val_up.get(), values, sizeof(double) * q, s);
            didx = idx_up.get();
            dval = val_up.get();
        }
        DevBuf<int> flag(1);
        DevBuf<int64_t> dshape(d);
        CPHIFI_CUDA(cudaMemsetAsync(flag.get(), 0, sizeof(int), s));
        h2d(dshape.get(), shape, sizeof(int64_t) * d, s);
        check_range(didx, d, q, dshape.get(), flag.get(), s);
        if (read_flag(ctx, flag.get())) throw_invalid("ObservationSet: index out of range");
        // Plan order: lexicographic in (i_k, other modes ascending).  For k = 0 this is the storage
        // order of the reference's std::set of multi-indices (observations.hpp:27-41), so each row's
        // observations are summed in the reference's order; the first other mode forms runs that the
        // operator kernel hoists (k_fused.cu).  A multi-index wider than 63 bits falls back to a
        // stable i_k-only order.
        unsigned __int128 prod = 1;
        for (int m = 0; m < d; ++m) prod *= (unsigned __int128)shape[m];
        const bool lex = prod <= ((unsigned __int128)1 << 63);
        // equal-count cut of the sorted order; replaced below by the cost-balanced cut
        int64_t lo = q * shard / shards, hi = q * (shard + 1) / shards;
        o->lex = lex;
        const int64_t qa = std::max<int64_t>(q, 1);
        DevBuf<int32_t> perm_in(qa), perm_out(qa);
        DevBuf<uint64_t> key(lex ? qa : 1), key_s(lex ? qa : 1);
        DevBuf<int32_t> keys_out(lex ? 1 : qa);
        const bool coalesce = (flags & CPHIFI_OBS_COALESCE_DUPLICATES) != 0;
        if (coalesce && !lex) throw_invalid("ObservationSet: coalescing needs a multi-index of at most 63 bits");
        uint64_t span = 1;
        std::vector<int64_t> stride(d);
        if (lex) {
            for (int m = d - 1; m >= 0; --m) {
                if (m == k) continue;
                stride[m] = (int64_t)span;
                span *= (uint64_t)shape[m];
            }
            stride[k] = (int64_t)span;
            h2d(dshape.get(), stride.data(), sizeof(int64_t) * d, s);
            if (q > 0) {
                int bits = 1;
                while (bits < 64 && ((unsigned __int128)1 << bits) < prod) ++bits;
                linear_index(didx, d, q, dshape.get(), key.get(), s);
                iota32(perm_in.get(), q, s);
                const size_t tb = radix_sort_pairs64_bytes(q, bits);
                DevBuf<unsigned char> tmp(tb);
                radix_sort_pairs64(tmp.get(), tb, key.get(), key_s.get(), perm_in.get(), perm_out.get(), q, bits, s);
            }
            if ((flags & CPHIFI_OBS_REJECT_DUPLICATES) && q > 1) {
                adjacent_equal(key_s.get(), q, flag.get(), s);
                if (read_flag(ctx, flag.get())) throw_invalid("ObservationSet: duplicate index");
            }
        } else {
            if ((flags & CPHIFI_OBS_REJECT_DUPLICATES) && q > 1) {
                std::vector<int64_t> stride(d);
                int64_t st = 1;
                for (int m = 0; m < d; ++m) { stride[m] = st; st *= shape[m]; }
                h2d(dshape.get(), stride.data(), sizeof(int64_t) * d, s);
                DevBuf<uint64_t> lin(q), lin2(q);
                linear_index(didx, d, q, dshape.get(), lin.get(), s);
                const size_t tb = radix_sort_keys64_bytes(q);
                DevBuf<unsigned char> tmp(tb);
                radix_sort_keys64(tmp.get(), tb, lin.get(), lin2.get(), q, s);
                adjacent_equal(lin2.get(), q, flag.get(), s);
                if (read_flag(ctx, flag.get())) throw_invalid("ObservationSet: duplicate index");
            }
            if (q > 0) {  // stable sort by i_k -> permutation
                int bits = 1;
                while ((int64_t(1) << bits) < nk) ++bits;
                iota32(perm_in.get(), q, s);
                const size_t tb = radix_sort_pairs_bytes(q, bits);
                DevBuf<unsigned char> tmp(tb);
                radix_sort_pairs(tmp.get(), tb, didx + (int64_t)k * q, keys_out.get(), perm_in.get(), perm_out.get(),
                                 q, bits, s);
            }
        }
        key = DevBuf<uint64_t>();
        o->own_hi = o->hull_hi = nk;
        if (shards > 1 && q > 0) {
            // row pointers of ALL draws, the (cost-balanced or equal-count) cuts, the shards' row ranges
            DevBuf<int64_t> rp_d(nk + 1);
            std::vector<int64_t> rp(nk + 1);
            if (lex) csr_from_sorted64(key_s.get(), q, nk, span, rp_d.get(), s);
            else csr_from_sorted(keys_out.get(), q, nk, rp_d.get(), s);
            d2h_sync(rp.data(), rp_d.get(), sizeof(int64_t) * (nk + 1), s);
            std::vector<int64_t> cuts(shards + 1);
            for (int t = 0; t <= shards; ++t) cuts[t] = q * t / shards;
            if (lex && !shard_equal_count(flags)) {
                int mf = 0;  // the first other mode: the run kernel's runs
                while (mf == k) ++mf;
                cuts = balanced_shard_cuts(key_s.get(), q, nk, span, d, shape[mf], coalesce,
                                           (flags & CPHIFI_OBS_SHARD_BY_ENTRIES) != 0, shards, rp, s);
            }
            lo = cuts[shard];
            hi = cuts[shard + 1];
            shard_rows(o, cuts, rp, shard);
        }
        const int64_t ql = hi - lo;
        o->q_local = ql;
        if (coalesce) {
            // merge repeated multi-indices of this shard: one entry per distinct key, carrying its
            // multiplicity (operator weight) and summed value (RHS); indices decoded from the key
            DevBuf<double> vs(std::max<int64_t>(ql, 1)), vsum(std::max<int64_t>(ql, 1));
            DevBuf<int32_t> cnt(std::max<int64_t>(ql, 1));
            DevBuf<uint64_t> ukey(std::max<int64_t>(ql, 1));
            gather_f64(dval, perm_out.get(), lo, ql, vs.get(), s);
            const int64_t nu = coalesce_sorted(key_s.get() + lo, vs.get(), ql, ukey.get(), cnt.get(), vsum.get(), s);
            o->q_local = nu;
            o->ldq = (nu + 3) / 4 * 4;
            o->coalesced = true;
            DevBuf<int64_t> dstride(d);
            h2d(dstride.get(), stride.data(), sizeof(int64_t) * d, s);
            h2d(dshape.get(), shape, sizeof(int64_t) * d, s);
            o->idx_o.alloc((int64_t)(d - 1) * o->ldq + OBS_PAD);
            decode_keys(ukey.get(), nu, d, k, dstride.get(), dshape.get(), o->idx_o.get(), o->ldq, s);
            o->values.alloc(nu + OBS_PAD);
            o->mult.alloc(nu + OBS_PAD);
            if (nu > 0) {
                CPHIFI_CUDA(cudaMemcpyAsync(o->values.get(), vsum.get(), sizeof(double) * nu, cudaMemcpyDeviceToDevice, s));
                CPHIFI_CUDA(cudaMemcpyAsync(o->mult.get(), cnt.get(), sizeof(int32_t) * nu, cudaMemcpyDeviceToDevice, s));
            }
            o->row_ptr.alloc(nk + 1);
            csr_from_sorted64(ukey.get(), nu, nk, span, o->row_ptr.get(), s);
            CPHIFI_CUDA(cudaStreamSynchronize(s));
            *out = hold.release();
            return;
        }
        o->ldq = (ql + 3) / 4 * 4;
        o->idx_o.alloc((int64_t)(d - 1) * o->ldq + OBS_PAD);
        o->values.alloc(ql + OBS_PAD);
        int mm = 0;
        for (int m = 0; m < d; ++m) {
            if (m == k) continue;
            gather_i32(didx + (int64_t)m * q, perm_out.get(), lo, ql, o->idx_o.get() + (int64_t)mm * o->ldq, s);
            ++mm;
        }
        gather_f64(dval, perm_out.get(), lo, ql, o->values.get(), s);
        o->row_ptr.alloc(nk + 1);
        if (lex) csr_from_sorted64(key_s.get() + lo, ql, nk, span, o->row_ptr.get(), s);
        else csr_from_sorted(keys_out.get() + lo, ql, nk, o->row_ptr.get(), s);
        CPHIFI_CUDA(cudaStreamSynchronize(s));
        *out = hold.release();
    });
}

int cphifi_obs_shard_rows(cphifi_obs obs, int64_t* own_lo, int64_t* own_hi, int64_t* hull_hi) {
    return guard([&] {
        need(obs, "obs");
        if (own_lo) *own_lo = obs->own_lo;
        if (own_hi) *own_hi = obs->own_hi;
        if (hull_hi) *hull_hi = obs->hull_hi;
    });
}

int cphifi_obs_destroy(cphifi_obs obs) {
    return guard([&] {
        if (!obs) return;
        DeviceGuard dg(obs->ctx->device);
        cudaStreamSynchronize(obs->ctx->stream);
        delete obs;
    });
}

int cphifi_obs_info(cphifi_obs obs, int64_t* q_total, int64_t* q_local, double* density) {
    return guard([&] {
        need(obs, "obs");
        if (q_total) *q_total = obs->q_total;
        if (q_local) *q_local = obs->q_local;
        if (density) *density = obs->density;
    });
}

// ---- unaligned subproblem (unaligned.hpp:35-48) ----------------------------------------
int cphifi_unaligned_create(cphifi_obs obs, cphifi_mode mode, int64_t r, const double* const* factors, double rho,
                            cphifi_unaligned* out) {
    return guard([&] {
        need(obs, "obs");
        need(factors, "factors");
        need(out, "out");
        if (r < 1) throw_invalid("KruskalModel: rank must be positive");
        if (r > 128) throw_invalid("unaligned: rank above 128 is not supported");
        // mode == NULL: a finite-mode subproblem (B, V, row Grams; no operator, no solve)
        if (mode && mode->n != obs->shape[obs->k]) throw_invalid("unaligned: kernel size mismatch");
        cphifi_ctx ctx = obs->ctx;
        DeviceGuard dg(ctx->device);
        cudaStream_t s = ctx->stream;
        auto* p = new cphifi_unaligned_s;
        std::unique_ptr<cphifi_unaligned_s> hold(p);
        p->obs = obs;
        p->mode = mode;
        p->n = obs->shape[obs->k];
        p->r = r;
        p->rp = pow2_at_least(r, 4);
        p->rho = rho;
        const int d = obs->d, k = obs->k;
        // factors: column-major upload, then row-major padded packing for the K1 gathers
        DevBuf<double> fcm;
        std::vector<const double*> fptr;
        upload_factors_cm(ctx, d, obs->shape.data(), k, r, factors, fcm, fptr);
        int64_t tot = 0;
        p->fac_off.clear();
        for (int m = 0; m < d; ++m) {
            if (m == k) continue;
            p->fac_off.push_back(tot);
            tot += obs->shape[m] * p->rp;
        }
        p->fac.alloc(tot);
        int mm = 0;
        for (int m = 0; m < d; ++m) {
            if (m == k) continue;
            pack_rows(fptr[m], obs->shape[m], obs->shape[m], r, p->rp, p->fac.get() + p->fac_off[mm], s);
            ++mm;
        }
        // V = gram_khatri_rao (tensor.hpp:186-194)
        p->v.alloc(r * r);
        gram_kr(d, obs->shape.data(), r, fptr.data(), k, p->v.get(), s);
        // scratch
        const int64_t n = p->n;
        // fused-kernel launch shape: all CTAs co-resident (cooperative launch)
        p->small_n = n <= 512 && n * r <= 8192;
        if (const char* e = std::getenv("CPHIFI_SMALL_N")) p->small_n = p->small_n && std::atoi(e) != 0;
        p->prefetch = p->small_n;
        p->smem_factors = (int64_t)p->fac.n * 8 <= 96 * 1024;  // keeps two CTAs per SM
        if (const char* e = std::getenv("CPHIFI_SMEM_FACTORS")) p->smem_factors = p->smem_factors && std::atoi(e) != 0;
        const int64_t crows = (n + ctx->num_sms - 1) / ctx->num_sms;  // >= rows per CTA in PH_C2
        const int64_t pref = p->prefetch ? fused_ldx(n) * r + (fused_maxloc() + crows) * n : 0;
        // large plans with >= 2 other modes in lexicographic order: k_stream.cu, one CTA per SM
        p->stream = !p->small_n && obs->lex && stream_supported(p->rp, d - 1);
        if (const char* e = std::getenv("CPHIFI_STREAM")) p->stream = p->stream && std::atoi(e) != 0;
        int cmax;
        if (p->stream) {
            const int64_t sf = (int64_t)p->fac.n - obs->shape[k == 0 ? 1 : 0] * p->rp;  // all but the hoisted mode
            const int o_aux = obs->coalesced ? 4 : 0;  // the operator launches' staged aux column
            bool use_sf = stream_smem_bytes(p->rp, d - 1, sf, o_aux) <= stream_smem_cap();
            if (const char* e = std::getenv("CPHIFI_STREAM_SF")) use_sf = use_sf && std::atoi(e) != 0;
            p->stream_sf = use_sf ? sf : 0;
            cmax = ctx->num_sms;
            // the operator's q-pass on the run kernel (k_runs.cu) over the plan's parts, built on the
            // first stream-operator application (ensure_runs): a row-Gram solve never needs them
            bool runs = p->mode && runs_supported(p->rp, d - 1);
            if (const char* e = std::getenv("CPHIFI_RUNS")) runs = runs && std::atoi(e) != 0;
            p->runs_pending = runs;
            p->runs_sf = sf;
        } else {
            p->smem = fused_smem_bytes(p->rp, d - 1, (int64_t)p->fac.n, p->smem_factors, pref);
            cmax = fused_grid(p->rp, d - 1, p->smem_factors, p->smem, ctx->num_sms);
        }
        PartitionPlan plan;
        {
            std::vector<int64_t> rp_host(n + 1);
            d2h_sync(rp_host.data(), obs->row_ptr.get(), sizeof(int64_t) * (n + 1), s);
            // optional equal-count plan (CPHIFI_EQUAL_PART=<ctas>); measured slower than the
            // row-aligned plan at config 1 (split rows cost a slot round trip per CTA)
            int equal = 0;
            if (const char* e = std::getenv("CPHIFI_EQUAL_PART")) equal = p->small_n ? std::atoi(e) : 0;
            if (equal > cmax) equal = 0;
            if (equal > 0) {
                plan_partition(rp_host, cmax, std::min(cmax, ctx->num_sms), plan, equal);
                if (plan.max_span > fused_maxloc()) equal = 0;  // too many rows per CTA for local Xhat
            }
            if (equal <= 0) plan_partition(rp_host, cmax, std::min(cmax, ctx->num_sms), plan);
        }
        p->grid = plan.ctas;
        p->local_x = p->small_n && plan.max_span <= fused_maxloc();
        p->cta_beg.alloc(plan.beg.size());
        h2d(p->cta_beg.get(), plan.beg.data(), sizeof(int64_t) * plan.beg.size(), s);
        p->cta_rows.alloc(plan.rows.size());
        h2d(p->cta_rows.get(), plan.rows.data(), sizeof(int64_t) * plan.rows.size(), s);
        p->row_first_cta.alloc(n);
        h2d(p->row_first_cta.get(), plan.row_first_cta.data(), sizeof(int32_t) * n, s);
        p->row_ncta.alloc(n);
        h2d(p->row_ncta.get(), plan.row_ncta.data(), sizeof(int32_t) * n, s);
        p->rowcnt.alloc(n);
        CPHIFI_CUDA(cudaMemsetAsync(p->rowcnt.get(), 0, n * sizeof(unsigned), s));
        p->slot_a.alloc((size_t)p->grid * p->rp);
        p->slot_b.alloc((size_t)p->grid * p->rp);
        const size_t bw = barrier_words(p->grid, 16);
        p->barrier.alloc(bw);
        CPHIFI_CUDA(cudaMemsetAsync(p->barrier.get(), 0, bw * sizeof(unsigned), s));
        CPHIFI_CUDA(cudaStreamSynchronize(s));  // plan vectors are freed on scope exit
        p->xhat_rm.alloc(n * p->rp);
        p->yhat_rm.alloc(n * p->rp);
        // rows without observations in this shard are never written: keep them zero
        CPHIFI_CUDA(cudaMemsetAsync(p->yhat_rm.get(), 0, sizeof(double) * n * p->rp, s));
        CPHIFI_CUDA(cudaMemsetAsync(p->xhat_rm.get(), 0, sizeof(double) * n * p->rp, s));
        if (ctx_multi(ctx) || obs->shards > 1) p->yhat_sum.alloc(n * p->rp);
        if (obs->shards > 1) p->y_part.alloc(n * r);  // row-sharded operator (y_gemm_rows)
        p->xhat_cm.alloc(n * r);
        p->t1.alloc(n * r);
        p->t2.alloc(n * r);
        p->vx.alloc(n * r);
        p->vy.alloc(n * r);
        // B = sampled_mttkrp(obs, zhat, k) with the observed values (observations.hpp:186-188)
        FusedArgs a = fused_args(p, PH_B);
        a.weights = obs->values.get();
        if (!(p->stream && rhs_over_parts(p, a))) launch_phase_b(p, a);
        allreduce_yhat(p);
        p->b.alloc(n * r);
        rm_to_cm(yhat_result(p), n, p->rp, r, p->b.get(), s);
        CPHIFI_CUDA(cudaStreamSynchronize(s));
        p->op = auto_operator(p);  // the drop-in default (cphifi_unaligned_set_operator overrides)
        *out = hold.release();
    });
}

int cphifi_unaligned_destroy(cphifi_unaligned p) {
    return guard([&] {
        if (!p) return;
        DeviceGuard dg(p->obs->ctx->device);
        cudaStreamSynchronize(p->obs->ctx->stream);
        delete p;
    });
}

int cphifi_unaligned_get_b(cphifi_unaligned p, double* b_out) {
    return guard([&] {
        need(p, "p");
        need(b_out, "b_out");
        DeviceGuard dg(p->obs->ctx->device);
        d2h_sync(b_out, p->b.get(), sizeof(double) * p->n * p->r, p->obs->ctx->stream);
    });
}
int cphifi_unaligned_get_v(cphifi_unaligned p, double* v_out) {
    return guard([&] {
        need(p, "p");
        need(v_out, "v_out");
        DeviceGuard dg(p->obs->ctx->device);
        d2h_sync(v_out, p->v.get(), sizeof(double) * p->r * p->r, p->obs->ctx->stream);
    });
}

int cphifi_unaligned_set_operator(cphifi_unaligned p, int op) {
    return guard([&] {
        need(p, "p");
        if (op < CPHIFI_OP_STREAM || op > CPHIFI_OP_AUTO) throw_invalid("cphifi_unaligned_set_operator: unknown operator");
        if (op == CPHIFI_OP_AUTO) op = auto_operator(p);
        if (op == CPHIFI_OP_GRAM && p->rp > 64) throw_invalid("gram operator: padded rank above 64 is not supported");
        p->op = op;
    });
}

int cphifi_unaligned_get_operator(cphifi_unaligned p, int* op) {
    return guard([&] {
        need(p, "p");
        need(op, "op");
        *op = p->op;
    });
}

int cphifi_unaligned_matvec_device(cphifi_unaligned p, const double* x, double* y) {
    return guard([&] {
        need(p, "p");
        need(x, "x");
        need(y, "y");
        DeviceGuard dg(p->obs->ctx->device);
        matvec_dev(p, x, y);
    });
}

// One graph launch instead of three API calls (~4 us each here, profiles/micro/launch_rate.cu):
// x is staged by the host into a plan-owned pinned, device-mapped buffer; the graph copies it to
// HBM with a kernel (a PCIe read stream, no DMA node), applies the operator and copies y back the
// same way; the host copies it out.  Fixed staging pointers: the graph is captured once per plan.
bool host_matvec_graph(cphifi_unaligned p, const double* x, double* y) {
    cphifi_ctx ctx = p->obs->ctx;
    if (p->hv_failed || is_multi(p)) return false;
    if (const char* e = std::getenv("CPHIFI_HOST_GRAPH"))
        if (std::atoi(e) == 0) return false;
    const int64_t nr = p->n * p->r;
    const size_t bytes = sizeof(double) * nr;
    if (p->hv_exec && p->hv_op != p->op) {  // captured with another operator form
        cudaGraphExecDestroy(p->hv_exec);
        cudaGraphDestroy(p->hv_graph);
        p->hv_exec = nullptr;
        p->hv_graph = nullptr;
    }
    if (!p->hv_exec) {
        if (p->op == 1) ensure_gram(p);
        matvec_dev(p, p->vx.get(), p->vy.get());  // lazily built state and launch attributes first
        CPHIFI_CUDA(cudaStreamSynchronize(ctx->stream));
        cudaGraph_t g = nullptr;
        try {
            if (!p->hv_hx) CPHIFI_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&p->hv_hx), bytes, cudaHostAllocMapped));
            if (!p->hv_hy) CPHIFI_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&p->hv_hy), bytes, cudaHostAllocMapped));
            double *dhx = nullptr, *dhy = nullptr;
            CPHIFI_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dhx), p->hv_hx, 0));
            CPHIFI_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dhy), p->hv_hy, 0));
            CPHIFI_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed));
            try {
                copy_doubles(p->vx.get(), dhx, nr, ctx->stream);
                matvec_dev(p, p->vx.get(), p->vy.get());
                copy_doubles(dhy, p->vy.get(), nr, ctx->stream);
            } catch (...) {
                cudaGraph_t junk = nullptr;
                cudaStreamEndCapture(ctx->stream, &junk);
                if (junk) cudaGraphDestroy(junk);
                throw;
            }
            CPHIFI_CUDA(cudaStreamEndCapture(ctx->stream, &g));
            cudaGraphExec_t ex = nullptr;
            CPHIFI_CUDA(cudaGraphInstantiate(&ex, g, 0));
            p->hv_graph = g;
            p->hv_exec = ex;
            p->hv_op = p->op;
        } catch (const Error& e) {
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            p->hv_failed = true;
            if (std::getenv("CPHIFI_DEBUG")) std::fprintf(stderr, "cphifi: host matvec graph disabled: %s\n", e.what());
            return false;
        }
    }
    std::memcpy(p->hv_hx, x, bytes);
    CPHIFI_CUDA(cudaGraphLaunch(p->hv_exec, ctx->stream));
    CPHIFI_CUDA(cudaStreamSynchronize(ctx->stream));
    std::memcpy(y, p->hv_hy, bytes);
    return true;
}

// Large x / y already in pinned host memory (the caller's, e.g. a framework's pinned tensors): DMA
// straight from / to them around an operator-only graph.  The staging copies of host_matvec_graph
// cost two host memcpys of n r doubles (config 4: 2 x 2 MB, ~0.3 ms against a 6.2 ms operator).
bool host_pinned(const void* ptr) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

bool host_matvec_dma(cphifi_unaligned p, const double* x, double* y) {
    cphifi_ctx ctx = p->obs->ctx;
    const size_t bytes = sizeof(double) * p->n * p->r;
    if (bytes < ((size_t)1 << 20) || is_multi(p) || p->hv_failed) return false;
    if (!host_pinned(x) || !host_pinned(y)) return false;
    cudaStream_t s = ctx->stream;
    if (p->hd_exec && p->hd_op != p->op) {
        cudaGraphExecDestroy(p->hd_exec);
        cudaGraphDestroy(p->hd_graph);
        p->hd_exec = nullptr;
        p->hd_graph = nullptr;
    }
    if (!p->hd_exec) {
        if (p->op == 1) ensure_gram(p);
        matvec_dev(p, p->vx.get(), p->vy.get());  // lazily built state and launch attributes first
        CPHIFI_CUDA(cudaStreamSynchronize(s));
        cudaGraph_t g = nullptr;
        try {
            CPHIFI_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
            try {
                matvec_dev(p, p->vx.get(), p->vy.get());
            } catch (...) {
                cudaGraph_t junk = nullptr;
                cudaStreamEndCapture(s, &junk);
                if (junk) cudaGraphDestroy(junk);
                throw;
            }
            CPHIFI_CUDA(cudaStreamEndCapture(s, &g));
            cudaGraphExec_t ex = nullptr;
            CPHIFI_CUDA(cudaGraphInstantiate(&ex, g, 0));
            p->hd_graph = g;
            p->hd_exec = ex;
            p->hd_op = p->op;
        } catch (const Error& e) {
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
            p->hv_failed = true;
            if (std::getenv("CPHIFI_DEBUG")) std::fprintf(stderr, "cphifi: host matvec graph disabled: %s\n", e.what());
            return false;
        }
    }
    CPHIFI_CUDA(cudaMemcpyAsync(p->vx.get(), x, bytes, cudaMemcpyHostToDevice, s));
    CPHIFI_CUDA(cudaGraphLaunch(p->hd_exec, s));
    CPHIFI_CUDA(cudaMemcpyAsync(y, p->vy.get(), bytes, cudaMemcpyDeviceToHost, s));
    CPHIFI_CUDA(cudaStreamSynchronize(s));
    return true;
}

int cphifi_unaligned_matvec(cphifi_unaligned p, const double* x, double* y) {
    return guard([&] {
        need(p, "p");
        need(x, "x");
        need(y, "y");
        cphifi_ctx ctx = p->obs->ctx;
        DeviceGuard dg(ctx->device);
        if (host_matvec_dma(p, x, y)) return;
        if (host_matvec_graph(p, x, y)) return;
        const size_t bytes = sizeof(double) * p->n * p->r;
        h2d(p->vx.get(), x, bytes, ctx->stream);
        matvec_dev(p, p->vx.get(), p->vy.get());
        d2h_sync(y, p->vy.get(), bytes, ctx->stream);
    });
}

// Throughput hook: `steps` operator applications back to back in ONE CUDA graph, step i on plan
// i % m with its own x / y (device buffers).  With m plans whose combined working set exceeds L2,
// every application starts L2-cold without a flush inside the timed region.
int cphifi_unaligned_matvec_cycle_timed(const cphifi_unaligned* ps, const double* const* xs, double* const* ys, int m,
                                        int steps, float* total_ms) {
    return guard([&] {
        need(ps, "ps");
        need(xs, "xs");
        need(ys, "ys");
        need(total_ms, "total_ms");
        if (m < 1 || steps < 1) throw_invalid("cphifi_unaligned_matvec_cycle_timed: m and steps must be positive");
        cphifi_ctx ctx = ps[0]->obs->ctx;
        for (int i = 0; i < m; ++i) {
            need(ps[i], "p");
            if (ps[i]->obs->ctx != ctx) throw_invalid("cphifi_unaligned_matvec_cycle_timed: plans on different contexts");
        }
        DeviceGuard dg(ctx->device);
        cudaStream_t s = ctx->stream;
        for (int i = 0; i < m; ++i) {  // lazily built state before the capture
            if (ps[i]->op == 1) ensure_gram(ps[i]);
            matvec_dev(ps[i], xs[i], ys[i]);
        }
        CPHIFI_CUDA(cudaStreamSynchronize(s));
        cudaEvent_t e0, e1;
        CPHIFI_CUDA(cudaEventCreate(&e0));
        CPHIFI_CUDA(cudaEventCreate(&e1));
        cudaGraph_t g = nullptr;
        cudaGraphExec_t ex = nullptr;
        try {
            CPHIFI_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
            try {
                for (int t = 0; t < steps; ++t) matvec_dev(ps[t % m], xs[t % m], ys[t % m]);
            } catch (...) {
                cudaGraph_t junk = nullptr;
                cudaStreamEndCapture(s, &junk);
                if (junk) cudaGraphDestroy(junk);
                throw;
            }
            CPHIFI_CUDA(cudaStreamEndCapture(s, &g));
            CPHIFI_CUDA(cudaGraphInstantiate(&ex, g, 0));
            CPHIFI_CUDA(cudaGraphLaunch(ex, s));  // warm-up
            CPHIFI_CUDA(cudaStreamSynchronize(s));
            // evict the last plans of the warm-up from L2 the same way the steps do: by the cycle
            CPHIFI_CUDA(cudaEventRecord(e0, s));
            CPHIFI_CUDA(cudaGraphLaunch(ex, s));
            CPHIFI_CUDA(cudaEventRecord(e1, s));
            CPHIFI_CUDA(cudaEventSynchronize(e1));
            CPHIFI_CUDA(cudaEventElapsedTime(total_ms, e0, e1));
        } catch (...) {
            if (ex) cudaGraphExecDestroy(ex);
            if (g) cudaGraphDestroy(g);
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
            throw;
        }
        cudaGraphExecDestroy(ex);
        cudaGraphDestroy(g);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    });
}

int cphifi_unaligned_matvec_graph_timed(cphifi_unaligned p, const double* x, double* y, void* flush,
                                        size_t flush_bytes, int steps, float* ms_out) {
    return guard([&] {
        need(p, "p");
        need(x, "x");
        need(y, "y");
        need(ms_out, "ms_out");
        if (steps < 1) throw_invalid("cphifi_unaligned_matvec_graph_timed: steps must be positive");
        cphifi_ctx ctx = p->obs->ctx;
        DeviceGuard dg(ctx->device);
        cudaStream_t s = ctx->stream;
        if (p->op == 1) ensure_gram(p);
        matvec_dev(p, x, y);  // lazily built state before the capture
        CPHIFI_CUDA(cudaStreamSynchronize(s));
        std::vector<cudaEvent_t> ev(2 * (size_t)steps);
        for (auto& e : ev) CPHIFI_CUDA(cudaEventCreate(&e));
        cudaGraph_t g = nullptr;
        cudaGraphExec_t ex = nullptr;
        auto cleanup = [&] {
            if (ex) cudaGraphExecDestroy(ex);
            if (g) cudaGraphDestroy(g);
            for (auto& e : ev) cudaEventDestroy(e);
        };
        try {
            CPHIFI_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
            try {
                for (int i = 0; i < steps; ++i) {
                    if (flush && flush_bytes) CPHIFI_CUDA(cudaMemsetAsync(flush, i & 0xff, flush_bytes, s));
                    CPHIFI_CUDA(cudaEventRecordWithFlags(ev[2 * i], s, cudaEventRecordExternal));
                    matvec_dev(p, x, y);
                    CPHIFI_CUDA(cudaEventRecordWithFlags(ev[2 * i + 1], s, cudaEventRecordExternal));
                }
            } catch (...) {
                cudaGraph_t junk = nullptr;
                cudaStreamEndCapture(s, &junk);
                if (junk) cudaGraphDestroy(junk);
                throw;
            }
            CPHIFI_CUDA(cudaStreamEndCapture(s, &g));
            CPHIFI_CUDA(cudaGraphInstantiate(&ex, g, 0));
            CPHIFI_CUDA(cudaGraphLaunch(ex, s));  // warm-up
            CPHIFI_CUDA(cudaStreamSynchronize(s));
            CPHIFI_CUDA(cudaGraphLaunch(ex, s));
            CPHIFI_CUDA(cudaStreamSynchronize(s));
            for (int i = 0; i < steps; ++i) CPHIFI_CUDA(cudaEventElapsedTime(&ms_out[i], ev[2 * i], ev[2 * i + 1]));
        } catch (...) {
            cleanup();
            throw;
        }
        cleanup();
    });
}

int cphifi_unaligned_matvec_timed(cphifi_unaligned p, const double* x, double* y, int iters, double* ms_out) {
    return guard([&] {
        need(p, "p");
        need(x, "x");
        need(y, "y");
        need(ms_out, "ms_out");
        if (iters < 1) throw_invalid("cphifi_unaligned_matvec_timed: iters must be positive");
        cphifi_ctx ctx = p->obs->ctx;
        DeviceGuard dg(ctx->device);
        cudaStream_t s = ctx->stream;
        const bool multi = ctx_multi(ctx);
        cudaEvent_t ev[6];
        for (auto& e : ev) CPHIFI_CUDA(cudaEventCreate(&e));
        double acc[6] = {0, 0, 0, 0, 0, 0};
        if (p->op == 1) ensure_gram(p);
        const double* gr = p->op == 1 ? p->gram.get() : nullptr;
        for (int it = 0; it < iters; ++it) {
            CPHIFI_CUDA(cudaEventRecord(ev[0], s));
            const bool rows = row_sharded(p);
            if (rows) xhat_gemm_rows(p, x);
            else if (!p->small_n) xhat_gemm(p, x);
            CPHIFI_CUDA(cudaEventRecord(ev[1], s));
            FusedArgs a = fused_args(p, matvec_phases(p, multi, 0));
            a.x = x;
            a.y = y;
            a.gram = gr;
            g_dense_event = ev[2];  // launch_phase_b records it between the run kernel and the dense rows
            g_dense_recorded = false;
            if (!p->small_n && gr) gram_apply(gr, p->xhat_rm.get(), p->obs->row_ptr.get(), p->n, p->rp, p->yhat_rm.get(), s);
            else if (!p->small_n) launch_phase_b(p, a);
            else launch_fused(p, a);
            g_dense_event = nullptr;
            if (!g_dense_recorded) CPHIFI_CUDA(cudaEventRecord(ev[2], s));
            CPHIFI_CUDA(cudaEventRecord(ev[3], s));
            if (!rows) allreduce_yhat(p);
            CPHIFI_CUDA(cudaEventRecord(ev[4], s));
            if (rows) {
                y_gemm_rows(p, x, y);  // (its all-reduce of y inside this phase)
            } else if (!p->small_n) {
                y_gemm(p, x, y);
            } else if (multi) {
                a.phases = matvec_phases(p, multi, 1);
                launch_fused(p, a);
            }
            CPHIFI_CUDA(cudaEventRecord(ev[5], s));
            CPHIFI_CUDA(cudaEventSynchronize(ev[5]));
            float ms;
            for (int ph = 0; ph < 5; ++ph) {
                CPHIFI_CUDA(cudaEventElapsedTime(&ms, ev[ph], ev[ph + 1]));
                acc[ph] += ms;
            }
            CPHIFI_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[5]));
            acc[5] += ms;
        }
        for (auto& e : ev) cudaEventDestroy(e);
        for (int i = 0; i < 6; ++i) ms_out[i] = acc[i] / iters;
    });
}

int cphifi_unaligned_matvec_launches(cphifi_unaligned p, const double* x, double* y, int* kernels) {
    return guard([&] {
        need(p, "p");
        need(x, "x");
        need(y, "y");
        need(kernels, "kernels");
        cphifi_ctx ctx = p->obs->ctx;
        DeviceGuard dg(ctx->device);
        cudaStream_t s = ctx->stream;
        if (p->op == 1) ensure_gram(p);
        matvec_dev(p, x, y);  // lazily built state and launch attributes before the capture
        CPHIFI_CUDA(cudaStreamSynchronize(s));
        cudaGraph_t g = nullptr;
        g_count_only = true;
        try {
            CPHIFI_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
            try {
                matvec_dev(p, x, y);
            } catch (...) {
                cudaGraph_t junk = nullptr;
                cudaStreamEndCapture(s, &junk);
                if (junk) cudaGraphDestroy(junk);
                throw;
            }
            CPHIFI_CUDA(cudaStreamEndCapture(s, &g));
        } catch (...) {
            g_count_only = false;
            throw;
        }
        g_count_only = false;
        size_t nn = 0;
        CPHIFI_CUDA(cudaGraphGetNodes(g, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        CPHIFI_CUDA(cudaGraphGetNodes(g, nodes.data(), &nn));
        int cnt = 0;
        for (auto nd : nodes) {
            cudaGraphNodeType t;
            CPHIFI_CUDA(cudaGraphNodeGetType(nd, &t));
            if (t == cudaGraphNodeTypeKernel) ++cnt;
        }
        cudaGraphDestroy(g);
        *kernels = cnt;
    });
}

int cphifi_unaligned_matvec_trace(cphifi_unaligned p, const double* x, double* y, uint64_t* stamps, int capacity,
                                  int* ctas) {
    return guard([&] {
        need(p, "p");
        need(x, "x");
        need(y, "y");
        need(ctas, "ctas");
        cphifi_ctx ctx = p->obs->ctx;
        DeviceGuard dg(ctx->device);
        *ctas = p->grid;
        const size_t cnt = (size_t)p->grid * TRACE_SLOTS;
        DevBuf<unsigned long long> tr(cnt);
        CPHIFI_CUDA(cudaMemsetAsync(tr.get(), 0, cnt * sizeof(unsigned long long), ctx->stream));
        const bool multi = ctx_multi(ctx);
        if (p->op == 1) ensure_gram(p);
        if (!p->small_n) xhat_gemm(p, x);
        FusedArgs a = fused_args(p, matvec_phases(p, multi, 0));
        a.x = x;
        a.y = y;
        a.trace = tr.get();
        a.gram = p->op == 1 ? p->gram.get() : nullptr;
        DevBuf<long long> dbg;
        const bool want_dbg = std::getenv("CPHIFI_DBG") != nullptr;  // developer timeline
        if (want_dbg) {
            dbg.alloc((size_t)p->grid * DBG_SLOTS);
            CPHIFI_CUDA(cudaMemsetAsync(dbg.get(), 0xff, dbg.n * sizeof(long long), ctx->stream));
            a.dbg = dbg.get();
        }
        if (p->stream) launch_phase_b(p, a);  // no phase stamps in k_stream.cu
        else launch_fused(p, a);
        if (want_dbg) {
            std::vector<long long> h(dbg.n);
            d2h_sync(h.data(), dbg.get(), sizeof(long long) * h.size(), ctx->stream);
            // the CTAs with the longest and the median event span (clock64 is per SM: deltas only)
            std::vector<std::pair<long long, int>> span;
            for (int c = 0; c < p->grid; ++c) {
                long long lo = -1, hi = -1;
                for (int e = 0; e < DBG_SLOTS / 2 && h[(size_t)c * DBG_SLOTS + 2 * e] >= 0; ++e) {
                    const long long t = h[(size_t)c * DBG_SLOTS + 2 * e + 1];
                    if (lo < 0) lo = t;
                    hi = t;
                }
                span.push_back({hi - lo, c});
            }
            std::sort(span.begin(), span.end());
            std::vector<int> show = {span.back().second, span[span.size() - 2].second, span[span.size() / 2].second,
                                     span.front().second};
            for (int c : show) {
                std::printf("cta %d:", c);
                const long long t0 = h[(size_t)c * DBG_SLOTS + 1];
                for (int e = 0; e < DBG_SLOTS / 2 && h[(size_t)c * DBG_SLOTS + 2 * e] >= 0; ++e)
                    std::printf(" %lld@%lld", h[(size_t)c * DBG_SLOTS + 2 * e], h[(size_t)c * DBG_SLOTS + 2 * e + 1] - t0);
                std::printf("\n");
            }
            std::fflush(stdout);
        }
        if (stamps && capacity > 0)
            d2h_sync(stamps, tr.get(), sizeof(uint64_t) * std::min(cnt, (size_t)capacity), ctx->stream);
        CPHIFI_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int cphifi_unaligned_scatter_gather(cphifi_unaligned p, const double* xhat, double* yhat_out) {
    return guard([&] {
        need(p, "p");
        need(xhat, "xhat");
        need(yhat_out, "yhat_out");
        cphifi_ctx ctx = p->obs->ctx;
        DeviceGuard dg(ctx->device);
        const int64_t n = p->n, r = p->r;
        h2d(p->vx.get(), xhat, sizeof(double) * n * r, ctx->stream);
        pack_rows(p->vx.get(), n, n, r, p->rp, p->xhat_rm.get(), ctx->stream);
        launch_phase_b(p, fused_args(p, PH_B));
        allreduce_yhat(p);
        rm_to_cm(yhat_result(p), n, p->rp, r, p->vy.get(), ctx->stream);
        d2h_sync(yhat_out, p->vy.get(), sizeof(double) * n * r, ctx->stream);
    });
}

int cphifi_unaligned_qpass_plan(cphifi_unaligned p, int64_t* info, int count) {
    return guard([&] {
        need(p, "p");
        need(info, "info");
        if (count < 1) throw_invalid("cphifi_unaligned_qpass_plan: count must be positive");
        DeviceGuard dg(p->obs->ctx->device);
        ensure_runs(p);
        static const QpassPlan none;
        const QpassPlan& Q = p->qp ? *p->qp : none;
        int64_t q = 0, dr = 0, xp = 0, qr = 0;
        for (const auto& sp : Q.parts) {
            q += sp.q;
            dr += sp.draws;
            xp += sp.padded ? 1 : 0;
            qr += sp.q_real;
        }
        const int64_t v[8] = {(int64_t)Q.parts.size(), Q.dense_nd, Q.parts.empty() ? p->obs->q_local : q,
                              Q.parts.empty() ? -1 : dr, Q.dense_n1p, Q.dense_n2p, xp,
                              Q.parts.empty() ? p->obs->q_local : qr};
        for (int i = 0; i < count; ++i) info[i] = i < 8 ? v[i] : 0;
    });
}

int cphifi_unaligned_set_v_eig(cphifi_unaligned p, const double* u_v, const double* sigma_v) {
    return guard([&] {
        need(p, "p");
        need(u_v, "u_v");
        need(sigma_v, "sigma_v");
        cphifi_ctx ctx = p->obs->ctx;
        DeviceGuard dg(ctx->device);
        const int64_t r = p->r;
        p->uv.alloc(r * r);
        p->sv.alloc(r);
        h2d(p->uv.get(), u_v, sizeof(double) * r * r, ctx->stream);
        h2d(p->sv.get(), sigma_v, sizeof(double) * r, ctx->stream);
        clamp_nonneg(p->sv.get(), r, ctx->stream);
        p->have_veig = true;
        p->dmat.release();
        ++p->veig_gen;  // the PCG graphs captured U_V / D: recapture (eig_generation)
        CPHIFI_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int cphifi_unaligned_get_v_eig(cphifi_unaligned p, double* u_v_out, double* sigma_v_out) {
    return guard([&] {
        need(p, "p");
        cphifi_ctx ctx = p->obs->ctx;
        DeviceGuard dg(ctx->device);
        ensure_precond(p);
        if (u_v_out) d2h_sync(u_v_out, p->uv.get(), sizeof(double) * p->r * p->r, ctx->stream);
        if (sigma_v_out) d2h_sync(sigma_v_out, p->sv.get(), sizeof(double) * p->r, ctx->stream);
    });
}

int cphifi_unaligned_precond_apply_device(cphifi_unaligned p, const double* x, double* y) {
    return guard([&] {
        need(p, "p");
        need(x, "x");
        need(y, "y");
        DeviceGuard dg(p->obs->ctx->device);
        ensure_precond(p);
        precond_dev(p, x, y);
    });
}

int cphifi_unaligned_precond_apply(cphifi_unaligned p, const double* x, double* y) {
    return guard([&] {
        need(p, "p");
        need(x, "x");
        need(y, "y");
        cphifi_ctx ctx = p->obs->ctx;
        DeviceGuard dg(ctx->device);
        ensure_precond(p);
        const size_t bytes = sizeof(double) * p->n * p->r;
        h2d(p->vx.get(), x, bytes, ctx->stream);
        precond_dev(p, p->vx.get(), p->vy.get());
        d2h_sync(y, p->vy.get(), bytes, ctx->stream);
    });
}

// solve_unaligned_pcg (unaligned.hpp:143-161) + pcg (solvers.hpp:38-88)
int cphifi_solve_unaligned_pcg(cphifi_unaligned p, const cphifi_pcg_config* cfg, cphifi_solve_report* report,
                               const double* warm_start, double* w_out) {
    return guard([&] {
        need(p, "p");
        need(cfg, "cfg");
        need(w_out, "w_out");
        cphifi_ctx ctx = p->obs->ctx;
        DeviceGuard dg(ctx->device);
        cudaStream_t s = ctx->stream;
        const auto t0 = std::chrono::steady_clock::now();
        if (p->rho <= 0.0) throw_invalid("solve_unaligned_pcg: rho must be positive");
        const int64_t n = p->n, r = p->r, nr = n * r;
        if (!p->pcg_vec.n) {
            p->pcg_vec.alloc(6 * nr);
            p->pcg_aux.alloc(RED_PARTIALS + (sizeof(PcgState) + sizeof(PcgCtl) + 7) / 8);
        }
        double* bvec = p->pcg_vec.get();
        double *x = bvec + nr, *res = bvec + 2 * nr, *z = bvec + 3 * nr, *pv = bvec + 4 * nr, *ap = bvec + 5 * nr;
        double* partial = p->pcg_aux.get();
        PcgState* st = reinterpret_cast<PcgState*>(partial + RED_PARTIALS);
        PcgCtl* ctl = reinterpret_cast<PcgCtl*>(partial + RED_PARTIALS + (sizeof(PcgState) + 7) / 8);
        CPHIFI_CUDA(cudaMemsetAsync(partial, 0, sizeof(double) * RED_PARTIALS, s));
        CPHIFI_CUDA(cudaMemsetAsync(st, 0, sizeof(PcgState), s));
        const bool stime = std::getenv("CPHIFI_SOLVE_TIMING") != nullptr;  // developer: setup phases
        auto lap = [&](const char* what) {
            if (!stime) return;
            CPHIFI_CUDA(cudaStreamSynchronize(s));
            std::fprintf(stderr, "cphifi: solve setup %s at %.3f ms\n", what,
                         1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
        };
        ensure_precond(p);                                                        // build_preconditioner
        lap("preconditioner");
        const bool rot = pcg_eigbasis(p);
        if (rot && !p->small_n) mode_nzero(p->mode);  // host read here, never inside a graph capture
        if (rot) rotate(p, true, true, p->b.get(), bvec);  // rhs~ = (I x U') vec(K B) = mu o (U' B)
        else gemm_nn(ctx, n, r, n, p->mode->kernel.get(), n, p->b.get(), n, bvec, n);  // rhs = vec(K B)
        lap("rhs");
        if (cfg->tol <= 0.0 || cfg->max_iter < 1) throw_invalid("pcg: invalid config");
        if (p->op == 1) ensure_gram(p);  // the row-Gram operator's G: per-solve setup, timed as such
        else ensure_runs(p);             // the stream operator's run tables and warp ranges
        lap("operator state");
        CPHIFI_CUDA(cudaStreamSynchronize(s));
        const auto t_setup = std::chrono::steady_clock::now();
        double* hs = ctx->host_scalars;
        auto apply_a = [&](const double* xin, double* yout) {
            if (rot) matvec_rot(p, xin, yout);
            else matvec_dev(p, xin, yout);
        };
        auto apply_m = [&](const double* rin, double* zout) {
            if (rot) precond_rot(p, rin, zout);
            else precond_dev(p, rin, zout);
        };
        // large-n eigenbasis PCG: the iteration's vector work after Ap in one cooperative launch
        // (k_pcgstep.cu) instead of pap / x,r / control / preconditioner / rz / p launches
        bool fused_step = rot && !p->small_n && r <= 64;
        if (const char* e = std::getenv("CPHIFI_PCG_FUSED")) fused_step = fused_step && std::atoi(e) != 0;
        if (fused_step && !p->pcg_step.n) {
            p->pcg_step.alloc(1 + pcg_step_fused_partials(n, ctx->num_sms));
            CPHIFI_CUDA(cudaMemsetAsync(p->pcg_step.get(), 0, sizeof(double), s));
        }
        const double* ap_parts = nullptr;  // set by matvec_rot(..., &ap_parts, &ap_np) per operator call
        int ap_np = 0;
        auto step_fused = [&](PcgCtl* c, cudaGraphConditionalHandle h, bool set_cond = true) {
            PcgStepArgs sa;
            sa.n = n; sa.r = (int)r;
            sa.uv = p->uv.get(); sa.dmat = p->dmat.get();
            sa.x = x; sa.res = res; sa.p = pv; sa.z = z; sa.ap = ap;
            sa.st = st; sa.ctl = c; sa.h = h; sa.set_cond = set_cond ? 1 : 0;
            sa.null_rows = rot_null_rows(p);  // Ap rows i < z = rho p: matvec_rot leaves them to the step
            sa.rho = p->rho;
            sa.ap_parts = ap_parts;  // unreduced output GEMM (EPI_PARTIALS), or null: Ap as written
            sa.ap_p = ap_np;
            sa.mu = p->mode->mu.get();
            sa.lambda = p->mode->lambda;
            sa.barrier = reinterpret_cast<unsigned long long*>(p->pcg_step.get());
            sa.partial = p->pcg_step.get() + 1;
            pcg_step_fused(sa, ctx->num_sms, s);
        };
        // ---- whole solve on device: one graph launch, one synchronisation -----------------
        if (p->op == 1) ensure_gram(p);
        if (pcg_graph_ok(p)) {
            if (warm_start) {  // r0 = b - A x0 before the graph (x0 rotated in the eigenbasis)
                if (rot) {
                    h2d(ap, warm_start, sizeof(double) * nr, s);
                    rotate(p, true, false, ap, x);
                } else {
                    h2d(x, warm_start, sizeof(double) * nr, s);
                }
                apply_a(x, ap);
                axpby(res, bvec, 1.0, ap, -1.0, nr, s);
            }
            const bool ok = ensure_pcg_full_graph(
                p, rot,
                [&](cudaGraphConditionalHandle h) {
                    dot_to(bvec, bvec, nr, partial, &st->bnorm, s);
                    pcg_prologue(st, ctl, s);
                    pcg_x0(x, res, bvec, nr, ctl, s);
                    apply_m(res, z);
                    pcg_init(res, z, pv, nr, st, partial, s);
                    pcg_loopctl(st, ctl, h, s);
                },
                [&](cudaGraphConditionalHandle h) {
                    if (fused_step) {
                        matvec_rot(p, pv, ap, false, &ap_parts, &ap_np);
                        step_fused(ctl, h);
                        return;
                    }
                    apply_a(pv, ap);
                    pcg_step_a_ctl(x, res, pv, ap, nr, st, partial, ctl, h, s);
                    apply_m(res, z);
                    pcg_step_b(res, z, pv, nr, st, partial, s);
                },
                [&] {
                    if (rot) {  // W = (I x U) x~
                        rotate(p, false, false, x, ap);
                        CPHIFI_CUDA(cudaMemcpyAsync(x, ap, sizeof(double) * nr, cudaMemcpyDeviceToDevice, s));
                    }
                });
            if (ok) {
                const int cap = cfg->record_history ? cfg->max_iter : 0;
                if (cap > 0 && p->pcg_hist.n < (size_t)cap) p->pcg_hist.alloc(cap);
                PcgCtl hc{};
                hc.tol = cfg->tol;
                hc.max_iter = cfg->max_iter;
                hc.hist = cap > 0 ? p->pcg_hist.get() : nullptr;
                hc.hist_cap = cap;
                hc.warm = warm_start ? 1 : 0;
                CPHIFI_CUDA(cudaMemcpyAsync(ctl, &hc, sizeof(PcgCtl), cudaMemcpyHostToDevice, s));
                CPHIFI_CUDA(cudaGraphLaunch(p->pcgf_exec, s));
                PcgCtl* hcp = reinterpret_cast<PcgCtl*>(hs);
                PcgState* hst = reinterpret_cast<PcgState*>(hs + (sizeof(PcgCtl) + 7) / 8);
                CPHIFI_CUDA(cudaMemcpyAsync(hcp, ctl, sizeof(PcgCtl), cudaMemcpyDeviceToHost, s));
                CPHIFI_CUDA(cudaMemcpyAsync(hst, st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
                d2h_sync(w_out, x, sizeof(double) * nr, s);  // the one synchronisation
                cphifi_solve_report rep{};
                std::vector<double> hist;
                if (hcp->zero_b) {
                    rep.converged = 1;  // x = 0 (solvers.hpp:49-53)
                } else {
                    if (hst->flag == 1) throw_runtime("pcg: non-finite value encountered");
                    if (hst->flag == 2) throw_runtime("pcg: operator not positive definite (p'Ap <= 0)");
                    const int it = hcp->it;
                    const double rel = it > 0 ? hst->rel : hcp->rel0;
                    if (cfg->record_history) {
                        hist.push_back(hcp->rel0);
                        const int m = std::min(it, cap);
                        hist.resize(1 + m);
                        if (m > 0) d2h_sync(hist.data() + 1, p->pcg_hist.get(), sizeof(double) * m, s);
                    }
                    rep.iterations = it;
                    rep.relative_residual = rel;
                    rep.converged = rel <= cfg->tol;
                    rep.matvecs = it + (warm_start ? 1 : 0);
                }
                const auto t1 = std::chrono::steady_clock::now();
                rep.wall_time_s = std::chrono::duration<double>(t1 - t0).count();
                rep.setup_s = std::chrono::duration<double>(t_setup - t0).count();
                if (report) {
                    double* hbuf = report->residual_history;
                    const int hcap = report->history_capacity;
                    rep.residual_history = hbuf;
                    rep.history_capacity = hcap;
                    rep.history_len = (int32_t)hist.size();
                    if (hbuf) std::memcpy(hbuf, hist.data(), sizeof(double) * std::min<size_t>(hist.size(), (size_t)std::max(hcap, 0)));
                    *report = rep;
                }
                return;
            }
        }
        dot_to(bvec, bvec, nr, partial, &st->bnorm, s);
        d2h_sync(hs, &st->bnorm, sizeof(double), s);
        const double bnorm = std::sqrt(hs[0]);
        std::vector<double> hist;
        cphifi_solve_report rep{};
        int matvecs = 0;
        if (bnorm == 0.0) {
            CPHIFI_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * nr, s));
            rep.converged = 1;
        } else {
            CPHIFI_CUDA(cudaMemcpyAsync(&st->bnorm, &bnorm, sizeof(double), cudaMemcpyHostToDevice, s));
            if (warm_start) {
                if (rot) {  // x0~ = (I x U') x0
                    h2d(ap, warm_start, sizeof(double) * nr, s);
                    rotate(p, true, false, ap, x);
                } else {
                    h2d(x, warm_start, sizeof(double) * nr, s);
                }
                apply_a(x, ap);
                ++matvecs;
                axpby(res, bvec, 1.0, ap, -1.0, nr, s);  // r = b - A x0
            } else {
                CPHIFI_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * nr, s));
                CPHIFI_CUDA(cudaMemcpyAsync(res, bvec, sizeof(double) * nr, cudaMemcpyDeviceToDevice, s));
            }
            apply_m(res, z);
            pcg_init(res, z, pv, nr, st, partial, s);
            PcgState hst;
            d2h_sync(&hst, st, sizeof(PcgState), s);
            double rel = hst.rel;
            if (cfg->record_history) hist.push_back(rel);
            int it = 0;
            // one PCG iteration (solvers.hpp:59-80): the host loop below and the graph body
            auto body_a = [&] {
                apply_a(pv, ap);
                pcg_step_a(x, res, pv, ap, nr, st, partial, s);
            };
            auto body_b = [&] {
                apply_m(res, z);
                pcg_step_b(res, z, pv, nr, st, partial, s);
            };
            bool done = false;
            if (p->op == 1) ensure_gram(p);  // lazily built state must exist before the capture
            if (rel > cfg->tol && pcg_graph_ok(p)) {
                // device-resident loop: a CUDA graph whose WHILE node repeats the iteration until
                // pcg_ctl clears the condition; no host round trip per iteration
                if (ensure_pcg_graph(p, rot, [&](cudaGraphConditionalHandle h) {
                        if (fused_step) {
                            matvec_rot(p, pv, ap, false, &ap_parts, &ap_np);
                            step_fused(ctl, h);
                            return;
                        }
                        body_a();
                        pcg_ctl(st, ctl, h, s);
                        body_b();
                    })) {
                    const int cap = cfg->record_history ? cfg->max_iter : 0;
                    if (cap > 0 && p->pcg_hist.n < (size_t)cap) p->pcg_hist.alloc(cap);
                    PcgCtl hc{};
                    hc.tol = cfg->tol;
                    hc.max_iter = cfg->max_iter;
                    hc.hist = cap > 0 ? p->pcg_hist.get() : nullptr;
                    hc.hist_cap = cap;
                    CPHIFI_CUDA(cudaMemcpyAsync(ctl, &hc, sizeof(PcgCtl), cudaMemcpyHostToDevice, s));
                    CPHIFI_CUDA(cudaGraphLaunch(p->pcg_exec, s));
                    d2h_sync(&hc, ctl, sizeof(PcgCtl), s);
                    d2h_sync(&hst, st, sizeof(PcgState), s);
                    if (hst.flag == 1) throw_runtime("pcg: non-finite value encountered");
                    if (hst.flag == 2) throw_runtime("pcg: operator not positive definite (p'Ap <= 0)");
                    it = hc.it;
                    matvecs += it;
                    rel = hst.rel;
                    if (cap > 0) {
                        const size_t h0 = hist.size();
                        hist.resize(h0 + std::min(it, cap));
                        d2h_sync(hist.data() + h0, p->pcg_hist.get(), sizeof(double) * std::min(it, cap), s);
                    }
                    done = true;
                }
            }
            if (!done && fused_step && rel > cfg->tol && it < cfg->max_iter) {
                // speculative host loop: iteration k + 1 is enqueued before iteration k's residual
                // is read back (event + pinned snapshot), so the GPU never idles on the host round
                // trip; the fused step of an iteration after the stopping one returns at entry
                // (ctl->stop, set on device exactly where solvers.hpp:59-80 leaves the loop)
                PcgCtl hc{};
                hc.tol = cfg->tol;
                hc.max_iter = cfg->max_iter;
                hc.it = it;
                h2d(ctl, &hc, sizeof(PcgCtl), s);
                PcgState* snap = reinterpret_cast<PcgState*>(hs);  // two pinned slots
                static_assert(2 * sizeof(PcgState) <= 64 * sizeof(double), "host scalar area");
                cudaEvent_t ev[2] = {nullptr, nullptr};
                CPHIFI_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
                CPHIFI_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
                struct EvGuard {
                    cudaEvent_t* e;
                    ~EvGuard() { cudaEventDestroy(e[0]); cudaEventDestroy(e[1]); }
                } evg{ev};
                auto enqueue = [&](int slot) {
                    matvec_rot(p, pv, ap, false, &ap_parts, &ap_np);
                    step_fused(ctl, cudaGraphConditionalHandle{}, false);
                    CPHIFI_CUDA(cudaMemcpyAsync(snap + slot, st, sizeof(PcgState), cudaMemcpyDeviceToHost, s));
                    CPHIFI_CUDA(cudaEventRecord(ev[slot], s));
                };
                enqueue(0);
                for (int k = 0;; ++k) {
                    const int slot = k & 1;
                    if (it + 1 < cfg->max_iter) enqueue(slot ^ 1);  // may be skipped on device
                    CPHIFI_CUDA(cudaEventSynchronize(ev[slot]));
                    const PcgState hs2 = snap[slot];
                    ++matvecs;
                    if (hs2.flag == 1) throw_runtime("pcg: non-finite value encountered");
                    if (hs2.flag == 2) throw_runtime("pcg: operator not positive definite (p'Ap <= 0)");
                    ++it;
                    rel = hs2.rel;
                    if (cfg->record_history) hist.push_back(rel);
                    if (!(rel > cfg->tol) || it >= cfg->max_iter) break;
                }
                done = true;
            }
            while (!done && rel > cfg->tol && it < cfg->max_iter) {
                if (fused_step) {  // step B runs inside the same launch (harmless after the last one)
                    matvec_rot(p, pv, ap, false, &ap_parts, &ap_np);
                    step_fused(nullptr, cudaGraphConditionalHandle{});
                } else {
                    body_a();
                }
                ++matvecs;
                d2h_sync(&hst, st, sizeof(PcgState), s);
                if (hst.flag == 1) throw_runtime("pcg: non-finite value encountered");
                if (hst.flag == 2) throw_runtime("pcg: operator not positive definite (p'Ap <= 0)");
                ++it;
                rel = hst.rel;
                if (cfg->record_history) hist.push_back(rel);
                if (rel <= cfg->tol) break;
                if (!fused_step) body_b();
            }
            rep.iterations = it;
            rep.relative_residual = rel;
            rep.converged = rel <= cfg->tol;
        }
        if (rot && bnorm != 0.0) {  // W = (I x U) x~
            rotate(p, false, false, x, ap);
            CPHIFI_CUDA(cudaMemcpyAsync(x, ap, sizeof(double) * nr, cudaMemcpyDeviceToDevice, s));
        }
        d2h_sync(w_out, x, sizeof(double) * nr, s);
        const auto t1 = std::chrono::steady_clock::now();
        rep.wall_time_s = std::chrono::duration<double>(t1 - t0).count();
        rep.setup_s = std::chrono::duration<double>(t_setup - t0).count();
        rep.matvecs = matvecs;
        if (report) {
            double* hbuf = report->residual_history;
            const int cap = report->history_capacity;
            rep.residual_history = hbuf;
            rep.history_capacity = cap;
            rep.history_len = (int32_t)hist.size();
            if (hbuf) std::memcpy(hbuf, hist.data(), sizeof(double) * std::min<size_t>(hist.size(), (size_t)std::max(cap, 0)));
            *report = rep;
        }
    });
}

// ---- aligned path ----------------------------------------------------------------------
int cphifi_tensor_create(cphifi_ctx ctx, int d, const int64_t* shape, const double* data, uint32_t flags, int shard,
                         int shards, cphifi_tensor* out) {
    return guard([&] {
        need(ctx, "ctx");
        need(shape, "shape");
        need(data, "data");
        need(out, "out");
        if (d < 2 || d > 8) throw_invalid("DenseTensor: order must be in [2, 8]");
        for (int m = 0; m < d; ++m)
            if (shape[m] <= 0) throw_invalid("DenseTensor: nonpositive mode size");
        if (shards < 1 || shard < 0 || shard >= shards) throw_invalid("DenseTensor: bad shard");
        DeviceGuard dg(ctx->device);
        auto* t = new cphifi_tensor_s;
        std::unique_ptr<cphifi_tensor_s> hold(t);
        t->ctx = ctx;
        t->d = d;
        t->shape.assign(shape, shape + d);
        t->slab_lo = shape[1] * shard / shards;
        t->slab_hi = shape[1] * (shard + 1) / shards;
        const int64_t n0 = shape[0], n1 = shape[1], w = t->slab_hi - t->slab_lo;
        int64_t rest = 1;
        for (int m = 2; m < d; ++m) rest *= shape[m];
        t->data.alloc(std::max<int64_t>(n0 * w * rest, 1));
        if (flags & CPHIFI_TENSOR_DEVICE_INPUT) {
            CPHIFI_CUDA(cudaMemcpyAsync(t->data.get(), data, sizeof(double) * n0 * w * rest, cudaMemcpyDeviceToDevice,
                                        ctx->stream));
        } else if (w > 0) {
            CPHIFI_CUDA(cudaMemcpy2DAsync(t->data.get(), sizeof(double) * n0 * w, data + n0 * t->slab_lo,
                                          sizeof(double) * n0 * n1, sizeof(double) * n0 * w, rest,
                                          cudaMemcpyHostToDevice, ctx->stream));
        }
        CPHIFI_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = hold.release();
    });
}

int cphifi_tensor_destroy(cphifi_tensor t) {
    return guard([&] {
        if (!t) return;
        DeviceGuard dg(t->ctx->device);
        cudaStreamSynchronize(t->ctx->stream);
        delete t;
    });
}

namespace {
void mttkrp_dev(cphifi_tensor t, int k, int64_t r, const std::vector<const double*>& fptr, double* b_dev,
                DevBuf<double>& work) {
    cphifi_ctx ctx = t->ctx;
    if (k != 0) {  // middle / last mode of a 3-way tensor (the finite-mode updates)
        if (!mttkrp_k3_supported(t->d, t->shape.data(), k, r))
            throw_invalid("mttkrp: modes k > 0 are accelerated for 3-way tensors with even n0 and r <= 64");
        if (t->slab_lo != 0 || t->slab_hi != t->shape[1])
            throw_invalid("mttkrp: modes k > 0 need the unsharded tensor");
        mttkrp_mode_k3(t->data.get(), t->shape.data(), k, r, fptr[0], t->shape[0], fptr[3 - k], t->shape[3 - k], b_dev,
                       ctx->num_sms, ctx->stream, work);
        return;
    }
    MttkrpArgs a;
    a.d = t->d;
    for (int m = 0; m < t->d; ++m) {
        a.shape[m] = t->shape[m];
        a.fac[m] = fptr[m];
        a.ld[m] = t->shape[m];
    }
    a.shape[1] = t->slab_hi - t->slab_lo;
    a.off1 = t->slab_lo;
    a.r = r;
    a.t = t->data.get();
    a.b = b_dev;
    if (a.shape[1] > 0) {
        mttkrp_mode0(a, ctx->num_sms, ctx->stream, work);
    } else {
        CPHIFI_CUDA(cudaMemsetAsync(b_dev, 0, sizeof(double) * t->shape[0] * r, ctx->stream));
    }
    allreduce(ctx, b_dev, (size_t)t->shape[0] * r);
}
}  // namespace

int cphifi_mttkrp(cphifi_tensor t, int k, int64_t r, const double* const* factors, double* b_out) {
    return guard([&] {
        need(t, "tensor");
        need(factors, "factors");
        need(b_out, "b_out");
        if (k < 0 || k >= t->d) throw_invalid("unfold: mode out of range");
        if (r < 1) throw_invalid("KruskalModel: rank must be positive");
        cphifi_ctx ctx = t->ctx;
        DeviceGuard dg(ctx->device);
        DevBuf<double> fbuf, b(t->shape[k] * r), work;
        std::vector<const double*> fptr;
        upload_factors_cm(ctx, t->d, t->shape.data(), k, r, factors, fbuf, fptr);
        mttkrp_dev(t, k, r, fptr, b.get(), work);
        d2h_sync(b_out, b.get(), sizeof(double) * t->shape[k] * r, ctx->stream);
    });
}

int cphifi_gram_khatri_rao(cphifi_ctx ctx, int d, const int64_t* shape, int64_t r, const double* const* factors,
                           int k, double* v_out) {
    return guard([&] {
        need(ctx, "ctx");
        need(shape, "shape");
        need(factors, "factors");
        need(v_out, "v_out");
        if (d < 1 || d > 8) throw_invalid("KruskalModel: bad order");
        if (r < 1) throw_invalid("KruskalModel: rank must be positive");
        DeviceGuard dg(ctx->device);
        DevBuf<double> fbuf, v(r * r);
        std::vector<const double*> fptr;
        upload_factors_cm(ctx, d, shape, k, r, factors, fbuf, fptr);
        gram_kr(d, shape, r, fptr.data(), k, v.get(), ctx->stream);
        d2h_sync(v_out, v.get(), sizeof(double) * r * r, ctx->stream);
    });
}

int cphifi_synth_observations(cphifi_ctx ctx, int d, const int64_t* shape, int64_t q, uint64_t seed, int zipf_mode,
                              double zipf_s, int64_t r, const double* const* factors, double noise_std, int32_t* idx_out,
                              double* vals_out) {
    return guard([&] {
        need(ctx, "ctx");
        need(shape, "shape");
        need(factors, "factors");
        if (d < 1 || d > 8) throw_invalid("synth: bad order");
        if (q < 0 || r < 1) throw_invalid("synth: bad size");
        if (q > 0) {
            need(idx_out, "idx_out");
            need(vals_out, "vals_out");
        }
        DeviceGuard dg(ctx->device);
        DevBuf<double> fbuf;
        std::vector<const double*> fptr;
        upload_factors_cm(ctx, d, shape, -1, r, factors, fbuf, fptr);
        synth_observations(d, shape, q, seed, zipf_mode, zipf_s, r, fptr.data(), noise_std, idx_out, vals_out,
                           ctx->num_sms, ctx->stream);
    });
}

int cphifi_solve_aligned_decoupled(cphifi_mode mode, int64_t r, const double* b, const double* v, const double* u_v,
                                   const double* sigma_v, double* w_out) {
    return guard([&] {
        need(mode, "mode");
        need(b, "b");
        need(w_out, "w_out");
        if (r < 1) throw_invalid("solve_aligned_decoupled: rank must be positive");
        if (!(u_v && sigma_v)) need(v, "v");
        cphifi_ctx ctx = mode->ctx;
        DeviceGuard dg(ctx->device);
        mode_eig_once(mode);
        const int64_t n = mode->n;
        DevBuf<double> db(n * r), uv(r * r), sv(r), w(n * r), t1, core;
        h2d(db.get(), b, sizeof(double) * n * r, ctx->stream);
        if (u_v && sigma_v) {
            h2d(uv.get(), u_v, sizeof(double) * r * r, ctx->stream);
            h2d(sv.get(), sigma_v, sizeof(double) * r, ctx->stream);
            clamp_nonneg(sv.get(), r, ctx->stream);
        } else {
            DevBuf<double> dv(r * r);
            h2d(dv.get(), v, sizeof(double) * r * r, ctx->stream);
            device_sym_eig(ctx, dv.get(), r, uv.get(), sv.get());
        }
        const int* flag = decoupled_dev(mode, r, db.get(), uv.get(), sv.get(), w.get(), t1, core);
        CPHIFI_CUDA(cudaStreamSynchronize(ctx->stream));
        decoupled_check(flag);
        d2h_sync(w_out, w.get(), sizeof(double) * n * r, ctx->stream);
    });
}

// ---- aligned baselines -----------------------------------------------------
int cphifi_aligned_matvec(cphifi_ctx ctx, int64_t n, int64_t r, const double* x, const double* d_k, const double* v,
                          double lambda, double* y) {
    return guard([&] {
        need(ctx, "ctx");
        need(x, "x");
        need(d_k, "d_k");
        need(v, "v");
        need(y, "y");
        if (n < 0 || r < 0) throw_invalid("aligned_matvec: size mismatch");
        DeviceGuard dg(ctx->device);
        cudaStream_t s = ctx->stream;
        DevBuf<double> dx(n * r), dd(n), dv(r * r), dy(n * r);
        h2d(dx.get(), x, sizeof(double) * n * r, s);
        h2d(dd.get(), d_k, sizeof(double) * n, s);
        h2d(dv.get(), v, sizeof(double) * r * r, s);
        aligned_matvec_dev(dx.get(), dd.get(), dv.get(), n, r, lambda, dy.get(), s);
        d2h_sync(y, dy.get(), sizeof(double) * n * r, s);
    });
}

// solve_aligned_pcg (aligned.hpp:72-100) with the pcg recurrence of solvers.hpp:38-88 (the same
// device vector kernels as the unaligned host loop), host-driven
int cphifi_solve_aligned_pcg(cphifi_mode mode, int64_t r, const double* b, const double* v,
                             const cphifi_pcg_config* cfg, cphifi_solve_report* report, const double* warm_start,
                             double* w_out) {
    return guard([&] {
        need(mode, "mode");
        need(b, "b");
        need(v, "v");
        need(cfg, "cfg");
        need(w_out, "w_out");
        if (r < 1) throw_invalid("solve_aligned_pcg: rank must be positive");
        const auto t0 = std::chrono::steady_clock::now();
        cphifi_ctx ctx = mode->ctx;
        DeviceGuard dg(ctx->device);
        cudaStream_t s = ctx->stream;
        mode_eig_once(mode);  // ek = mode->eig() (kernel.hpp:77-83)
        const int64_t n = mode->n, nr = n * r;
        DevBuf<double> db(nr), dv(r * r), bbar(nr), x(nr), res(nr), z(nr), pv(nr), ap(nr), dinv(nr);
        DevBuf<double> aux(RED_PARTIALS + (sizeof(PcgState) + 7) / 8);
        double* partial = aux.get();
        PcgState* st = reinterpret_cast<PcgState*>(partial + RED_PARTIALS);
        CPHIFI_CUDA(cudaMemsetAsync(aux.get(), 0, sizeof(double) * aux.n, s));
        h2d(db.get(), b, sizeof(double) * nr, s);
        h2d(dv.get(), v, sizeof(double) * r * r, s);
        auto rot = [&](bool transpose, const double* in, double* out) {  // out = U_K' in  /  U_K in
            GemmArgs g;
            g.m = n; g.n = r; g.k = n;
            g.a = mode->u.get();
            if (transpose) { g.a_rs = n; g.a_cs = 1; } else { g.a_rs = 1; g.a_cs = n; }
            g.b = in; g.b_rs = 1; g.b_cs = n;
            g.c = out; g.c_rs = 1; g.c_cs = n;
            gemm(g, ctx->num_sms, s);
        };
        rot(true, db.get(), bbar.get());  // bbar = U_K' B
        aligned_dinv(mode->mu.get(), dv.get(), n, r, mode->lambda, dinv.get(), s);
        auto apply_a = [&](const double* in, double* out) {
            aligned_matvec_dev(in, mode->mu.get(), dv.get(), n, r, mode->lambda, out, s);
        };
        auto apply_m = [&](const double* in, double* out) { hadamard(dinv.get(), in, nr, out, s); };
        if (cfg->tol <= 0.0 || cfg->max_iter < 1) throw_invalid("pcg: invalid config");
        double* hs = ctx->host_scalars;
        dot_to(bbar.get(), bbar.get(), nr, partial, &st->bnorm, s);
        d2h_sync(hs, &st->bnorm, sizeof(double), s);
        const double bnorm = std::sqrt(hs[0]);
        std::vector<double> hist;
        cphifi_solve_report rep{};
        int it = 0, matvecs = 0;
        double rel = 0.0;
        if (bnorm == 0.0) {  // solvers.hpp:49-53
            CPHIFI_CUDA(cudaMemsetAsync(x.get(), 0, sizeof(double) * nr, s));
            rep.converged = 1;
        } else {
            CPHIFI_CUDA(cudaMemcpyAsync(&st->bnorm, &bnorm, sizeof(double), cudaMemcpyHostToDevice, s));
            if (warm_start) {  // x0 = vec(U_K' W0)  (aligned.hpp:92-96)
                h2d(ap.get(), warm_start, sizeof(double) * nr, s);
                rot(true, ap.get(), x.get());
                apply_a(x.get(), ap.get());
                ++matvecs;
                axpby(res.get(), bbar.get(), 1.0, ap.get(), -1.0, nr, s);
            } else {
                CPHIFI_CUDA(cudaMemsetAsync(x.get(), 0, sizeof(double) * nr, s));
                CPHIFI_CUDA(cudaMemcpyAsync(res.get(), bbar.get(), sizeof(double) * nr, cudaMemcpyDeviceToDevice, s));
            }
            apply_m(res.get(), z.get());
            pcg_init(res.get(), z.get(), pv.get(), nr, st, partial, s);
            PcgState hst;
            d2h_sync(&hst, st, sizeof(PcgState), s);
            rel = hst.rel;
            if (cfg->record_history) hist.push_back(rel);
            while (rel > cfg->tol && it < cfg->max_iter) {
                apply_a(pv.get(), ap.get());
                ++matvecs;
                pcg_step_a(x.get(), res.get(), pv.get(), ap.get(), nr, st, partial, s);
                d2h_sync(&hst, st, sizeof(PcgState), s);
                if (hst.flag == 1) throw_runtime("pcg: non-finite value encountered");
                if (hst.flag == 2) throw_runtime("pcg: operator not positive definite (p'Ap <= 0)");
                ++it;
                rel = hst.rel;
                if (cfg->record_history) hist.push_back(rel);
                if (rel <= cfg->tol) break;
                apply_m(res.get(), z.get());
                pcg_step_b(res.get(), z.get(), pv.get(), nr, st, partial, s);
            }
            rep.iterations = it;
            rep.relative_residual = rel;
            rep.converged = rel <= cfg->tol;
        }
        rot(false, x.get(), ap.get());  // W = U_K Wbar
        d2h_sync(w_out, ap.get(), sizeof(double) * nr, s);
        rep.matvecs = matvecs;
        rep.wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (report) {
            double* hbuf = report->residual_history;
            const int hcap = report->history_capacity;
            rep.residual_history = hbuf;
            rep.history_capacity = hcap;
            rep.history_len = (int32_t)hist.size();
            if (hbuf) std::memcpy(hbuf, hist.data(), sizeof(double) * std::min<size_t>(hist.size(), (size_t)std::max(hcap, 0)));
            *report = rep;
        }
    });
}

// solve_aligned_direct (aligned.hpp:28-37): Cholesky of the materialised Kronecker system
int cphifi_solve_aligned_direct(cphifi_mode mode, int64_t r, const double* b, const double* v, int64_t direct_cap,
                                double* w_out) {
    return guard([&] {
        need(mode, "mode");
        need(b, "b");
        need(v, "v");
        need(w_out, "w_out");
        if (r < 1) throw_invalid("solve_aligned_direct: rank must be positive");
        const int64_t n = mode->n, rn = n * r;
        if (rn > direct_cap) throw_invalid("solve_aligned_direct: rn exceeds memory cap");
        cphifi_ctx ctx = mode->ctx;
        DeviceGuard dg(ctx->device);
        cudaStream_t s = ctx->stream;
        DevBuf<double> dv(r * r), sys((size_t)rn * rn), rhs(rn);
        h2d(dv.get(), v, sizeof(double) * r * r, s);
        h2d(rhs.get(), b, sizeof(double) * rn, s);
        kron_system(dv.get(), mode->kernel.get(), n, r, mode->lambda, sys.get(), s);
        int lwork = 0;
        CPHIFI_SOLVER(cusolverDnDpotrf_bufferSize(ctx->solver, CUBLAS_FILL_MODE_LOWER, (int)rn, sys.get(), (int)rn, &lwork));
        DevBuf<double> work(std::max(lwork, 1));
        DevBuf<int> info(1);
        CPHIFI_SOLVER(cusolverDnDpotrf(ctx->solver, CUBLAS_FILL_MODE_LOWER, (int)rn, sys.get(), (int)rn, work.get(), lwork,
                                       info.get()));
        int hinfo = 0;
        d2h_sync(&hinfo, info.get(), sizeof(int), s);
        if (hinfo != 0) throw_runtime("cholesky_solve: matrix is not positive definite");
        CPHIFI_SOLVER(cusolverDnDpotrs(ctx->solver, CUBLAS_FILL_MODE_LOWER, (int)rn, 1, sys.get(), (int)rn, rhs.get(),
                                       (int)rn, info.get()));
        d2h_sync(w_out, rhs.get(), sizeof(double) * rn, s);
    });
}

// ---- unaligned direct / dense baselines (unaligned.hpp:52-96, 164-174) -------
namespace {
// The all-shard row Grams of the plan (G_i over every observation of row i): this rank's G, summed
// over the ranks on a multi-rank plan.
const double* full_row_grams(cphifi_unaligned p, DevBuf<double>& tmp) {
    if (p->rp > 64) throw_invalid("gram operator: padded rank above 64 is not supported");
    ensure_gram(p);
    if (!is_multi(p)) return p->gram.get();
    const size_t cnt = (size_t)p->n * p->rp * p->rp;
    tmp.alloc(cnt);
    allreduce_sum(p->obs->ctx, p->gram.get(), tmp.get(), cnt);
    return tmp.get();
}
}  // namespace

int cphifi_solve_unaligned_direct_nonsym(cphifi_unaligned p, int64_t dense_cap, cphifi_solve_report* report,
                                         double* w_out) {
    return guard([&] {
        need(p, "p");
        need(w_out, "w_out");
        need_mode(p);
        const auto t0 = std::chrono::steady_clock::now();
        const int64_t n = p->n, r = p->r, rn = n * r;
        // build_G(p).transpose() * build_F(p): both materialisations carry the same cap (unaligned.hpp:54, 67)
        if (rn > dense_cap) throw_invalid("build_F: rn exceeds memory cap");
        cphifi_ctx ctx = p->obs->ctx;
        DeviceGuard dg(ctx->device);
        cudaStream_t s = ctx->stream;
        DevBuf<double> gtmp;
        const double* g = full_row_grams(p, gtmp);
        DevBuf<double> sys((size_t)rn * rn), a0((size_t)rn * rn), x(rn), res(rn), scal(2);
        nonsym_system(g, p->mode->kernel.get(), n, r, p->rp, p->mode->lambda, sys.get(), s);
        CPHIFI_CUDA(cudaMemcpyAsync(a0.get(), sys.get(), sizeof(double) * rn * rn, cudaMemcpyDeviceToDevice, s));
        CPHIFI_CUDA(cudaMemcpyAsync(x.get(), p->b.get(), sizeof(double) * rn, cudaMemcpyDeviceToDevice, s));
        // lu_solve (solvers.hpp:99-106): partial-pivot LU, then the residual check
        int lwork = 0;
        CPHIFI_SOLVER(cusolverDnDgetrf_bufferSize(ctx->solver, (int)rn, (int)rn, sys.get(), (int)rn, &lwork));
        DevBuf<double> work(std::max(lwork, 1));
        DevBuf<int> piv(std::max<int64_t>(rn, 1)), info(1);
        CPHIFI_SOLVER(cusolverDnDgetrf(ctx->solver, (int)rn, (int)rn, sys.get(), (int)rn, work.get(), piv.get(), info.get()));
        int hinfo = 0;
        d2h_sync(&hinfo, info.get(), sizeof(int), s);
        bool singular = hinfo > 0;
        if (!singular)
            CPHIFI_SOLVER(cusolverDnDgetrs(ctx->solver, CUBLAS_OP_N, (int)rn, 1, sys.get(), (int)rn, piv.get(), x.get(),
                                           (int)rn, info.get()));
        // res = A x - b with the DMMA GEMM, norms on device
        GemmArgs gm;
        gm.m = rn; gm.n = 1; gm.k = rn;
        gm.a = a0.get(); gm.a_rs = 1; gm.a_cs = rn;
        gm.b = x.get(); gm.b_rs = 1; gm.b_cs = rn;
        gm.c = res.get(); gm.c_rs = 1; gm.c_cs = rn;
        gm.epi = EPI_AXPY2; gm.e1 = p->b.get(); gm.e2 = p->b.get(); gm.ld_e = rn; gm.beta1 = -1.0; gm.beta2 = 0.0;
        gemm(gm, ctx->num_sms, s);
        std::vector<double> hres(rn), hb(rn), hx(rn);
        d2h_sync(hres.data(), res.get(), sizeof(double) * rn, s);
        d2h_sync(hb.data(), p->b.get(), sizeof(double) * rn, s);
        d2h_sync(hx.data(), x.get(), sizeof(double) * rn, s);
        double rr = 0.0, bb = 0.0;
        for (int64_t i = 0; i < rn; ++i) {
            rr += hres[i] * hres[i];
            bb += hb[i] * hb[i];
        }
        const double resn = std::sqrt(rr), bn = std::sqrt(bb);
        if (singular || !std::isfinite(resn) || resn > 1e-6 * std::max(bn, 1.0))
            throw_runtime("lu_solve: matrix is singular or severely ill-conditioned");
        std::memcpy(w_out, hx.data(), sizeof(double) * rn);
        if (report) {
            cphifi_solve_report rep = *report;
            rep.iterations = 1;
            rep.relative_residual = bn == 0.0 ? 0.0 : resn / bn;
            rep.converged = 1;
            rep.wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            rep.history_len = 0;
            *report = rep;
        }
    });
}

int cphifi_unaligned_assemble_sym_dense(cphifi_unaligned p, int64_t dense_cap, double* sys_out, double* rhs_out) {
    return guard([&] {
        need(p, "p");
        need(sys_out, "sys_out");
        need(rhs_out, "rhs_out");
        need_mode(p);
        const int64_t n = p->n, r = p->r, rn = n * r;
        if (rn > dense_cap) throw_invalid("assemble_unaligned_sym_dense: rn exceeds memory cap");
        cphifi_ctx ctx = p->obs->ctx;
        DeviceGuard dg(ctx->device);
        cudaStream_t s = ctx->stream;
        DevBuf<double> gtmp;
        const double* g = full_row_grams(p, gtmp);
        DevBuf<double> sm((size_t)rn * rn), cm((size_t)rn * rn), sys((size_t)rn * rn), rhs(rn);
        gram_scaled(g, p->mode->kernel.get(), n, r, p->rp, sm.get(), s);
        GemmArgs gm;  // C = K S  (n x r^2 n)
        gm.m = n; gm.n = r * r * n; gm.k = n;
        gm.a = p->mode->kernel.get(); gm.a_rs = 1; gm.a_cs = n;
        gm.b = sm.get(); gm.b_rs = 1; gm.b_cs = n;
        gm.c = cm.get(); gm.c_rs = 1; gm.c_cs = n;
        gemm(gm, ctx->num_sms, s);
        sym_place(cm.get(), p->mode->kernel.get(), n, r, p->mode->lambda, p->rho, sys.get(), s);
        gemm_nn(ctx, n, r, n, p->mode->kernel.get(), n, p->b.get(), n, rhs.get(), n);  // vec(K B)
        d2h_sync(sys_out, sys.get(), sizeof(double) * rn * rn, s);
        d2h_sync(rhs_out, rhs.get(), sizeof(double) * rn, s);
    });
}

int cphifi_aligned_solve_timed(cphifi_tensor t, cphifi_mode mode, int k, int64_t r, const double* const* factors,
                               int iters, double* w_out, double* ms_out) {
    return guard([&] {
        need(t, "tensor");
        need(mode, "mode");
        need(factors, "factors");
        need(w_out, "w_out");
        need(ms_out, "ms_out");
        if (iters < 1) throw_invalid("cphifi_aligned_solve_timed: iters must be positive");
        if (k < 0 || k >= t->d) throw_invalid("unfold: mode out of range");
        if (mode->n != t->shape[k]) throw_invalid("aligned: kernel size mismatch");
        cphifi_ctx ctx = t->ctx;
        DeviceGuard dg(ctx->device);
        cudaStream_t s = ctx->stream;
        mode_eig_once(mode);
        const int64_t n = mode->n;
        DevBuf<double> fbuf, b(n * r), v(r * r), uv(r * r), sv(r), w(n * r), t1, core, work;
        std::vector<const double*> fptr;
        upload_factors_cm(ctx, t->d, t->shape.data(), k, r, factors, fbuf, fptr);
        cudaEvent_t ev[5];
        for (auto& e : ev) CPHIFI_CUDA(cudaEventCreate(&e));
        double acc[5] = {0, 0, 0, 0, 0};
        double eig_ms = 0.0;
        for (int it = 0; it <= iters; ++it) {  // iteration 0 warms up (workspace allocation)
            CPHIFI_CUDA(cudaEventRecord(ev[0], s));
            mttkrp_dev(t, k, r, fptr, b.get(), work);
            CPHIFI_CUDA(cudaEventRecord(ev[1], s));
            gram_kr(t->d, t->shape.data(), r, fptr.data(), k, v.get(), s);
            CPHIFI_CUDA(cudaEventRecord(ev[2], s));
            // eig(V) is setup (north_star): computed in the warm-up pass, timed there, and reused,
            // so the timed passes run MTTKRP -> Gram -> decoupled back to back without the host
            // synchronisation cuSOLVER performs (it would put launch latency into the window)
            if (it == 0) {
                const auto te0 = std::chrono::steady_clock::now();
                device_sym_eig(ctx, v.get(), r, uv.get(), sv.get());
                eig_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - te0).count();
            }
            CPHIFI_CUDA(cudaEventRecord(ev[3], s));
            const int* flag = decoupled_dev(mode, r, b.get(), uv.get(), sv.get(), w.get(), t1, core);
            CPHIFI_CUDA(cudaEventRecord(ev[4], s));
            CPHIFI_CUDA(cudaEventSynchronize(ev[4]));
            decoupled_check(flag);
            if (it == 0) continue;
            float ms;
            for (int ph = 0; ph < 4; ++ph) {
                CPHIFI_CUDA(cudaEventElapsedTime(&ms, ev[ph], ev[ph + 1]));
                acc[ph] += ms;
            }
        }
        for (int i = 0; i < 4; ++i) ms_out[i] = acc[i] / iters;
        ms_out[2] = eig_ms;                              // eig(V) setup (wall clock, warm-up pass)
        ms_out[4] = ms_out[0] + ms_out[1] + ms_out[3];  // the timed solve excludes eig(V) (setup)
        // The per-phase passes above synchronise every solve, so each phase also carries the
        // host launch latency of its kernels (~4 us per plain launch here).  The timed solve is
        // the same MTTKRP -> Gram -> decoupled sequence captured once as a CUDA graph and
        // replayed `iters` times back to back (single GPU; no NCCL inside the capture).
        if (!(ctx_multi(ctx))) {
            cudaGraph_t g = nullptr;
            cudaGraphExec_t ex = nullptr;
            const int* flag = nullptr;
            // the Gram V = (*_{m != k} A_m'A_m) does not depend on the MTTKRP: a branch of the graph on a
            // second stream, concurrent with it (forked and joined inside the capture)
            cudaStream_t s2 = nullptr;
            cudaEvent_t efork = nullptr, ejoin = nullptr;
            CPHIFI_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
            CPHIFI_CUDA(cudaEventCreateWithFlags(&efork, cudaEventDisableTiming));
            CPHIFI_CUDA(cudaEventCreateWithFlags(&ejoin, cudaEventDisableTiming));
            struct Side {
                cudaStream_t s;
                cudaEvent_t a, b;
                ~Side() {
                    cudaEventDestroy(a);
                    cudaEventDestroy(b);
                    cudaStreamDestroy(s);
                }
            } side{s2, efork, ejoin};
            try {
                CPHIFI_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
                try {
                    CPHIFI_CUDA(cudaEventRecord(efork, s));
                    CPHIFI_CUDA(cudaStreamWaitEvent(s2, efork, 0));
                    gram_kr(t->d, t->shape.data(), r, fptr.data(), k, v.get(), s2);
                    CPHIFI_CUDA(cudaEventRecord(ejoin, s2));
                    mttkrp_dev(t, k, r, fptr, b.get(), work);
                    flag = decoupled_dev(mode, r, b.get(), uv.get(), sv.get(), w.get(), t1, core);
                    CPHIFI_CUDA(cudaStreamWaitEvent(s, ejoin, 0));
                } catch (...) {
                    cudaGraph_t junk = nullptr;
                    cudaStreamEndCapture(s, &junk);
                    if (junk) cudaGraphDestroy(junk);
                    throw;
                }
                CPHIFI_CUDA(cudaStreamEndCapture(s, &g));
                CPHIFI_CUDA(cudaGraphInstantiate(&ex, g, 0));
                CPHIFI_CUDA(cudaGraphLaunch(ex, s));
                CPHIFI_CUDA(cudaEventRecord(ev[0], s));
                for (int it = 0; it < iters; ++it) CPHIFI_CUDA(cudaGraphLaunch(ex, s));
                CPHIFI_CUDA(cudaEventRecord(ev[1], s));
                CPHIFI_CUDA(cudaEventSynchronize(ev[1]));
                decoupled_check(flag);
                float ms;
                CPHIFI_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
                ms_out[4] = ms / iters;
            } catch (...) {
                if (ex) cudaGraphExecDestroy(ex);
                if (g) cudaGraphDestroy(g);
                for (auto& e : ev) cudaEventDestroy(e);
                throw;
            }
            cudaGraphExecDestroy(ex);
            cudaGraphDestroy(g);
        }
        for (auto& e : ev) cudaEventDestroy(e);
        d2h_sync(w_out, w.get(), sizeof(double) * n * r, s);
    });
}

int cphifi_aligned_solve(cphifi_tensor t, cphifi_mode mode, int k, int64_t r, const double* const* factors,
                         double* w_out, double* b_out, double* v_out) {
    return guard([&] {
        need(t, "tensor");
        need(mode, "mode");
        need(factors, "factors");
        need(w_out, "w_out");
        if (k < 0 || k >= t->d) throw_invalid("unfold: mode out of range");
        if (mode->n != t->shape[k]) throw_invalid("aligned: kernel size mismatch");
        cphifi_ctx ctx = t->ctx;
        DeviceGuard dg(ctx->device);
        mode_eig_once(mode);
        const int64_t n = mode->n;
        DevBuf<double> fbuf, b(n * r), v(r * r), uv(r * r), sv(r), w(n * r), t1, core, work;
        std::vector<const double*> fptr;
        upload_factors_cm(ctx, t->d, t->shape.data(), k, r, factors, fbuf, fptr);
        mttkrp_dev(t, k, r, fptr, b.get(), work);
        gram_kr(t->d, t->shape.data(), r, fptr.data(), k, v.get(), ctx->stream);
        device_sym_eig(ctx, v.get(), r, uv.get(), sv.get());
        const int* flag = decoupled_dev(mode, r, b.get(), uv.get(), sv.get(), w.get(), t1, core);
        CPHIFI_CUDA(cudaStreamSynchronize(ctx->stream));
        decoupled_check(flag);
        d2h_sync(w_out, w.get(), sizeof(double) * n * r, ctx->stream);
        if (b_out) d2h_sync(b_out, b.get(), sizeof(double) * n * r, ctx->stream);
        if (v_out) d2h_sync(v_out, v.get(), sizeof(double) * r * r, ctx->stream);
    });
}


// relative_error (als.hpp:221-237) of the model whose mode-k factor is a_k (host n x r column-major)
// and whose other factors are the plan's: the residual pass of the infinite-mode update alone.
int cphifi_unaligned_relative_error(cphifi_unaligned p, const double* a_k, double* rel_error, double* data_norm) {
    return guard([&] {
        need(p, "p");
        need(a_k, "a_k");
        need(rel_error, "rel_error");
        cphifi_obs o = p->obs;
        if (o->coalesced) throw_invalid("relative_error: a plan with coalesced duplicates has no per-draw values");
        cphifi_ctx ctx = o->ctx;
        DeviceGuard dg(ctx->device);
        cudaStream_t s = ctx->stream;
        const int64_t n = p->n, r = p->r;
        DevBuf<double> a(n * r), arm((size_t)n * p->rp), scal(2),
            part(std::max<int64_t>(sq_residual_blocks(o->q_local), 1024));
        h2d(a.get(), a_k, sizeof(double) * n * r, s);
        pack_rows(a.get(), n, n, r, p->rp, arm.get(), s);
        SqResidualArgs ra;
        ra.n = n; ra.r = r; ra.rp = p->rp; ra.q = o->q_local; ra.ldq = o->ldq; ra.dother = o->d - 1;
        ra.row_ptr = o->row_ptr.get(); ra.idx = o->idx_o.get(); ra.values = o->values.get();
        ra.fac = p->fac.get();
        for (int m = 0; m < o->d - 1; ++m) ra.fac_off[m] = p->fac_off[m];
        ra.ak = arm.get();
        sq_residual(ra, part.get(), scal.get(), s);
        const int64_t nbn = std::min<int64_t>(std::max<int64_t>(1, (o->q_local + 2047) / 2048), 1024);
        if (o->q_local > 0) sq_norm(o->values.get(), o->q_local, part.get(), nbn, scal.get() + 1, s);
        else CPHIFI_CUDA(cudaMemsetAsync(scal.get() + 1, 0, sizeof(double), s));
        allreduce(ctx, scal.get(), 2);
        double h[2];
        d2h_sync(h, scal.get(), sizeof(double) * 2, s);
        const double dn = std::sqrt(h[1]);
        if (dn == 0.0) throw_runtime("relative_error: zero data norm");
        *rel_error = std::sqrt(h[0]) / dn;
        if (data_norm) *data_norm = dn;
    });
}

// ---- ALS finite-mode update, aligned (als.hpp:139-143): A_k = B_k V_k^+ (COD of V_k) ----------
int cphifi_als_update_finite_aligned(cphifi_tensor t, int k, int64_t r, const double* const* factors, double* a_out,
                                     double* rel_error_out) {
    return guard([&] {
        need(t, "tensor");
        need(factors, "factors");
        need(a_out, "a_out");
        if (k < 0 || k >= t->d) throw_invalid("unfold: mode out of range");
        cphifi_ctx ctx = t->ctx;
        DeviceGuard dg(ctx->device);
        cudaStream_t s = ctx->stream;
        const int64_t nk = t->shape[k], nr = nk * r;
        DevBuf<double> fbuf, b(nr), v(r * r), uv(r * r), sv(r), t1(nr), a(nr), g(r * r), scal(4), part(1024 + 80), work;
        std::vector<const double*> fptr;
        upload_factors_cm(ctx, t->d, t->shape.data(), k, r, factors, fbuf, fptr);
        mttkrp_dev(t, k, r, fptr, b.get(), work);                       // B_k = T_(k) Z_k
        gram_kr(t->d, t->shape.data(), r, fptr.data(), k, v.get(), s);  // V_k
        device_sym_eig(ctx, v.get(), r, uv.get(), sv.get());
        // V^+ on its eigenbasis: eigenvalues below r eps sigma_max dropped (COD's rank decision)
        invert_spectrum(sv.get(), r, s);
        GemmArgs h;  // t1 = (B U_V) diag(1 / sigma)
        h.m = nk; h.n = r; h.k = r;
        h.a = b.get(); h.a_rs = 1; h.a_cs = nk;
        h.b = uv.get(); h.b_rs = 1; h.b_cs = r;
        h.c = t1.get(); h.c_rs = 1; h.c_cs = nk;
        gemm(h, ctx->num_sms, s);
        scale_columns(t1.get(), nk, r, sv.get(), s);
        GemmArgs o;  // A = t1 U_V'
        o.m = nk; o.n = r; o.k = r;
        o.a = t1.get(); o.a_rs = 1; o.a_cs = nk;
        o.b = uv.get(); o.b_rs = r; o.b_cs = 1;
        o.c = a.get(); o.c_rs = 1; o.c_cs = nk;
        gemm(o, ctx->num_sms, s);
        if (rel_error_out) {  // relative error of the model after this update (Gram identity)
            GemmArgs gg;
            gg.m = r; gg.n = r; gg.k = nk;
            gg.a = a.get(); gg.a_rs = nk; gg.a_cs = 1;
            gg.b = a.get(); gg.b_rs = 1; gg.b_cs = nk;
            gg.c = g.get(); gg.c_rs = 1; gg.c_cs = r;
            gemm(gg, ctx->num_sms, s);
            CPHIFI_CUDA(cudaMemsetAsync(part.get(), 0, sizeof(double) * RED_PARTIALS, s));
            dot_to(a.get(), b.get(), nr, part.get(), scal.get(), s);
            CPHIFI_CUDA(cudaMemsetAsync(part.get(), 0, sizeof(double) * RED_PARTIALS, s));
            dot_to(g.get(), v.get(), r * r, part.get(), scal.get() + 1, s);
            if (!t->have_norm) {
                int64_t cnt = t->shape[0] * (t->slab_hi - t->slab_lo);
                for (int m = 2; m < t->d; ++m) cnt *= t->shape[m];
                t->norm2.alloc(1);
                sq_norm(t->data.get(), cnt, part.get(), 1024, t->norm2.get(), s);
                allreduce(ctx, t->norm2.get(), 1);
                t->have_norm = true;
            }
            CPHIFI_CUDA(cudaMemcpyAsync(scal.get() + 2, t->norm2.get(), sizeof(double), cudaMemcpyDeviceToDevice, s));
            double hsc[3];
            d2h_sync(hsc, scal.get(), sizeof(double) * 3, s);
            const double tn = std::sqrt(hsc[2]);
            if (tn == 0.0) throw_runtime("relative_error: zero data norm");
            *rel_error_out = std::sqrt(std::max(hsc[2] - 2.0 * hsc[0] + hsc[1], 0.0)) / tn;
        }
        d2h_sync(a_out, a.get(), sizeof(double) * nr, s);
    });
}

// ---- ALS finite-mode update, unaligned (als.hpp:144-162) --------------------
int cphifi_als_update_finite_unaligned(cphifi_unaligned p, double* a_out) {
    return guard([&] {
        need(p, "p");
        need(a_out, "a_out");
        cphifi_ctx ctx = p->obs->ctx;
        DeviceGuard dg(ctx->device);
        cudaStream_t s = ctx->stream;
        const int64_t n = p->n, r = p->r;
        if (p->rp > 64) throw_invalid("finite-mode update: padded rank above 64 is not supported");
        ensure_gram(p);  // G_i = Z_i' Z_i (this shard's observations)
        // multi-rank: the row solves need the all-shard Grams; they are summed into a separate
        // buffer so p->gram keeps this shard's G_i (the GRAM operator applies it per rank and then
        // sums Yhat over ranks)
        const double* g_all = p->gram.get();
        if (is_multi(p)) {
            const size_t cnt = (size_t)n * p->rp * p->rp;
            if (p->gram_sum.n < cnt) p->gram_sum.alloc(cnt);
            allreduce_sum(ctx, p->gram.get(), p->gram_sum.get(), cnt);
            g_all = p->gram_sum.get();
        }
        DevBuf<double> a(n * r);
        rowls_solve(g_all, p->b.get(), n, r, p->rp, a.get(), s);  // b = Z_i' t_i (all shards)
        d2h_sync(a_out, a.get(), sizeof(double) * n * r, s);
    });
}

// ---- ALS infinite-mode update (als.hpp:170-255) ---------------------------------------------
int cphifi_als_update_infinite_unaligned(cphifi_unaligned p, const cphifi_pcg_config* cfg, const double* warm_start,
                                         double* w_out, double* a_out, cphifi_solve_report* solve_report,
                                         cphifi_als_report* als) {
    return guard([&] {
        need(p, "p");
        need(cfg, "cfg");
        need(w_out, "w_out");
        need(als, "als");
        cphifi_obs o = p->obs;
        if (o->coalesced)
            throw_invalid("relative_error: a plan with coalesced duplicates has no per-draw values");
        cphifi_ctx ctx = o->ctx;
        DeviceGuard dg(ctx->device);
        cudaStream_t s = ctx->stream;
        const int64_t n = p->n, r = p->r, nr = n * r;
        cudaEvent_t ev[3];
        for (auto& e : ev) CPHIFI_CUDA(cudaEventCreate(&e));
        CPHIFI_CUDA(cudaEventRecord(ev[0], s));
        cphifi_solve_report rep{};
        if (solve_report) rep = *solve_report;
        const int st = cphifi_solve_unaligned_pcg(p, cfg, &rep, warm_start, w_out);
        if (st != CPHIFI_OK) {
            for (auto& e : ev) cudaEventDestroy(e);
            throw Error(st, g_last_error);
        }
        if (solve_report) *solve_report = rep;
        CPHIFI_CUDA(cudaEventRecord(ev[1], s));
        const double* wdev = p->pcg_vec.get() + nr;  // the solution stays in the plan's x slot
        DevBuf<double> a(nr), arm((size_t)n * p->rp), scal(4), part(std::max<int64_t>(sq_residual_blocks(o->q_local), RED_PARTIALS) + 80);
        gemm_nn(ctx, n, r, n, p->mode->kernel.get(), n, wdev, n, a.get(), n);  // A_k = K W (als.hpp:214)
        pack_rows(a.get(), n, n, r, p->rp, arm.get(), s);
        SqResidualArgs ra;
        ra.n = n; ra.r = r; ra.rp = p->rp; ra.q = o->q_local; ra.ldq = o->ldq; ra.dother = o->d - 1;
        ra.row_ptr = o->row_ptr.get(); ra.idx = o->idx_o.get(); ra.values = o->values.get();
        ra.fac = p->fac.get();
        for (int m = 0; m < o->d - 1; ++m) ra.fac_off[m] = p->fac_off[m];
        ra.ak = arm.get();
        sq_residual(ra, part.get(), scal.get(), s);                                          // [0] fit^2
        const int64_t nbn = std::min<int64_t>(std::max<int64_t>(1, (o->q_local + 2047) / 2048), 1024);
        if (o->q_local > 0) sq_norm(o->values.get(), o->q_local, part.get(), nbn, scal.get() + 1, s);  // [1] ||v||^2
        else CPHIFI_CUDA(cudaMemsetAsync(scal.get() + 1, 0, sizeof(double), s));
        CPHIFI_CUDA(cudaMemsetAsync(part.get(), 0, sizeof(double) * RED_PARTIALS, s));
        dot_to(wdev, a.get(), nr, part.get(), scal.get() + 2, s);                            // [2] trace(W'KW)
        allreduce(ctx, scal.get(), 2);  // sharded observations: sum the fit and norm terms
        CPHIFI_CUDA(cudaEventRecord(ev[2], s));
        double h[3];
        d2h_sync(h, scal.get(), sizeof(double) * 3, s);
        if (a_out) d2h_sync(a_out, a.get(), sizeof(double) * nr, s);
        float m0 = 0.f, m1 = 0.f;
        CPHIFI_CUDA(cudaEventElapsedTime(&m0, ev[0], ev[1]));
        CPHIFI_CUDA(cudaEventElapsedTime(&m1, ev[1], ev[2]));
        for (auto& e : ev) cudaEventDestroy(e);
        const double dn = std::sqrt(h[1]);
        if (dn == 0.0) throw_runtime("relative_error: zero data norm");
        als->relative_error = std::sqrt(h[0]) / dn;
        als->data_norm = dn;
        als->reg = p->mode->lambda * h[2];
        als->residual = rep.relative_residual;
        als->solve_s = m0 * 1e-3;
        als->update_s = m1 * 1e-3;
    });
}

int cphifi_als_update_infinite_aligned(cphifi_tensor t, cphifi_mode mode, int k, int64_t r,
                                       const double* const* factors, double* w_out, double* a_out,
                                       cphifi_als_report* als) {
    return guard([&] {
        need(t, "tensor");
        need(mode, "mode");
        need(factors, "factors");
        need(w_out, "w_out");
        need(als, "als");
        if (k < 0 || k >= t->d) throw_invalid("unfold: mode out of range");
        if (mode->n != t->shape[k]) throw_invalid("aligned: kernel size mismatch");
        cphifi_ctx ctx = t->ctx;
        DeviceGuard dg(ctx->device);
        cudaStream_t s = ctx->stream;
        mode_eig_once(mode);
        const int64_t n = mode->n, nr = n * r;
        cudaEvent_t ev[3];
        for (auto& e : ev) CPHIFI_CUDA(cudaEventCreate(&e));
        DevBuf<double> fbuf, b(nr), v(r * r), uv(r * r), sv(r), w(nr), t1, core, work;
        std::vector<const double*> fptr;
        upload_factors_cm(ctx, t->d, t->shape.data(), k, r, factors, fbuf, fptr);
        CPHIFI_CUDA(cudaEventRecord(ev[0], s));
        mttkrp_dev(t, k, r, fptr, b.get(), work);
        gram_kr(t->d, t->shape.data(), r, fptr.data(), k, v.get(), s);
        device_sym_eig(ctx, v.get(), r, uv.get(), sv.get());
        const int* flag = decoupled_dev(mode, r, b.get(), uv.get(), sv.get(), w.get(), t1, core);
        CPHIFI_CUDA(cudaEventRecord(ev[1], s));
        DevBuf<double> a(nr), wv(nr), res(nr), g(r * r), scal(8), part(1024 + 80);
        gemm_nn(ctx, n, r, n, mode->kernel.get(), n, w.get(), n, a.get(), n);  // A_k = K W
        // aligned_residual: || K W V + lambda W - B || / ||B||  (as K (W V), one association)
        gemm_nn(ctx, n, r, r, w.get(), n, v.get(), r, wv.get(), n);
        GemmArgs ga;
        ga.m = n; ga.n = r; ga.k = n;
        ga.a = mode->kernel.get(); ga.a_rs = 1; ga.a_cs = n;
        ga.b = wv.get(); ga.b_rs = 1; ga.b_cs = n;
        ga.c = res.get(); ga.c_rs = 1; ga.c_cs = n;
        ga.epi = EPI_AXPY2; ga.e1 = w.get(); ga.e2 = b.get(); ga.ld_e = n; ga.beta1 = mode->lambda; ga.beta2 = -1.0;
        gemm(ga, ctx->num_sms, s);
        // G = A_k' A_k
        GemmArgs gg;
        gg.m = r; gg.n = r; gg.k = n;
        gg.a = a.get(); gg.a_rs = n; gg.a_cs = 1;
        gg.b = a.get(); gg.b_rs = 1; gg.b_cs = n;
        gg.c = g.get(); gg.c_rs = 1; gg.c_cs = r;
        gemm(gg, ctx->num_sms, s);
        auto dot = [&](const double* x, const double* y, int64_t cnt, double* out) {
            CPHIFI_CUDA(cudaMemsetAsync(part.get(), 0, sizeof(double) * RED_PARTIALS, s));
            dot_to(x, y, cnt, part.get(), out, s);
        };
        dot(res.get(), res.get(), nr, scal.get() + 0);  // ||R||^2
        dot(b.get(), b.get(), nr, scal.get() + 1);      // ||B||^2
        dot(a.get(), b.get(), nr, scal.get() + 2);      // <A_k, B>
        dot(g.get(), v.get(), r * r, scal.get() + 3);   // 1'(A_k'A_k o V)1
        dot(w.get(), a.get(), nr, scal.get() + 4);      // trace(W' K W)
        if (!t->have_norm) {  // ||T||^2 of the local slab, once per tensor, summed over shards
            int64_t cnt = n * (t->slab_hi - t->slab_lo);
            for (int m = 2; m < t->d; ++m) cnt *= t->shape[m];
            t->norm2.alloc(1);
            sq_norm(t->data.get(), cnt, part.get(), 1024, t->norm2.get(), s);
            allreduce(ctx, t->norm2.get(), 1);
            t->have_norm = true;
        }
        CPHIFI_CUDA(cudaMemcpyAsync(scal.get() + 5, t->norm2.get(), sizeof(double), cudaMemcpyDeviceToDevice, s));
        CPHIFI_CUDA(cudaEventRecord(ev[2], s));
        double h[6];
        d2h_sync(h, scal.get(), sizeof(double) * 6, s);
        decoupled_check(flag);
        d2h_sync(w_out, w.get(), sizeof(double) * nr, s);
        if (a_out) d2h_sync(a_out, a.get(), sizeof(double) * nr, s);
        float m0 = 0.f, m1 = 0.f;
        CPHIFI_CUDA(cudaEventElapsedTime(&m0, ev[0], ev[1]));
        CPHIFI_CUDA(cudaEventElapsedTime(&m1, ev[1], ev[2]));
        for (auto& e : ev) cudaEventDestroy(e);
        const double tn = std::sqrt(h[5]);
        if (tn == 0.0) throw_runtime("relative_error: zero data norm");
        const double fit2 = h[5] - 2.0 * h[2] + h[3];
        als->relative_error = std::sqrt(std::max(fit2, 0.0)) / tn;
        als->data_norm = tn;
        als->reg = mode->lambda * h[4];
        const double bn = std::sqrt(h[1]);
        als->residual = bn == 0.0 ? std::sqrt(h[0]) : std::sqrt(h[0]) / bn;
        als->solve_s = m0 * 1e-3;
        als->update_s = m1 * 1e-3;
    });
}
}  // extern "C"
