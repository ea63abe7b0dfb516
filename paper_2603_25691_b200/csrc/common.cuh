// common.cuh — shared internals of libcphifi_b200 (not part of the public ABI).
#pragma once

#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <nccl.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/cphifi_b200.h"

namespace cphifi {

// ---- error plumbing: C++ exceptions inside, int status at the ABI --------------------
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void throw_invalid(const std::string& m) { throw Error(CPHIFI_INVALID_ARGUMENT, m); }
[[noreturn]] inline void throw_runtime(const std::string& m) { throw Error(CPHIFI_RUNTIME_ERROR, m); }

void set_last_error(const std::string& m);

#define CPHIFI_CUDA(call)                                                                   \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            throw ::cphifi::Error(CPHIFI_CUDA_ERROR, std::string(#call) + ": " +             \
                                                         cudaGetErrorString(e_));           \
    } while (0)
#define CPHIFI_CHECK_LAUNCH() CPHIFI_CUDA(cudaGetLastError())
#define CPHIFI_NCCL(call)                                                                   \
    do {                                                                                    \
        ncclResult_t r_ = (call);                                                           \
        if (r_ != ncclSuccess)                                                              \
            throw ::cphifi::Error(CPHIFI_NCCL_ERROR, std::string(#call) + ": " +             \
                                                         ncclGetErrorString(r_));           \
    } while (0)
#define CPHIFI_SOLVER(call)                                                                 \
    do {                                                                                    \
        cusolverStatus_t s_ = (call);                                                       \
        if (s_ != CUSOLVER_STATUS_SUCCESS)                                                  \
            throw ::cphifi::Error(CPHIFI_CUDA_ERROR,                                        \
                                  std::string(#call) + ": cusolver status " + std::to_string((int)s_)); \
    } while (0)

// ---- device buffer (RAII) ------------------------------------------------------------
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t count) {
        release();
        if (count) CPHIFI_CUDA(cudaMalloc(&p, count * sizeof(T)));
        n = count;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    T* get() const { return p; }
};

// cudaFuncSetAttribute once per (kernel, attribute, device): attributes are per device, so a
// process-wide "done" flag would leave a second GPU without them.  Thread-safe.
void func_attr_once(const void* f, cudaFuncAttribute attr, int value);

inline int64_t pow2_at_least(int64_t v, int64_t lo) {
    int64_t p = lo;
    while (p < v) p <<= 1;
    return p;
}

}  // namespace cphifi

// ---- opaque handle definitions -------------------------------------------------------
// Virtual communicator (test hook, include/cphifi_b200.h): `nranks` contexts on ONE GPU, each
// driven by its own host thread, exchange partial sums the way NCCL ranks do.  A collective is a
// host barrier (every rank has published its send buffer and a "ready" event), a rank-order sum
// on each rank's own stream after waiting on every ready event, and a "done" event every rank
// waits on before touching its buffers again.  No kernel ever waits on another kernel.
struct cphifi_vcomm_s {
    int nranks = 0;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    std::vector<const double*> send;
    std::vector<cudaEvent_t> ready, done;
    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const uint64_t g = gen;
        if (++arrived == nranks) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

struct cphifi_ctx_s {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    cusolverDnHandle_t solver = nullptr;
    ncclComm_t comm = nullptr;
    cphifi_vcomm_s* vcomm = nullptr;     // virtual communicator (one-GPU test hook), or null
    cphifi::DevBuf<double> vc_scratch;   // this rank's reduction output before the copy-out
    int nranks = 1, rank = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // pinned scratch for small D2H reads (PCG scalars)
    double* host_scalars = nullptr;
};

struct cphifi_mode_s {
    cphifi_ctx ctx = nullptr;
    int64_t n = 0;
    double lambda = 0.0;
    cphifi::DevBuf<double> kernel;  // n x n column-major (symmetric)
    cphifi::DevBuf<double> u;       // eigenvectors, n x n column-major
    cphifi::DevBuf<double> mu;      // eigenvalues (ascending, clamped at 0)
    cphifi::DevBuf<double> ut;      // U' (k_sandwich.cu phase 2), built on first use
    bool have_ut = false;
    cphifi::DevBuf<double> um;      // U diag(mu) (eigenbasis PCG: K X = U diag(mu) U'X), lazily
    bool have_um = false;
    cphifi::DevBuf<double> umt;     // diag(mu) U' (the fused kernel's Xhat columns in the eigenbasis)
    bool have_umt = false;
    int64_t nzero = -1;             // leading exactly-zero (clamped) eigenvalues, rounded down to 8; lazily
    uint64_t eig_gen = 0;           // bumped whenever (U, mu) are replaced: keys the plans' captured graphs
    bool psd = true;                // K positive semidefinite up to rounding (eigenbasis PCG allowed)
    std::once_flag once;
    bool have_eig = false;
    int eig_count = 0;
    std::mutex mu_lock;
};

// One part of the operator's q-pass for the run kernel (k_runs.cu): the plan entries whose LAST
// other-mode index falls in rows [row_lo, row_lo + rows) of that factor (all of them when the
// whole factor fits shared memory: the part then aliases the plan), in plan order, that index
// rebased to the block, with their own CSR, run table and per-warp entry ranges.
struct StreamPart {
    int64_t q = 0, ldq = 0;              // entries; column stride (multiple of 4)
    int64_t row_lo = 0, rows = 0;        // block of the last other mode
    const int32_t* idx = nullptr;        // (d-1) x ldq, last column rebased
    const int32_t* mult = nullptr;       // coalesced plans
    const int64_t* row_ptr = nullptr;    // n + 1
    cphifi::DevBuf<int32_t> idx_own, mult_own;  // owned copies (block parts)
    cphifi::DevBuf<int64_t> row_ptr_own;
    int64_t sf = 0;                      // staged factor doubles
    cphifi::DevBuf<int32_t> run_start, run_i1;  // run table (nruns + 1 / nruns)
    int64_t nruns = 0;
    int64_t draws = 0;                   // draws the part's entries stand for (sum of multiplicities)
    int warps = 0;                       // equal-count warp ranges
    cphifi::DevBuf<int64_t> warp_beg, warp_rows;
    cphifi::DevBuf<int32_t> row_first_w, row_nw;
    bool padded = false;                 // runs padded to even lengths, run starts flagged (k_xruns.cu)
    cphifi::DevBuf<double> vals_own;     // the observed values in part order (the right-hand side B)
    const double* vals = nullptr;
    int64_t q_real = 0;                  // entries before the padding
    int g_units = 0;                     // the row-Gram build's equal-count units (built on first use)
    cphifi::DevBuf<int64_t> g_beg, g_rows;
    cphifi::DevBuf<int32_t> g_rfc, g_rnc;
};

// The stream operator's q-pass plan for one padded rank (capi.cu build_run_parts): the run kernel's
// parts over the sparse rows, the dense rows' multiplicity grids (k_dense_rows.cu), and the dense
// rows' entries cut into the same factor blocks (the row-Gram build over parts).  It depends only on
// the observation plan and the padded rank, so every subproblem built on the same plan shares it
// (cphifi_obs_s::qp_cache): an ALS sweep's fresh subproblems reuse it.
struct QpassPlan {
    std::vector<StreamPart> parts;        // non-empty: the q-pass is the run kernel over these
    std::vector<StreamPart> dense_parts;  // the dense rows' entries, block h in dense_parts[h]
    int dense_nd = 0;                     // dense rows, 0: none
    int64_t dense_n1 = 0, dense_n2 = 0, dense_n1p = 0, dense_n2p = 0;
    cphifi::DevBuf<int32_t> dense_rows, dense_w;  // their row indices; nd x n1p x n2p multiplicities
    int max_warps = 0;                    // over the parts
};

struct cphifi_obs_s {
    cphifi_ctx ctx = nullptr;
    int d = 0, k = 0;
    std::vector<int64_t> shape;
    int64_t q_total = 0;  // all shards
    int64_t q_local = 0;  // this shard
    double density = 0.0; // q_total / prod(shape)  (observations.hpp:58-60)
    bool lex = false;     // plan order is lexicographic (i_k, other modes ascending)
    cphifi::DevBuf<int64_t> row_ptr;  // n_k + 1, local CSR over sorted i_k
    cphifi::DevBuf<int32_t> idx_o;    // (d-1) columns of stride ldq, other modes ascending, sorted by i_k
    int64_t ldq = 0;                  // idx_o column stride: q_local rounded up to a multiple of 4
    cphifi::DevBuf<double> values;    // q_local, sorted (coalesced: summed over duplicates)
    cphifi::DevBuf<int32_t> mult;     // q_local multiplicities (coalesced plans only)
    bool coalesced = false;
    // multi-rank row ranges (capi.cu shard_rows), multiples of 8 rows: this rank OWNS rows [own_lo,
    // own_hi) (a partition of [0, n_k) over the shards) and its observations lie inside [own_lo, hull_hi)
    int shards = 1, shard = 0;
    int64_t own_lo = 0, own_hi = 0, hull_hi = 0;
    std::mutex qp_mu;                 // q-pass plans by padded rank (and the tuning knobs they read)
    std::map<std::string, std::shared_ptr<QpassPlan>> qp_cache;
};

struct cphifi_unaligned_s {
    cphifi_obs obs = nullptr;
    cphifi_mode mode = nullptr;
    int64_t n = 0, r = 0, rp = 0;  // rank and padded rank (power of two >= 4)
    double rho = 1e-6;
    std::vector<int64_t> fac_off;     // offsets of the packed row-major padded factors
    cphifi::DevBuf<double> fac;       // packed other-mode factors, row-major n_m x rp
    cphifi::DevBuf<double> b;         // n x r column-major (sampled MTTKRP with values)
    cphifi::DevBuf<double> v;         // r x r
    // preconditioner state (lazy): eig(V), D
    bool have_veig = false;
    cphifi::DevBuf<double> uv, sv, dmat;
    uint64_t veig_gen = 0;        // bumped whenever (U_V, sigma_V) / D are replaced (graph key)
    // fused operator kernel launch shape (k_fused.cu)
    int grid = 0;                 // CTAs (all co-resident)
    cphifi::DevBuf<int64_t> cta_beg;        // grid + 1 partition boundaries
    cphifi::DevBuf<int32_t> row_first_cta;  // n
    cphifi::DevBuf<int32_t> row_ncta;       // n
    size_t smem = 0;              // dynamic shared memory bytes
    bool smem_factors = false;    // factors staged in shared memory
    bool small_n = false;         // phases A and C2 inside the fused kernel
    bool local_x = false;         // every CTA spans <= MAXLOC rows: CTA-local Xhat (PH_AL)
    bool prefetch = false;        // X and K columns staged in shared memory (small n * r)
    bool stream = false;          // phase B runs k_stream.cu (large plans) instead of k_fused.cu
    int64_t stream_sf = 0;        // doubles of per-observation factors k_stream.cu stages in smem (0: L1)
    std::shared_ptr<QpassPlan> qp;  // the plan's shared q-pass plan (ensure_runs); null: not built
    cphifi::DevBuf<double> runs_slot_a, runs_slot_b;  // warps x rp: split-row partials of the run kernel
    cphifi::DevBuf<double> dense_partial;         // per-task partial rows of the dense-rows kernel
    cphifi::DevBuf<unsigned> dense_cnt;           // per-row arrival counters
    bool runs_pending = false;    // parts not built yet (ensure_runs)
    int64_t runs_sf = 0;          // staged per-observation factor doubles of the whole plan
    cphifi::DevBuf<unsigned> rowcnt;   // n per-row arrival counters
    // row-Gram operator (k_gram.cu): op = 0 per-observation stream, 1 row-Gram
    int op = 0;
    cphifi::DevBuf<double> gram;            // n x rp x rp (built lazily)
    cphifi::DevBuf<double> gram_sum;         // multi-rank finite-mode update: the all-shard row Grams
    cphifi::DevBuf<double> yhat_sum;   // n x rp NCCL all-reduce output (multi-GPU); the row-sharded output operand
    cphifi::DevBuf<double> y_part;     // n x r: this rank's K[:, rows] B[rows, :] (row-sharded operator)
    cphifi::DevBuf<int64_t> cta_rows;   // 2 x grid
    cphifi::DevBuf<unsigned> barrier;   // grid barrier state
    cphifi::DevBuf<double> slot_a, slot_b;  // grid x rp
    cphifi::DevBuf<double> xhat_rm, yhat_rm;  // n x rp row-major
    cphifi::DevBuf<double> xhat_cm;           // n x r column-major
    cphifi::DevBuf<double> t1, t2;            // n x r scratch (preconditioner)
    cphifi::DevBuf<double> vx, vy;            // n x r device in/out for host-buffer calls
    // device-resident PCG: persistent vectors + a CUDA graph whose WHILE node runs the iterations
    cphifi::DevBuf<double> pcg_vec;           // b, x, r, z, p, Ap (n r each)
    cphifi::DevBuf<double> pcg_aux;           // reduction partials | PcgState | PcgCtl
    cphifi::DevBuf<double> pcg_step;          // fused vector step (k_pcgstep.cu): barrier word | partials
    int64_t pcg_graph_z = -1, pcgf_z = -1;    // mode_nzero baked into the captured graphs
    uint64_t pcg_graph_gen = ~0ull, pcgf_gen = ~0ull;  // eigendecomposition generations baked into them
    cphifi::DevBuf<double> pcg_hist;          // device residual history
    cudaGraph_t pcg_graph = nullptr;
    cudaGraphExec_t pcg_exec = nullptr;
    // host-buffer matvec (cphifi_unaligned_matvec) as one graph [copy in, operator, copy out]
    // over plan-owned pinned, device-mapped staging buffers hv_hx / hv_hy
    cudaGraph_t hv_graph = nullptr;
    cudaGraphExec_t hv_exec = nullptr;
    double* hv_hx = nullptr;
    double* hv_hy = nullptr;
    bool hv_failed = false;
    int hv_op = -1;                           // operator form baked into hv_exec / hd_exec
    // large x / y in pinned host memory: [DMA in] operator graph [DMA out] (no host staging copy)
    cudaGraph_t hd_graph = nullptr;
    cudaGraphExec_t hd_exec = nullptr;
    int hd_op = -1;
    // the dense rows' q-pass on a second stream, concurrent with the run kernel's parts (they write
    // disjoint rows of Yhat): forked after the Yhat zeroing, joined before the output GEMM
    cudaStream_t side = nullptr;
    cudaEvent_t side_fork = nullptr, side_join = nullptr;
    int pcg_graph_op = -1;                    // operator form the graph was captured with
    int pcg_graph_rot = -1;                   // basis (0 original, 1 eigenbasis) of the captured graph
    // the whole solve after the right-hand side as one graph: [bnorm, x0, M^-1 r0, init, loop
    // control] -> WHILE(iteration) -> [W = U x~]
    cudaGraph_t pcgf_graph = nullptr;
    cudaGraphExec_t pcgf_exec = nullptr;
    int pcgf_op = -1, pcgf_rot = -1;
    bool pcg_graph_failed = false;
    ~cphifi_unaligned_s() {
        if (pcg_exec) cudaGraphExecDestroy(pcg_exec);
        if (pcg_graph) cudaGraphDestroy(pcg_graph);
        if (pcgf_exec) cudaGraphExecDestroy(pcgf_exec);
        if (pcgf_graph) cudaGraphDestroy(pcgf_graph);
        if (hv_exec) cudaGraphExecDestroy(hv_exec);
        if (hv_graph) cudaGraphDestroy(hv_graph);
        if (hd_exec) cudaGraphExecDestroy(hd_exec);
        if (hd_graph) cudaGraphDestroy(hd_graph);
        if (side_fork) cudaEventDestroy(side_fork);
        if (side_join) cudaEventDestroy(side_join);
        if (side) cudaStreamDestroy(side);
        if (hv_hx) cudaFreeHost(hv_hx);
        if (hv_hy) cudaFreeHost(hv_hy);
    }
};

struct cphifi_tensor_s {
    cphifi_ctx ctx = nullptr;
    int d = 0;
    std::vector<int64_t> shape;        // full shape
    int64_t slab_lo = 0, slab_hi = 0;  // mode-1 slice range held locally
    cphifi::DevBuf<double> data;       // local slab, column-major n0 x (hi-lo) x n2 x ...
    cphifi::DevBuf<double> norm2;      // ||T||^2 over all shards (ALS relative error), lazily
    bool have_norm = false;
};

