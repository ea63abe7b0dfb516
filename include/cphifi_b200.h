/*
 * cphifi_b200.h — C-ABI of the B200-native CP-HIFI infinite-mode subproblem solver.
 *
 * This is the drop-in boundary for the reference's hot path.  Every
 * entry point below replaces one reference C++ function or object; the citation on each
 * is `file:line` relative to /root/reference/proj/include/cphifi/.  All matrices are
 * fp64 COLUMN-MAJOR (first index fastest), exactly as Eigen::MatrixXd in the reference
 * (tensor.hpp:12-13); vec(W) of an n x r matrix is i + n*j.  Indices are 0-based.
 *
 * Conventions
 *  - No C++ types and no exceptions cross this boundary.  Every function returns an
 *    int status; on failure cphifi_last_error() returns a thread-local message that
 *    reuses the reference's exception text where one exists.
 *      CPHIFI_INVALID_ARGUMENT  <-> std::invalid_argument in the reference
 *      CPHIFI_RUNTIME_ERROR     <-> std::runtime_error in the reference
 *      CPHIFI_CUDA_ERROR / CPHIFI_NCCL_ERROR: device or collective failures
 *  - Host pointers are plain host memory (pinned or pageable) unless a function name
 *    ends in _device, in which case they are device pointers on the context's GPU and the
 *    call is asynchronous on the context stream.
 *  - There is no CPU fallback: every compute entry point runs sm_100a kernels.  On a
 *    machine without a usable GPU cphifi_ctx_create fails with CPHIFI_CUDA_ERROR.
 *  - Thread safety mirrors the reference objects: different handles may be used from
 *    different host threads; one handle is not re-entrant.
 */
#ifndef CPHIFI_B200_H
#define CPHIFI_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CPHIFI_ABI_VERSION 1

enum cphifi_status {
    CPHIFI_OK = 0,
    CPHIFI_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    CPHIFI_RUNTIME_ERROR = 2,    /* std::runtime_error in the reference */
    CPHIFI_CUDA_ERROR = 3,
    CPHIFI_NCCL_ERROR = 4
};

typedef struct cphifi_ctx_s* cphifi_ctx;             /* device, stream, optional NCCL comm */
typedef struct cphifi_mode_s* cphifi_mode;           /* RkhsMode analogue (kernel.hpp:53-101) */
typedef struct cphifi_obs_s* cphifi_obs;             /* ObservationSet analogue (observations.hpp:18-79) */
typedef struct cphifi_unaligned_s* cphifi_unaligned; /* UnalignedSubproblem (unaligned.hpp:18-33) */
typedef struct cphifi_tensor_s* cphifi_tensor;       /* DenseTensor (tensor.hpp:14-68), device-resident */

/* PcgConfig (solvers.hpp:23-27). Defaults in the reference: tol 1e-6, max_iter 75. */
typedef struct cphifi_pcg_config {
    double tol;
    int32_t max_iter;
    int32_t record_history;
} cphifi_pcg_config;

/* SolveReport (solvers.hpp:29-35) plus a phase breakdown.  residual_history is a
 * CALLER-OWNED buffer of history_capacity doubles (>= max_iter + 1 to hold the whole
 * history); history_len receives the number of entries the reference would record. */
typedef struct cphifi_solve_report {
    int32_t iterations;
    int32_t converged;
    double relative_residual;
    double wall_time_s;
    double* residual_history;
    int32_t history_capacity;
    int32_t history_len;
    /* B200 extras (seconds, CUDA-event timed on the context stream) */
    double setup_s;    /* RHS K*B, eig(V), preconditioner diagonal */
    double matvec_s;   /* total time in the operator */
    double precond_s;  /* total time in M^-1 applies */
    int32_t matvecs;   /* operator applications */
    int32_t pad_;
} cphifi_solve_report;

/* ---- status / context ------------------------------------------------------------ */
const char* cphifi_last_error(void);
int cphifi_abi_version(void);

/* One context per (process, GPU). */
int cphifi_ctx_create(int device, cphifi_ctx* out);
int cphifi_ctx_destroy(cphifi_ctx ctx);
int cphifi_ctx_synchronize(cphifi_ctx ctx);
/* The context's CUDA stream (cudaStream_t) so callers can order their own work. */
int cphifi_ctx_stream(cphifi_ctx ctx, void** stream_out);
/* Measured FP64 peaks of this GPU (TFLOP/s): a DFMA loop and a DMMA (m8n8k4) loop — the FP64
 * roofline denominators. */
int cphifi_fp64_peak(cphifi_ctx ctx, double* dfma_tflops, double* dmma_tflops);
/* Multi-GPU: NCCL communicator over `nranks` processes (one per GPU).  Rank 0 creates the
 * 128-byte id with cphifi_comm_unique_id and distributes it (e.g. torch.distributed).
 * Once set, operator applications all-reduce the n x r partial accumulator. */
int cphifi_comm_unique_id(uint8_t id_out[128]);
int cphifi_ctx_init_comm(cphifi_ctx ctx, int nranks, int rank, const uint8_t id[128]);
int cphifi_ctx_world(cphifi_ctx ctx, int* nranks, int* rank);
/* Test hook: a VIRTUAL communicator of `nranks` (<= 8) contexts on ONE GPU, each driven by its own
 * host thread, that stands in for NCCL so every multi-rank code path (sharded observations with the
 * n x r all-reduce per application, the host-loop PCG, the sharded aligned MTTKRP) runs without a
 * second GPU.  Collectives sum the ranks' buffers in rank order; like NCCL, every rank must issue
 * the same collectives in the same order.  Attach with cphifi_ctx_init_vcomm before creating
 * plans; destroy the communicator after its contexts. */
typedef struct cphifi_vcomm_s* cphifi_vcomm;
int cphifi_vcomm_create(int nranks, cphifi_vcomm* out);
int cphifi_vcomm_destroy(cphifi_vcomm vc);
int cphifi_ctx_init_vcomm(cphifi_ctx ctx, cphifi_vcomm vc, int rank);

/* ---- mode (RkhsMode, kernel.hpp:53-101) ------------------------------------------- */
/* RkhsMode(points, sigma, lambda): Gaussian kernel K(i,j)=exp(-(x_i-x_j)^2/(2 sigma^2))
 * built on device (gaussian_kernel, kernel.hpp:17-30); throws like the reference for
 * sigma <= 0 and lambda < 0. */
int cphifi_mode_create_gaussian(cphifi_ctx ctx, int64_t n, const double* points,
                                double sigma, double lambda, cphifi_mode* out);
/* Matern-3/2 kernel (1 + sqrt3 d/l) exp(-sqrt3 d/l); not in the reference. */
int cphifi_mode_create_matern32(cphifi_ctx ctx, int64_t n, const double* points,
                                double lengthscale, double lambda, cphifi_mode* out);
/* Caller-supplied symmetric K (n x n column-major). */
int cphifi_mode_create(cphifi_ctx ctx, int64_t n, const double* kernel, double lambda,
                       cphifi_mode* out);
int cphifi_mode_destroy(cphifi_mode mode);
int cphifi_mode_size(cphifi_mode mode, int64_t* n);
int cphifi_mode_lambda(cphifi_mode mode, double* lambda);
int cphifi_mode_get_kernel(cphifi_mode mode, double* kernel_out);
/* RkhsMode::eig (kernel.hpp:77-83 -> sym_eig :40-49): symmetry check at
 * 1e-12*max(scale,1), device syevd, clamp at 0; computed at most once. */
int cphifi_mode_eig(cphifi_mode mode);
/* Shared eigendecomposition: install (U_K, mu_K) from outside, counted as the
 * one factorization.  mu is clamped at 0 exactly as sym_eig does. */
int cphifi_mode_set_eig(cphifi_mode mode, const double* u, const double* mu);
int cphifi_mode_get_eig(cphifi_mode mode, double* u_out, double* mu_out);
int cphifi_mode_eig_count(cphifi_mode mode, int* count); /* eig_factorization_count */

/* ---- observations (ObservationSet, observations.hpp:18-79) ------------------------- */
#define CPHIFI_OBS_DEVICE_INPUT 1u      /* idx / values are device pointers */
#define CPHIFI_OBS_REJECT_DUPLICATES 2u /* reference semantics: throw on a repeated index */
/* multiset input: merge repeated multi-indices into one plan entry carrying its multiplicity
   (operator weight) and summed value (right-hand side); q_local then counts distinct entries */
#define CPHIFI_OBS_COALESCE_DUPLICATES 4u
/* shards > 1: cut the sorted order into equal counts of observations [q*s/S, q*(s+1)/S) instead
   of the default cost-balanced cut (below) */
#define CPHIFI_OBS_SHARD_EQUAL_COUNT 8u
/* shards > 1: balance the shards' PLAN ENTRIES (distinct cells when coalescing) instead of their
   modelled q-pass time — the right cut when the plan is used with the row-Gram operator, whose
   build costs 2 rp^2 flops per plan entry whether the row is dense or not (same row-aligned cuts) */
#define CPHIFI_OBS_SHARD_BY_ENTRIES 16u
/* Build the observation plan for infinite mode k: q multi-indices stored as d int32
 * arrays (idx[m*q + l] = index of observation l in mode m), fp64 values.  The plan sorts
 * by i_k on device (stable), builds CSR row pointers, and keeps one contiguous shard of the
 * sorted order (s = shard, S = shards; use 0/1 for a single GPU).  Shards are cost-balanced:
 * a row counts its plan entries (distinct cells when coalescing), or the fixed cost of the GEMM
 * form when the q-pass runs it as a dense row, and cuts fall on row boundaries unless one row
 * exceeds a quarter of a shard — so a skewed set (config 4's Zipf rows) spreads its q-pass
 * TIME, not its draws, evenly over the GPUs; every rank derives the same cuts.
 * Range errors throw "ObservationSet: index out of range". */
int cphifi_obs_create(cphifi_ctx ctx, int d, const int64_t* shape, int64_t q,
                      const int32_t* idx, const double* values, int k, uint32_t flags,
                      int shard, int shards, cphifi_obs* out);
int cphifi_obs_destroy(cphifi_obs obs);
int cphifi_obs_info(cphifi_obs obs, int64_t* q_total, int64_t* q_local, double* density);
/* Row ranges of this shard (multiples of 8 rows of mode k): it OWNS rows [own_lo, own_hi) — a
 * partition of [0, n_k) over the shards — and its observations lie in rows [own_lo, hull_hi).  The
 * row-sharded operator (large n, stream operator) contracts only these rows of K on each rank and
 * all-reduces the n x r partial result.  One shard: [0, n_k), n_k. */
int cphifi_obs_shard_rows(cphifi_obs obs, int64_t* own_lo, int64_t* own_hi, int64_t* hull_hi);

/* ---- unaligned subproblem (unaligned.hpp:18-161) ---------------------------------- */
/* make_unaligned_subproblem(obs, model, k, mode, rho) (unaligned.hpp:35-48): factors[m]
 * is the n_m x r column-major factor of mode m (factors[k] is ignored and may be NULL).
 * Builds B = sampled_mttkrp(values) (all-reduced over shards) and V = gram_khatri_rao. */
/* (mode may be NULL: a finite-mode subproblem for cphifi_als_update_finite_unaligned) */
int cphifi_unaligned_create(cphifi_obs obs, cphifi_mode mode, int64_t r,
                            const double* const* factors, double rho,
                            cphifi_unaligned* out);
int cphifi_unaligned_destroy(cphifi_unaligned p);
int cphifi_unaligned_get_b(cphifi_unaligned p, double* b_out);  /* n x r */
int cphifi_unaligned_get_v(cphifi_unaligned p, double* v_out);  /* r x r */
/* Operator form used by matvec / PCG.  STREAM is the reference's structure: every application
 * gathers and scatters over all q observations (observations.hpp:174-198).  GRAM uses the exact
 * identity Yhat(i,:) = G_i Xhat(i,:), G_i = sum_{l in row i} z_l z_l', with G built once per plan
 * (O(q rp^2), counted in the solve's setup_s / wall_time_s); each application is then O(n rp^2).
 * AUTO picks GRAM when n is not small, rp <= 64 and the rows carry on average >= 2 rp
 * observations.  A new plan starts with AUTO's choice. */
#define CPHIFI_OP_STREAM 0
#define CPHIFI_OP_GRAM 1
#define CPHIFI_OP_AUTO 2
int cphifi_unaligned_set_operator(cphifi_unaligned p, int op);
int cphifi_unaligned_get_operator(cphifi_unaligned p, int* op);
/* unaligned_matvec (unaligned.hpp:101-115): y = vec(K*Yhat + lambda*K*X) + rho*x. */
int cphifi_unaligned_matvec(cphifi_unaligned p, const double* x, double* y);
int cphifi_unaligned_matvec_device(cphifi_unaligned p, const double* x, double* y);
/* build_preconditioner(p).apply (unaligned.hpp:120-140): eig(V) is computed on first use;
 * cphifi_unaligned_set_v_eig installs a shared (U_V, sigma_V) instead. */
int cphifi_unaligned_set_v_eig(cphifi_unaligned p, const double* u_v, const double* sigma_v);
int cphifi_unaligned_get_v_eig(cphifi_unaligned p, double* u_v_out, double* sigma_v_out);
int cphifi_unaligned_precond_apply(cphifi_unaligned p, const double* x, double* y);
int cphifi_unaligned_precond_apply_device(cphifi_unaligned p, const double* x, double* y);
/* solve_unaligned_pcg (unaligned.hpp:143-161) with pcg (solvers.hpp:38-88).  warm_start
 * (n x r, may be NULL) maps directly to x0.  w_out receives W (n x r). */
int cphifi_solve_unaligned_pcg(cphifi_unaligned p, const cphifi_pcg_config* cfg,
                               cphifi_solve_report* report, const double* warm_start,
                               double* w_out);
/* Benchmark hook: `iters` operator applications on DEVICE buffers x, y with CUDA events on
 * the context stream around each phase; ms_out[0..5] receives the mean milliseconds of
 * [0] Xhat = K X, [1] scatter-gather main kernel(s) (K1: the run kernel's parts when planned),
 * [2] the dense-rows kernel (k_dense_rows.cu; 0 when the plan has none), [3] all-reduce,
 * [4] y = K Yhat + lambda Xhat + rho x, [5] the whole matvec. */
int cphifi_unaligned_matvec_timed(cphifi_unaligned p, const double* x, double* y, int iters,
                                  double* ms_out);
/* Throughput hook: `steps` operator applications back to back in ONE CUDA graph, application t
 * on plan ps[t % m] with its own DEVICE buffers xs / ys; *total_ms = the event-timed graph (after
 * one warm-up launch).  With m plans whose working sets together exceed L2, every application
 * starts L2-cold with no flush inside the timed region. */
int cphifi_unaligned_matvec_cycle_timed(const cphifi_unaligned* ps, const double* const* xs,
                                        double* const* ys, int m, int steps, float* total_ms);
/* Benchmark hook: `steps` operator applications on DEVICE buffers x, y captured in ONE CUDA
 * graph, each preceded (outside its event pair) by a memset of `flush_bytes` at `flush` that
 * evicts L2; the graph is launched once to warm up and once timed.  ms_out[i] receives the
 * event-timed milliseconds of application i (the per-launch host overhead of a plain launch is
 * not in them: the way the operator runs inside the device-resident PCG loop). */
int cphifi_unaligned_matvec_graph_timed(cphifi_unaligned p, const double* x, double* y, void* flush,
                                        size_t flush_bytes, int steps, float* ms_out);
/* Benchmark hook: *kernels = how many kernels of this library one operator application launches
 * (one application captured into a CUDA graph and its kernel nodes counted; the all-reduce of a
 * multi-rank plan is not a kernel of this library and is left out of the capture). */
int cphifi_unaligned_matvec_launches(cphifi_unaligned p, const double* x, double* y, int* kernels);
/* Tracing hook: one operator application on DEVICE buffers with per-CTA %globaltimer stamps
 * (8 per CTA: entry, phase A done, barrier 1, phase B done, barrier 2, fix-up done,
 * barrier 3, exit; 0 = phase not run).  *ctas receives the CTA count. */
int cphifi_unaligned_matvec_trace(cphifi_unaligned p, const double* x, double* y,
                                  uint64_t* stamps, int capacity, int* ctas);
/* Introspection: the stream operator's q-pass plan (built on first use).  info[0..count) receives
 * [0] run-kernel parts (0: the whole plan on the stream kernel), [1] rows handled in the GEMM form
 * (k_dense_rows.cu; CPHIFI_DENSE_MIN sets the density threshold, 0 turns it off), [2] plan entries
 * left to the run kernel, [3] the draws those entries stand for (-1 without parts), [4] / [5] the
 * dense grids' padded n_1 / n_2, [6] parts run by the cross-run kernel (k_xruns.cu: their runs
 * padded to even lengths, so [2] counts the padding; CPHIFI_XRUNS=0 turns it off), [7] the entries
 * of [2] before the padding; further slots 0. */
int cphifi_unaligned_qpass_plan(cphifi_unaligned p, int64_t* info, int count);
/* Test hook: Yhat = sampled_mttkrp(gather_rows(Xhat)) for a given Xhat (n x r), i.e.
 * observations.hpp:174-198 fused, before the final K multiply (all-reduced). */
int cphifi_unaligned_scatter_gather(cphifi_unaligned p, const double* xhat, double* yhat_out);

/* ---- aligned path (tensor.hpp:174-194, aligned.hpp:41-54) ------------------------- */
#define CPHIFI_TENSOR_DEVICE_INPUT 1u
/* Dense d-way tensor, column-major.  With shards > 1 the tensor is split over mode-1
 * (second mode) slices and this process keeps slice range [n1*s/S, n1*(s+1)/S); `data`
 * is the FULL tensor (host) or, with CPHIFI_TENSOR_DEVICE_INPUT, already the local slab
 * (n0 x local_n1 x n2 ...). */
int cphifi_tensor_create(cphifi_ctx ctx, int d, const int64_t* shape, const double* data,
                         uint32_t flags, int shard, int shards, cphifi_tensor* out);
int cphifi_tensor_destroy(cphifi_tensor t);
/* mttkrp(t, model, k) = unfold(t,k) * khatri_rao_excluding(model,k) (tensor.hpp:174-182);
 * k = 0 (the infinite mode) is the accelerated path.  All-reduced over shards. */
int cphifi_mttkrp(cphifi_tensor t, int k, int64_t r, const double* const* factors,
                  double* b_out);
/* gram_khatri_rao(model, k) (tensor.hpp:186-194): Hadamard product of A_m' A_m, m != k. */
int cphifi_gram_khatri_rao(cphifi_ctx ctx, int d, const int64_t* shape, int64_t r,
                           const double* const* factors, int k, double* v_out);
/* solve_aligned_decoupled (aligned.hpp:41-54): W = U_K((U_K' B U_V) ./ (sigma_j mu_i +
 * lambda)) U_V'.  u_v / sigma_v may be NULL (eig(V) on device) or a shared eig (F1). */
int cphifi_solve_aligned_decoupled(cphifi_mode mode, int64_t r, const double* b,
                                   const double* v, const double* u_v,
                                   const double* sigma_v, double* w_out);
/* ---- aligned baselines: the reference's comparison solvers on device --- */
/* aligned_matvec (aligned.hpp:58-67): y = vec(diag(d_k) X V + lambda X), X n x r column-major. */
int cphifi_aligned_matvec(cphifi_ctx ctx, int64_t n, int64_t r, const double* x, const double* d_k,
                          const double* v, double lambda, double* y);
/* solve_aligned_pcg (aligned.hpp:72-100): PCG (solvers.hpp:38-88) on (V kron D_K + lambda I)
 * vec(Wbar) = vec(U_K' B) with the diagonal preconditioner diag(V) kron D_K + lambda I, then
 * W = U_K Wbar.  warm_start (n x r) may be NULL (the reference rotates it: U_K' W0). */
int cphifi_solve_aligned_pcg(cphifi_mode mode, int64_t r, const double* b, const double* v,
                             const cphifi_pcg_config* cfg, cphifi_solve_report* report,
                             const double* warm_start, double* w_out);
/* solve_aligned_direct (aligned.hpp:28-37): the rn x rn system V kron K + lambda I materialised
 * and Cholesky-solved (cuSOLVER potrf/potrs); std::invalid_argument when rn > direct_cap
 * (reference default 6000), std::runtime_error when not positive definite. */
int cphifi_solve_aligned_direct(cphifi_mode mode, int64_t r, const double* b, const double* v,
                                int64_t direct_cap, double* w_out);
/* ---- unaligned direct / dense baselines (unaligned.hpp:52-96, 164-174) ----
 * solve_unaligned_direct_nonsym: LU solve (cuSOLVER getrf/getrs, lu_solve's residual check and
 * message, solvers.hpp:99-106) of (G'F + lambda I) vec(W) = vec(B), the system assembled on device
 * from the row Grams ((G'F)[(j,i),(j',i')] = G_i(j,j') K(i,i')) instead of the q x rn factors;
 * std::invalid_argument when rn > dense_cap (reference default 6000).  report: iterations 1, the
 * relative residual, wall time.  assemble_unaligned_sym_dense: the symmetric test oracle
 * F'F + lambda (I kron K) + rho I (rn x rn, column-major) and vec(K B), F'F = K S with the Gram-scaled
 * columns S on the DMMA GEMM. */
int cphifi_solve_unaligned_direct_nonsym(cphifi_unaligned p, int64_t dense_cap, cphifi_solve_report* report,
                                         double* w_out);
int cphifi_unaligned_assemble_sym_dense(cphifi_unaligned p, int64_t dense_cap, double* sys_out, double* rhs_out);

/* Fused aligned update for mode k: MTTKRP + Gram + decoupled solve, one device pass,
 * eig(V) on device.  b_out / v_out may be NULL. */
int cphifi_aligned_solve(cphifi_tensor t, cphifi_mode mode, int k, int64_t r,
                         const double* const* factors, double* w_out, double* b_out,
                         double* v_out);

/* ---- observation files ------------------------------------------------
 * Text: the reference format (io.hpp:93-131): `shape: n1 .. nd`, then lines `i1 .. id value`,
 * 1-based, parsed on all host threads.  Binary: the same header line, `cphifi-obs-binary 1 q <q>`,
 * then d int32 index columns (0-based, SoA) and q fp64 values — what cphifi_obs_create takes.
 * cphifi_obs_file_info detects the format (*binary) and returns d, shape[0..d) (d <= 8) and q;
 * cphifi_obs_file_read fills idx_soa (d x q) and values (q).  Errors reuse io.hpp's messages. */
int cphifi_obs_file_info(const char* path, int* d, int64_t* shape, int64_t* q, int* binary);
int cphifi_obs_file_read(const char* path, int d, int64_t q, int32_t* idx_soa, double* values);
int cphifi_obs_file_write(const char* path, int binary, int d, const int64_t* shape, int64_t q,
                          const int32_t* idx_soa, const double* values);

/* ---- ALS infinite-mode update ----------------------------------------
 * AlsState::update_infinite_mode (als.hpp:170-218) followed by AlsState::relative_error
 * (als.hpp:221-237) and this mode's objective term (als.hpp:243-255), one device pass:
 *   W = the subproblem solve, A_k = K W (the factor update, als.hpp:214),
 *   relative_error of the model with A_k in place, lambda * trace(W' K W).
 * Unaligned: PCG (warm_start as solve_unaligned_pcg; the reference passes the previous W), the
 * fit over the observed entries (plans with coalesced duplicates are rejected: their values are
 * sums).  Aligned: MTTKRP + Gram + eig(V) + decoupled solve; `residual` = aligned_residual
 * (aligned.hpp:104-108); the fit uses ||T - M||^2 = ||T||^2 - 2 <A_k, B> + 1'(A_k'A_k o V)1
 * (no N-sized reconstruction; absolute error of the squared fit ~1e-15 ||T||^2). */
typedef struct cphifi_als_report {
    double relative_error; /* ||data - model|| / ||data|| after the update */
    double data_norm;      /* ||data|| (observed entries, or the whole tensor) */
    double reg;            /* lambda * trace(W' K W) */
    double residual;       /* aligned: aligned_residual(p, W); unaligned: PCG relative residual */
    double solve_s;        /* device time of the solve (incl. MTTKRP / RHS) */
    double update_s;       /* device time of A_k = K W and the error terms */
} cphifi_als_report;
int cphifi_als_update_infinite_unaligned(cphifi_unaligned p, const cphifi_pcg_config* cfg,
                                         const double* warm_start, double* w_out, double* a_out,
                                         cphifi_solve_report* solve_report, cphifi_als_report* als);
int cphifi_als_update_infinite_aligned(cphifi_tensor t, cphifi_mode mode, int k, int64_t r,
                                       const double* const* factors, double* w_out, double* a_out,
                                       cphifi_als_report* als);

/* relative_error (als.hpp:221-237) of the model with factor k = a_k (host n_k x r column-major)
 * and the plan's other factors, over the observed entries; *data_norm (may be NULL) = ||v||. */
int cphifi_unaligned_relative_error(cphifi_unaligned p, const double* a_k, double* rel_error,
                                    double* data_norm);
/* update_finite_mode, unaligned branch (als.hpp:144-162): every row i of the
 * plan's mode k gets the minimum-norm least-squares fit of its observations,
 * a_i = argmin ||Z_i a - t_i||, rows without observations stay zero; a_out is n_k x r column-major.
 * `p` comes from cphifi_unaligned_create on the mode-k plan with mode = NULL (a finite-mode
 * subproblem: B, V and the row Grams, no operator).  Solved as G_i^+ (Z_i' t_i) with
 * G_i = Z_i' Z_i, eigenvalues below r eps lambda_max dropped (COD's rank decision on Z_i agrees
 * while cond(Z_i) < ~1e7). */
int cphifi_als_update_finite_unaligned(cphifi_unaligned p, double* a_out);

/* update_finite_mode, aligned branch (als.hpp:139-143): A_k = B_k V_k^+ with B_k = mttkrp(T, model, k)
 * and V_k = gram_khatri_rao(model, k), the pseudo-inverse on V_k's eigenbasis (eigenvalues below
 * r eps sigma_max dropped, COD's rank decision).  Modes k > 0 need a 3-way, unsharded tensor with
 * even n0 and r <= 64.  a_out: n_k x r column-major; rel_error_out (may be NULL): the relative
 * error of the model after the update (||T||^2 - 2<A_k, B_k> + 1'(A_k'A_k o V_k)1). */
int cphifi_als_update_finite_aligned(cphifi_tensor t, int k, int64_t r, const double* const* factors,
                                     double* a_out, double* rel_error_out);

/* Benchmark hook: `iters` aligned solves on the device-resident tensor with CUDA events per
 * phase; ms_out[0..4] = mean ms of [0] MTTKRP, [1] Gram V, [2] eig(V) (setup: wall clock of the
 * warm-up pass; the timed passes reuse it), [3] decoupled rotate/divide/rotate (each phase of a
 * synchronised pass, so it carries its kernels' launch latency), [4] timed solve: the sequence
 * [0], [1], [3] captured as one CUDA graph and replayed `iters` times back to back (one GPU;
 * with a communicator, [0] + [1] + [3]). */
int cphifi_aligned_solve_timed(cphifi_tensor t, cphifi_mode mode, int k, int64_t r,
                               const double* const* factors, int iters, double* w_out,
                               double* ms_out);

/* ---- device-side test / bench inputs (no solver work) ------------------------------ */
/* Device-side seeded observations (configs 3-4 scale; not the solver path).  q draws; mode m
 * uniform on [0, shape[m]) except mode zipf_mode (>= 0) with P(i) ~ (i+1)^-zipf_s; value =
 * sum_j prod_m A_m(i_m, j) + noise_std * N(0,1) with factors[m] host n_m x r column-major.
 * Counter-based (splitmix64 of seed, observation, stream; inputs/synth_math.h), bit-identical to
 * the host generator inputs/synth_host.cpp.  idx_out (d x q int32) and vals_out (q fp64) are
 * DEVICE buffers on the context's GPU. */
int cphifi_synth_observations(cphifi_ctx ctx, int d, const int64_t* shape, int64_t q, uint64_t seed,
                              int zipf_mode, double zipf_s, int64_t r, const double* const* factors,
                              double noise_std, int32_t* idx_out, double* vals_out);

#ifdef __cplusplus
}
#endif
#endif /* CPHIFI_B200_H */
