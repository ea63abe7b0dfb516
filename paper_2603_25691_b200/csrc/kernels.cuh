// kernels.cuh — launch wrappers for the sm_100a kernels (internal).
#pragma once
#include "common.cuh"

namespace cphifi {

// ---- dense FP64 tensor-core (DMMA) GEMM: C = op(A) * B with fused epilogues ------------
// Element (i,k) of A is a[i*a_rs + k*a_cs]; (k,j) of B is b[k*b_rs + j*b_cs].  Output
// (i,j) goes to c[i*c_rs + j*c_cs] (optional) and to the row-major padded copy c2[i*ld2+j]
// (optional; columns j in [n, ld2) are written as 0).
enum EpiOp : int {
    EPI_STORE = 0,    // C = AB
    EPI_AXPY2 = 1,    // C = (AB + beta1*E1) + beta2*E2     (unaligned.hpp:112-114 order)
    EPI_HADAMARD = 2, // C = AB .* E1                        (unaligned.hpp:137)
    EPI_SCALE_DIV = 3, // C = AB / (e_row[i]*e_col[j] + beta1) with zero-denominator flag
    EPI_ROWSCALE = 4,  // C = e_row[i] * (AB + beta1*E1) + beta2*E1   (E1 may be null: 0)
    EPI_GRAM = 5,      // Yhat(i,:) = G_i (AB)(i,:) for rows with observations (row-Gram operator;
                       // tensor-map GEMM path only: the split-K reduction and the apply in one kernel)
    EPI_PARTIALS = 6   // no reduction: *parts_out = the P split-K partials (P x m x n, column-major
                       // each), *p_out = P, for a consumer that reduces them itself (tensor-map path)
};

struct GemmArgs {
    int64_t m = 0, n = 0, k = 0;
    const double* a = nullptr; int64_t a_rs = 1, a_cs = 0;
    const double* b = nullptr; int64_t b_rs = 1, b_cs = 0;
    double* c = nullptr; int64_t c_rs = 1, c_cs = 0;
    double* c2 = nullptr; int64_t ld2 = 0;
    int epi = EPI_STORE;
    const double* e1 = nullptr; const double* e2 = nullptr; int64_t ld_e = 0;  // col-major
    double beta1 = 0.0, beta2 = 0.0;
    const double* e_row = nullptr; const double* e_col = nullptr;
    int* flag = nullptr;  // set to 1 if EPI_SCALE_DIV meets a zero denominator
    // EPI_GRAM: n x rp x rp row Grams, CSR row pointers, Yhat (n x rp row-major) out; rp >= n cols
    const double* gram = nullptr;
    const int64_t* row_ptr = nullptr;
    int64_t rp = 0;
    double* yhat = nullptr;
    const double** parts_out = nullptr;  // EPI_PARTIALS
    int* p_out = nullptr;
};
void gemm(const GemmArgs& g, int num_sms, cudaStream_t s);
bool gemm_tma_ok(const GemmArgs& g);
int gemm_splitk_depth(const GemmArgs& g, int num_sms);  // split-K partials of the tensor-map path

// ---- dense MTTKRP for mode 0 (tensor.hpp:174-182): B = T_(1) * Z with Z generated on the
// fly from the factors (khatri_rao order, last listed factor fastest).  T is the local
// slab n0 x (n1 range) x n2 x ...; factors are column-major originals.  Deterministic
// split over the column range with an ordered reduction.
struct MttkrpArgs {
    int d = 0;
    int64_t shape[8] = {0};   // local slab shape (shape[1] = slab extent)
    int64_t off1 = 0;         // global offset of the slab in mode 1
    int64_t r = 0;
    const double* t = nullptr;
    const double* fac[8] = {nullptr};  // device column-major, fac[m] has ld = full n_m
    int64_t ld[8] = {0};
    double* b = nullptr;      // n0 x r column-major output
    int64_t ldw = 0;          // row stride of the Khatri-Rao outer rows Wout (r rounded up to even: 16-byte rows)
    int probe = 0;            // profiling only (CPHIFI_MTTKRP_PROBE, v3): 1 = stream T without the DMMA work,
                              // 2 = DMMA work on stale stages without the stream, 3 = as 2 without the B scaling
    int l2_ahead = 0;         // v3: tiles of T prefetched into L2 ahead of the ring (CPHIFI_MTTKRP_L2AHEAD)
};
void mttkrp_mode0(const MttkrpArgs& a, int num_sms, cudaStream_t s, DevBuf<double>& work);
// MTTKRP for mode k in {1, 2} of a 3-way column-major tensor (even n0): B_k = T_(k) (A_other (x) A_0)
bool mttkrp_k3_supported(int d, const int64_t* shape, int k, int64_t r);
void mttkrp_mode_k3(const double* t, const int64_t* shape, int k, int64_t r, const double* a0, int64_t ld0,
                    const double* aoth, int64_t ldo, double* b_out, int num_sms, cudaStream_t s, DevBuf<double>& work);

// FP64 peak probes (DFMA / DMMA loops, TFLOP/s) for the roofline denominators
void fp64_peaks(int num_sms, cudaStream_t s, double* dfma_tflops, double* dmma_tflops);

// ---- Khatri-Rao Gram (tensor.hpp:186-194), factors column-major device ----------------
void gram_kr(int d, const int64_t* shape, int64_t r, const double* const* fac, int k, double* v,
             cudaStream_t s);

// ---- small kernels ---------------------------------------------------------------------
void kernel_matrix(int kind, const double* pts, int64_t n, double param, double* kmat, cudaStream_t s);
void clamp_nonneg(double* v, int64_t n, cudaStream_t s);
void max_asym(const double* a, int64_t n, double* out2, cudaStream_t s);  // out2 = {max|a-a'|, max|a|}
void precond_diag(const double* mu, const double* sv, int64_t n, int64_t r, double gamma,
                  double lambda, double rho, double* dmat, int* flag, cudaStream_t s);
void pack_rows(const double* src_cm, int64_t rows, int64_t ld, int64_t r, int64_t rp, double* dst_rm,
               cudaStream_t s);
void rm_to_cm(const double* src_rm, int64_t rows, int64_t rp, int64_t r, double* dst_cm, cudaStream_t s);

// ---- eigenbasis sandwich Y = U ((U' X U_V) op E) U_V' (k_sandwich.cu): two row-local launches
enum : int { SW_MUL = 0, SW_DIV = 1 };
struct SandArgs {
    int64_t n = 0, r = 0, rp = 0;       // rp set by sandwich()
    const double* u = nullptr;          // n x n column-major
    const double* ut = nullptr;         // U' (n x n column-major)
    const double* x = nullptr;          // n x r, column stride ldx
    int64_t ldx = 0;
    const double* uv = nullptr;         // r x r column-major
    int op = SW_MUL;
    const double* dmat = nullptr;       // SW_MUL: n x r column-major
    const double* e_row = nullptr;      // SW_DIV: den = e_col[j] * e_row[i] + beta
    const double* e_col = nullptr;
    double beta = 0.0;
    int* flag = nullptr;                // SW_DIV: set to 1 on a zero denominator
    double* core_out = nullptr;         // sandwich_scratch_doubles(n, r) scratch (phase 1 output)
    const double* core = nullptr;       // the same buffer (phase 2 input)
    double* y = nullptr;                // n x r, column stride ldy
    int64_t ldy = 0;
};
bool sandwich_supported(int64_t n, int64_t r);
int64_t sandwich_rp(int64_t r);
int64_t sandwich_scratch_doubles(int64_t n, int64_t r);  // core_out size the sandwich needs
// offset (doubles) of the split-K row-block counters in that scratch: zero them when it is allocated
int64_t sandwich_counter_offset(int64_t n, int64_t r);
void sandwich(SandArgs a, int num_sms, cudaStream_t s);
void transpose_sq(const double* a, int64_t n, double* at, cudaStream_t s);
// eigenbasis preconditioner z~ = ((r~ U_V) o D) U_V' in one launch (r <= 64)
void precond_rot_small(const double* rt, const double* uv, const double* dmat, int64_t n, int64_t r, double* zt,
                       cudaStream_t s);
// sigma -> pseudo-inverse spectrum (1 / sigma above r eps sigma_max, else 0), in place
void invert_spectrum(double* sv, int64_t r, cudaStream_t s);
// a (m x r column-major) <- a diag(d)
void scale_columns(double* a, int64_t m, int64_t r, const double* d, cudaStream_t s);
// out = diag(d) a  (n x n column-major)
void scale_rows(const double* a, int64_t n, const double* d, double* out, cudaStream_t s);
// out = a diag(d)  (n x n column-major)
void scale_cols(const double* a, int64_t n, const double* d, double* out, cudaStream_t s);

// ---- the unaligned operator as one persistent cooperative kernel (k_fused.cu) -----------
// PH_A: Xhat rows distributed + barrier; PH_AL: each CTA computes only the Xhat rows its own
// observations touch (no barrier); PH_B: scatter-gather (Yhat complete in global memory at the
// end of the phase: split rows are finished by their last CTA); PH_C2: y rows (after a grid
// barrier when PH_B ran in the same launch).
enum : unsigned { PH_A = 1u, PH_B = 2u, PH_C2 = 8u, PH_AL = 16u };
struct FusedArgs {
    int64_t n = 0, r = 0, rp = 0, q = 0;  // q: column stride of idx (multiple of 4)
    int dother = 0;
    unsigned phases = 0;
    const int64_t* row_ptr = nullptr;   // local CSR over sorted i_k (n + 1)
    const int32_t* idx = nullptr;       // dother columns of stride q, other modes ascending
    const double* fac = nullptr;        // packed row-major rp-padded factors
    int64_t fac_off[8] = {0};
    int64_t fac_total = 0;              // doubles in fac
    const double* weights = nullptr;    // non-null: s_l = weights[l] (RHS B), else Xhat . z_l
    const int32_t* mult = nullptr;      // coalesced plan: operator weight of entry l (dot mode)
    int accumulate = 0;                 // k_stream.cu: add into yhat_rm instead of overwriting (stream parts > 0)
    const double* kmat = nullptr;       // n x n column-major, symmetric
    const double* x = nullptr;          // n x r column-major
    double* y = nullptr;                // n x r column-major
    double* xhat_rm = nullptr;          // n x rp
    double* yhat_rm = nullptr;          // n x rp
    double* slot_a = nullptr;           // C x rp
    double* slot_b = nullptr;
    // row-aligned CTA partition (host plan, see plan_partition in capi.cu)
    const int64_t* cta_beg = nullptr;   // C + 1: CTA c streams observations [cta_beg[c], cta_beg[c+1])
    const int64_t* cta_rows = nullptr;  // 2 x C: first / last row of each CTA's range
    const int32_t* row_first_cta = nullptr;  // n: first CTA touching the row
    const int32_t* row_ncta = nullptr;       // n: CTAs touching the row (> 1 = split row)
    double lambda = 0.0, rho = 0.0;
    const double* yhat_c2 = nullptr;    // complete Yhat read by PH_C2 (yhat_rm or the NCCL sum)
    const double* gram = nullptr;       // non-null: phase B applies the row-Gram operator instead
    // eigenbasis PCG (k_fused PH_C2): y~ rows = mu_i (U(:,i)' Yhat + lambda x~_i) + rho x~_i with the
    // columns of kmat_c2 (= U); kmat then holds diag(mu) U' so PH_AL/PH_A produce Xhat = U diag(mu) x~
    const double* kmat_c2 = nullptr;    // null: kmat
    const double* mu_rot = nullptr;     // non-null: the eigenbasis epilogue
    unsigned* rowcnt = nullptr;         // n per-row arrival counters, zero-initialised once
    int prefetch = 0;                   // stage X and the needed K columns in smem (small n)
    unsigned* barrier = nullptr;        // barrier_words(grid) uints, zero-initialised once
    int bar_groups = 16;                // CTAs per first-level barrier counter
    unsigned long long* trace = nullptr;  // optional: TRACE_SLOTS %globaltimer stamps per CTA
    long long* dbg = nullptr;             // optional: DBG_SLOTS (event, clock64) pairs per CTA
};
constexpr int DBG_SLOTS = 64;
constexpr int TRACE_SLOTS = 8;  // entry, A done, barrier 1, B done, barrier 2, C1 done, barrier 3, end
inline size_t barrier_words(int grid, int group) { return 64 + 32 * (size_t)((grid + group - 1) / group); }
// column stride of X staged in the fused kernel's shared memory: odd (conflict-free row dots)
// for odd n; n + 2 for even n so every column is a 16-byte aligned bulk copy
__host__ __device__ inline int64_t fused_ldx(int64_t n) { return (n & 1) ? n : n + 2; }
size_t fused_smem_bytes(int64_t rp, int dother, int64_t fac_total, bool smemf, int64_t prefetch_elems);
int fused_maxloc();
int fused_grid(int64_t rp, int dother, bool smemf, size_t smem, int num_sms);
void fused_matvec(const FusedArgs& a, int grid, size_t smem, bool smemf, cudaStream_t s);

// ---- large-plan scatter-gather (k_stream.cu): phase B as a streaming kernel with the first
// other mode hoisted per run (needs >= 2 other modes and the lexicographic plan order); a normal
// launch, one CTA per SM, TMA bulk-copied observation tiles, per-observation factors in shared
// memory when `sf`.
bool stream_supported(int64_t rp, int dother);
size_t stream_smem_bytes(int64_t rp, int dother, int64_t sf_doubles, int aux_bytes);
size_t stream_smem_cap();
// sf_doubles > 0: that many doubles of per-observation factors are staged in shared memory
void stream_scatter_gather(const FusedArgs& a, int grid, int64_t sf_doubles, cudaStream_t s);

// ---- the operator's q-pass as a run-structured streaming kernel (k_runs.cu) ---------------
// Per-observation factors staged in shared memory (a factor-block part of the plan when they do
// not fit), per-warp equal-count entry ranges, a precomputed run table (runs of equal first other
// index within a row), per-warp TMA rings of plan chunks.  Operator mode only (s_l = Xhat . z_l).
struct RunsArgs {
    int64_t rp = 0, ldq = 0;             // padded rank; column stride of idx (multiple of 4)
    int dother = 0;
    const int32_t* idx = nullptr;        // dother columns (other modes ascending), plan order
    const int32_t* mult = nullptr;       // coalesced plan: multiplicities, else null
    const double* fac = nullptr;         // packed row-major rp-padded factors
    int64_t fac_off[8] = {0};
    int64_t fac_total = 0;
    const int64_t* row_ptr = nullptr;    // n + 1
    const int32_t* run_start = nullptr;  // nruns + 1 (last = q)
    const int32_t* run_i1 = nullptr;     // nruns: first other index of each run
    int64_t nruns = 0;
    int warps = 0;                       // warp ranges
    const int64_t* warp_beg = nullptr;   // warps + 1
    const int64_t* warp_rows = nullptr;  // 2 x warps: first / last row
    const int32_t* row_first_w = nullptr;  // n: first warp touching the row
    const int32_t* row_nw = nullptr;       // n: warps touching the row (> 1 = split row)
    const double* xhat_rm = nullptr;     // n x rp
    double* yhat_rm = nullptr;           // n x rp
    double* slot_a = nullptr;            // warps x rp (a warp's first row when shared)
    double* slot_b = nullptr;            // warps x rp (its last row when shared)
    unsigned* rowcnt = nullptr;          // n arrival counters, zero between launches
    int accumulate = 0;                  // add into yhat_rm (stream parts) instead of overwriting
    const double* vals = nullptr;        // non-null: the right-hand side B (weights = the entries' values,
                                         // no dot with Xhat) instead of the operator's q-pass
};
// Dense rows of a 3-way plan (k_dense_rows.cu): the q-pass of rows whose cells are mostly drawn as
// two DMMA GEMMs per row over the row's multiplicity grid W_i (n1p x n2p int32, zero-padded).
struct DenseRowsArgs {
    int64_t rp = 0;
    int64_t n1 = 0, n2 = 0;              // other-mode sizes (A_1 rows, A_2 rows)
    int64_t n1p = 0, n2p = 0;            // padded to the kernel's blocks (dense_rows_block_a / _b)
    int nd = 0;                          // dense rows
    const int32_t* rows = nullptr;       // nd: their row indices i_k
    const int32_t* w = nullptr;          // nd x n1p x n2p multiplicities
    const double* a1 = nullptr;          // n1 x rp row-major
    const double* a2 = nullptr;          // n2 x rp row-major
    const double* xhat_rm = nullptr;     // n x rp
    double* yhat_rm = nullptr;           // n x rp: the dense rows are written (overwritten)
    double* partial = nullptr;           // nd x (n1p / block_a) x rp scratch
    unsigned* cnt = nullptr;             // nd arrival counters, zero between launches
};
int dense_rows_block_a();
int dense_rows_block_b();
bool dense_rows_supported(int64_t rp, int dother);
void dense_rows_qpass(const DenseRowsArgs& a, int num_sms, cudaStream_t s);
// W(slot[rows[l]], idx0[l], idx1[l]) += mult[l] (1 without multiplicities) for the entries of dense rows
void dense_grid_build(const int32_t* idx, int64_t ldq, const int32_t* mult, const int32_t* rows, const int32_t* slot,
                      int64_t q, int64_t n1p, int64_t n2p, int32_t* w, cudaStream_t s);
// *out += sum of v[0, q) (nonnegative int32; integer atomics: exact)
void sum_i32(const int32_t* v, int64_t q, unsigned long long* out, cudaStream_t s);
// key[l] += dense_key_value for the entries of dense rows (slot[rows[l]] >= 0)
void dense_key(const int32_t* rows, const int32_t* slot, int64_t q, int32_t dense_key_value, int32_t* key,
               cudaStream_t s);
bool runs_supported(int64_t rp, int dother);
size_t runs_smem_bytes(int64_t rp, int dother, bool mult, int64_t sf_doubles);
// k_xruns.cu: the q-pass of 3-way coalesced parts with steps across run boundaries.  The part's runs
// are padded to even lengths (a zero-multiplicity copy of an odd run's last entry) and run starts are
// flagged in bit 30 of the multiplicity: readers of a padded part's multiplicities mask it off.
constexpr int32_t RUN_MULT_MASK = (1 << 30) - 1;
bool xruns_supported(int64_t rp, int dother, bool mult);
size_t xruns_smem_bytes(int64_t rp, int64_t sf_doubles);
int xruns_warps_per_sm();
void xruns_scatter_gather(const RunsArgs& a, int64_t sf_doubles, cudaStream_t s);
// pads the runs [run_start[r], run_start[r+1]) of a part (columns ia / ib, multiplicities, rows) into
// oa / ob / om / orow (room for q + nr entries); returns the padded entry count
int64_t pad_runs_even(const int32_t* run_start, int64_t nr, const int32_t* ia, const int32_t* ib, const int32_t* mult,
                      const int32_t* rows, int32_t* oa, int32_t* ob, int32_t* om, int32_t* orow, int64_t q,
                      cudaStream_t s);
size_t runs_smem_cap();
int runs_warps_per_sm(int64_t rp);
int runs_chunk(int64_t rp);
void runs_scatter_gather(const RunsArgs& a, int64_t sf_doubles, cudaStream_t s);
// run table of a plan: run_start[j] = first entry of run j (entry l starts a run when it starts a
// row or its first other index differs from entry l-1's); returns the number of runs (synchronous)
int64_t build_run_starts(const int32_t* rows, const int32_t* col0, int64_t q, int32_t* run_start, cudaStream_t s);

// ---- row-Gram operator (k_gram.cu): Yhat(i,:) = G_i Xhat(i,:), G_i = sum_l z_l z_l' ---------
struct GramArgs {
    int64_t n = 0, rp = 0, q = 0;
    int dother = 0;
    const int64_t* row_ptr = nullptr;
    const int32_t* idx = nullptr;
    const double* fac = nullptr;
    int64_t fac_off[8] = {0};
    int64_t fac_total = 0;          // doubles in fac (shared-memory staging of the DMMA build)
    const int32_t* mult = nullptr;  // coalesced plan: G_i = sum_l mult_l z_l z_l'
    const int64_t* cta_beg = nullptr;
    const int64_t* cta_rows = nullptr;
    const int32_t* row_first_cta = nullptr;
    const int32_t* row_ncta = nullptr;
    unsigned* rowcnt = nullptr;
    double* slot_a = nullptr;  // grid x rp x rp
    double* slot_b = nullptr;
    double* g = nullptr;       // n x rp x rp
    int accumulate = 0;        // k_gramws.cu: add into g (factor-block parts) instead of overwriting
};
void gram_build(const GramArgs& a, int grid, cudaStream_t s);
// warp-specialised build (k_gramws.cu): producer warps build z batches from factors staged in shared
// memory (sf doubles: modes 1.. of the plan / of a factor-block part), consumer warps run the DMMA
bool gram_ws_supported(int64_t rp, int dother);
size_t gram_ws_smem_bytes(int64_t rp, int64_t sf);
void gram_build_ws(const GramArgs& a, int grid, int64_t sf, cudaStream_t s);
int gram_build_occupancy(const GramArgs& a);
// register-fragment build (k_gram3.cu): units = contiguous entry ranges of an equal-count partition
// (cta_beg / cta_rows / row_first_cta / row_ncta over `units`), gram3_units_per_sm(rp) per SM
// 2: every factor staged in shared memory, 1: modes 1.. staged (a factor-block part), 0: not applicable
int gram3_stage(int64_t rp, int dother, const GramArgs& a);
int gram3_units_per_sm(int64_t rp);
void gram3_build(const GramArgs& a, int units, int stage, cudaStream_t s);  // partition CTAs per SM for the build gram_build picks
void gram_apply(const double* g, const double* xhat_rm, const int64_t* row_ptr, int64_t n, int64_t rp, double* yhat_rm,
                cudaStream_t s);

// ---- seeded device-side observation generator (configs 3/4; k_synth.cu) -----------------
void synth_observations(int d, const int64_t* shape, int64_t q, uint64_t seed, int zipf_mode, double zipf_s, int64_t r,
                        const double* const* fac_dev, double noise_std, int32_t* idx, double* vals, int num_sms,
                        cudaStream_t s);

// ---- PCG vector kernels (deterministic reductions) --------------------------------------
struct PcgState {
    double rz, pap, alpha, rr, bnorm, rel, beta, rz_new;
    int flag;  // 1 = non-finite p'Ap, 2 = p'Ap <= 0
    int pad;
};
// Device-resident PCG loop control (the body of a CUDA-graph WHILE node): counts the iteration,
// records rel, and clears the loop condition exactly where solvers.hpp:59-80 leaves the loop
// (non-finite / non-positive p'Ap, rel <= tol, it == max_iter).
struct PcgCtl {
    double tol;
    int max_iter, it;
    double* hist;  // device history (rel after each iteration), hist_cap entries
    int hist_cap, stop;
    int warm, zero_b;  // whole-solve graph: warm start given; ||b|| == 0
    double rel0;       // relative residual of the initial guess
};
void pcg_ctl(const PcgState* st, PcgCtl* c, cudaGraphConditionalHandle h, cudaStream_t s);
// One PCG iteration's vector work after Ap (pap, x/r update, loop control, eigenbasis
// preconditioner, rz, p update) as one cooperative launch: k_pcgstep.cu.  r <= 64.
struct PcgStepArgs {
    int64_t n = 0;
    int r = 0;
    const double* uv = nullptr;    // U_V, r x r column-major
    const double* dmat = nullptr;  // D, n x r column-major
    double *x = nullptr, *res = nullptr, *p = nullptr, *z = nullptr;
    const double* ap = nullptr;
    PcgState* st = nullptr;
    PcgCtl* ctl = nullptr;         // loop control (graph body), or nullptr
    cudaGraphConditionalHandle h{};
    int set_cond = 0;              // 1: inside the graph's WHILE body (clear `h` on stop)
    int64_t null_rows = 0;         // rows i < null_rows of Ap are rho p (not written by the operator)
    double rho = 0.0;
    // non-null: rows i >= null_rows of Ap come as the operator GEMM's split-K partials (EPI_PARTIALS,
    // P x (n - null_rows) x r) and get its EPI_ROWSCALE epilogue here: mu_i (sum + lambda p) + rho p
    const double* ap_parts = nullptr;
    int ap_p = 0;
    const double* mu = nullptr;
    double lambda = 0.0;
    double* partial = nullptr;     // pcg_step_fused_partials(n, num_sms) doubles
    unsigned long long* barrier = nullptr;  // zero-initialised once per plan
};
int pcg_step_fused_partials(int64_t n, int num_sms);
void pcg_step_fused(const PcgStepArgs& a, int num_sms, cudaStream_t s);
// step A followed by the loop control (one launch for n <= 32768)
void pcg_step_a_ctl(double* x, double* r, const double* p, const double* ap, int64_t n, PcgState* st, double* partial,
                    PcgCtl* c, cudaGraphConditionalHandle h, cudaStream_t s);
// whole-solve graph pieces: bnorm = sqrt(bnorm), zero_b
void pcg_prologue(PcgState* st, PcgCtl* c, cudaStream_t s);
// x = 0 unless warm (zero_b: x = 0); res = b unless warm
void pcg_x0(double* x, double* res, const double* b, int64_t n, const PcgCtl* c, cudaStream_t s);
// after pcg_init: rel0; skip the WHILE body when zero_b or rel <= tol
void pcg_loopctl(const PcgState* st, PcgCtl* c, cudaGraphConditionalHandle hwhile, cudaStream_t s);
void dot_to(const double* x, const double* y, int64_t n, double* partial, double* out, cudaStream_t s);
// pap = p.ap; flag; alpha = rz/pap; x += alpha p; r -= alpha ap; rr = r.r; rel = sqrt(rr)/bnorm
void pcg_step_a(double* x, double* r, const double* p, const double* ap, int64_t n, PcgState* st,
                double* partial, cudaStream_t s);
// rz_new = r.z; beta = rz_new/rz; p = z + beta p; rz = rz_new
void pcg_step_b(const double* r, const double* z, double* p, int64_t n, PcgState* st, double* partial,
                cudaStream_t s);
// init: rz = r.z, rr = r.r, rel = sqrt(rr)/bnorm, p = z
void pcg_init(const double* r, const double* z, double* p, int64_t n, PcgState* st, double* partial,
              cudaStream_t s);
// dst <- src (n doubles), a kernel copy when 16-byte aligned (mapped host memory allowed)
void copy_doubles(double* dst, const double* src, int64_t n, cudaStream_t s);
// out[i] = sum_{s < nsrc} src[s][i] in rank order (virtual communicator reduction, nsrc <= 8)
void rank_order_sum(const double* const* src, int nsrc, double* out, size_t count, int num_sms, cudaStream_t s);
// ---- aligned baselines (k_aligned.cu) ------------------------------------
void aligned_matvec_dev(const double* x, const double* dk, const double* v, int64_t n, int64_t r, double lambda,
                        double* y, cudaStream_t s);
void aligned_dinv(const double* dk, const double* v, int64_t n, int64_t r, double lambda, double* dinv,
                  cudaStream_t s);
void hadamard(const double* a, const double* b, int64_t cnt, double* out, cudaStream_t s);
// unaligned direct / dense baselines from the row Grams (k_aligned.cu): the nonsymmetric system
// G'F + lambda I; S = G_i''(j,j') K(i'',i') scaled columns (F'F = K S, placed by sym_place with
// lambda (I kron K) + rho I)
void nonsym_system(const double* g, const double* kmat, int64_t n, int64_t r, int64_t rp, double lambda, double* sys,
                   cudaStream_t s);
void gram_scaled(const double* g, const double* kmat, int64_t n, int64_t r, int64_t rp, double* sm, cudaStream_t s);
void sym_place(const double* cm, const double* kmat, int64_t n, int64_t r, double lambda, double rho, double* sys,
               cudaStream_t s);
void kron_system(const double* v, const double* kmat, int64_t n, int64_t r, double lambda, double* sys,
                 cudaStream_t s);

// Grid of the deterministic vector reductions (dot_to / PCG steps); their `partial` scratch needs
// RED_PARTIALS doubles (RED_GRID partials + the ticket word).
constexpr int RED_GRID = 296;
constexpr int RED_PARTIALS = RED_GRID + 8;
void scale_row_block(double* y, const double* x, int64_t z, int64_t n, int64_t r, double alpha, cudaStream_t s);
void axpby(double* y, const double* a, double alpha, const double* b, double beta, int64_t n,
           cudaStream_t s);  // y = alpha*a + beta*b

// ---- ALS error terms (k_als.cu) ----------------------------------------
struct SqResidualArgs {
    int64_t n = 0, r = 0, rp = 0, q = 0, ldq = 0;
    int dother = 0;
    const int64_t* row_ptr = nullptr;  // CSR over i_k (n + 1)
    const int32_t* idx = nullptr;      // dother columns of stride ldq, other modes ascending
    const double* values = nullptr;    // q
    const double* fac = nullptr;       // packed row-major rp-padded other-mode factors
    int64_t fac_off[8] = {0};
    const double* ak = nullptr;        // the updated mode-k factor, n x rp row-major
};
int64_t sq_residual_blocks(int64_t q);
// finite-mode row least squares (k_rowls.cu): a_i = G_i^+ b_i for every row (G: n x rp x rp,
// b / a_out: n x r column-major)
void rowls_solve(const double* g, const double* b, int64_t n, int64_t r, int64_t rp, double* a_out, cudaStream_t s);
// *out = sum_l (v_l - <A_k(i_k(l),:), z_l>)^2 ; partial >= sq_residual_blocks(q) doubles
void sq_residual(const SqResidualArgs& a, double* partial, double* out, cudaStream_t s);
// *out = ||x||^2 with nb blocks (partial >= nb doubles)
void sq_norm(const double* x, int64_t n, double* partial, int64_t nb, double* out, cudaStream_t s);

// ---- observation plan helpers ------------------------------------------------------------
void check_range(const int32_t* idx, int d, int64_t q, const int64_t* shape_dev, int* flag, cudaStream_t s);
void linear_index(const int32_t* idx, int d, int64_t q, const int64_t* shape, uint64_t* lin, cudaStream_t s);
void adjacent_equal(const uint64_t* sorted, int64_t q, int* flag, cudaStream_t s);
void iota32(int32_t* p, int64_t q, cudaStream_t s);
void gather_i32(const int32_t* src, const int32_t* perm, int64_t lo, int64_t cnt, int32_t* dst, cudaStream_t s);
void gather_f64(const double* src, const int32_t* perm, int64_t lo, int64_t cnt, double* dst, cudaStream_t s);
void csr_from_sorted(const int32_t* keys, int64_t q, int64_t n, int64_t* row_ptr, cudaStream_t s);
// stream parts (capi.cu build_stream_parts): key[l] = col[l] / rows; rows[l] = the CSR row of entry l;
// p[l] += delta
void block_key(const int32_t* col, int64_t q, int32_t rows, int32_t* key, cudaStream_t s);
void row_of_entries(const int64_t* row_ptr, int64_t n, int64_t q, int32_t* rows, cudaStream_t s);
void add_i32(int32_t* p, int64_t cnt, int32_t delta, cudaStream_t s);
size_t radix_sort_pairs_bytes(int64_t q, int bits);
void radix_sort_pairs(void* temp, size_t temp_bytes, const int32_t* keys_in, int32_t* keys_out,
                      const int32_t* vals_in, int32_t* vals_out, int64_t q, int bits, cudaStream_t s);
void csr_from_sorted64(const uint64_t* keys, int64_t q, int64_t n, uint64_t span, int64_t* row_ptr, cudaStream_t s);
// cnt[i] = distinct keys of row i (sorted lexicographic keys, row = key / span), i < n
void row_distinct_counts(const uint64_t* keys, int64_t q, int64_t n, uint64_t span, unsigned long long* cnt,
                         cudaStream_t s);
// b(i,:) = yhat(i,:) (+ lambda x(i,:) on the owned rows) for rows [lo, hi): the row-sharded output GEMM's operand
void shard_operand(const double* yhat, const double* x, int64_t n, int64_t r, int64_t rp, int64_t lo, int64_t hi,
                   int64_t own_lo, int64_t own_hi, double lambda, double* b, cudaStream_t s);
size_t radix_sort_pairs64_bytes(int64_t q, int bits);
void radix_sort_pairs64(void* temp, size_t temp_bytes, const uint64_t* keys_in, uint64_t* keys_out,
                        const int32_t* vals_in, int32_t* vals_out, int64_t q, int bits, cudaStream_t s);
// sorted keys -> distinct keys, run lengths and per-run value sums; returns the run count
int64_t coalesce_sorted(const uint64_t* keys, const double* vals, int64_t q, uint64_t* ukeys, int32_t* counts,
                        double* vsum, cudaStream_t s);
// distinct lexicographic keys -> other-mode indices ((d-1) columns of stride ldq, modes ascending)
void decode_keys(const uint64_t* keys, int64_t nu, int d, int k, const int64_t* stride_dev, const int64_t* shape_dev,
                 int32_t* idx_o, int64_t ldq, cudaStream_t s);
size_t radix_sort_keys64_bytes(int64_t q);
void radix_sort_keys64(void* temp, size_t temp_bytes, const uint64_t* in, uint64_t* out, int64_t q,
                       cudaStream_t s);

}  // namespace cphifi
