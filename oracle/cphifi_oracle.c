/*
 * cphifi_oracle.c — CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference CP-HIFI hot path, used ONLY by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs as the
 * checker and as the timed CPU baseline.  Nothing in the product path
 * (paper_2603_25691_b200/) links, loads or calls this file.
 *
 * The reference itself (header-only C++ over Eigen 3) cannot be built here: Eigen,
 * GoogleTest and CLI11 are absent and there is no network.  Each function
 * below cites the reference `file:line` (relative to proj/include/cphifi/) it restates and
 * keeps the reference's operation order where it affects rounding (factor order in Zhat,
 * storage-order streaming in the scatter, left-to-right GEMM association).
 *
 * Pinning: tests/test_oracle_*.py check these functions against every known-answer and
 * dense-oracle test the reference holds for this path (SURVEY.md §8c list) plus the
 * libstdc++ golden vectors in tests/golden/.  Eigenvectors come from LAPACK (numpy) in the
 * Python wrapper and are SHARED with the device path.
 *
 * All matrices are column-major fp64; indices int32 SoA (idx[m*q + l]) like the device
 * input format; sizes int64.  Functions return 0 on success, 1 for the reference's
 * std::invalid_argument, 2 for std::runtime_error, with orc_last_error() holding text.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static __thread char g_err[256];
const char* orc_last_error(void) { return g_err; }
static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
void orc_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

/* ------------------------------------------------------------------------------------
 * Dense GEMM, C = alpha * op(A) * op(B) + beta * C, column-major.  Summation over the
 * inner index runs in ascending order for every output element.  `threads` > 1 splits
 * output rows across OpenMP threads (bit-identical to the serial result).
 * ---------------------------------------------------------------------------------- */
void orc_gemm(int ta, int tb, int64_t m, int64_t n, int64_t kk, double alpha, const double* a,
              int64_t lda, const double* b, int64_t ldb, double beta, double* c, int64_t ldc,
              int threads) {
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1) if (threads > 1)
    for (int64_t i0 = 0; i0 < m; i0 += 64) {
        const int64_t i1 = i0 + 64 < m ? i0 + 64 : m;
        double acc[64];
        for (int64_t j = 0; j < n; ++j) {
            for (int64_t i = i0; i < i1; ++i) acc[i - i0] = 0.0;
            for (int64_t p = 0; p < kk; ++p) {
                const double bv = tb ? b[j + ldb * p] : b[p + ldb * j];
                if (ta) {
                    for (int64_t i = i0; i < i1; ++i) acc[i - i0] += a[p + lda * i] * bv;
                } else {
                    const double* ac = a + lda * p;
                    for (int64_t i = i0; i < i1; ++i) acc[i - i0] += ac[i] * bv;
                }
            }
            for (int64_t i = i0; i < i1; ++i) {
                double* cij = c + i + ldc * j;
                *cij = (beta == 0.0 ? 0.0 : beta * *cij) + alpha * acc[i - i0];
            }
        }
    }
}

/* ---- kernel.hpp:17-30 gaussian_kernel --------------------------------------------- */
int orc_gaussian_kernel(const double* pts, int64_t n, double sigma, double* k) {
    if (sigma <= 0.0) return fail(1, "gaussian_kernel: sigma must be positive");
    const double inv = 1.0 / (2.0 * sigma * sigma);
    for (int64_t i = 0; i < n; ++i) {
        k[i + n * i] = 1.0;
        for (int64_t j = 0; j < i; ++j) {
            const double d = pts[i] - pts[j];
            const double v = exp(-d * d * inv);
            k[i + n * j] = v;
            k[j + n * i] = v;
        }
    }
    return 0;
}

/* Matern-3/2 — absent from the reference; both sides consume one K. */
int orc_matern32_kernel(const double* pts, int64_t n, double ell, double* k) {
    if (ell <= 0.0) return fail(1, "matern32_kernel: lengthscale must be positive");
    const double s3 = sqrt(3.0) / ell;
    for (int64_t i = 0; i < n; ++i) {
        k[i + n * i] = 1.0;
        for (int64_t j = 0; j < i; ++j) {
            const double a = s3 * fabs(pts[i] - pts[j]);
            const double v = (1.0 + a) * exp(-a);
            k[i + n * j] = v;
            k[j + n * i] = v;
        }
    }
    return 0;
}

/* ---- observations.hpp:142-158 build_zhat ------------------------------------------
 * zhat(l,:) = prod_{i != k} A_i(idx_i(l), :), multiplied in ascending mode order starting
 * from ones (:150-156).  zhat is q x r column-major. */
int orc_build_zhat(int d, const int64_t* shape, int k, int64_t q, const int32_t* idx, int64_t r,
                   const double* const* factors, double* zhat) {
    (void)shape;
    for (int64_t t = 0; t < q * r; ++t) zhat[t] = 1.0;
    for (int i = 0; i < d; ++i) {
        if (i == k) continue;
        const double* a = factors[i];
        const int64_t ni = shape[i];
        const int32_t* ix = idx + (int64_t)i * q;
        for (int64_t l = 0; l < q; ++l)
            for (int64_t j = 0; j < r; ++j) zhat[l + q * j] *= a[ix[l] + ni * j];
    }
    return 0;
}

/* ---- observations.hpp:191-198 gather_rows: out[l] = xhat(i_k(l),:) . zhat(l,:) ----- */
void orc_gather_rows(int64_t n, int64_t r, const double* xhat, int64_t q, const double* zhat,
                     const int32_t* idx_k, double* out) {
    for (int64_t l = 0; l < q; ++l) {
        double s = 0.0;
        for (int64_t j = 0; j < r; ++j) s += xhat[idx_k[l] + n * j] * zhat[l + q * j];
        out[l] = s;
    }
}

/* ---- observations.hpp:174-184 sampled_mttkrp: out(i_k(l),:) += w[l] zhat(l,:), l in
 * storage order (:181-182). ---------------------------------------------------------- */
void orc_sampled_mttkrp(int64_t n, int64_t r, int64_t q, const double* zhat,
                        const int32_t* idx_k, const double* w, double* out) {
    memset(out, 0, sizeof(double) * n * r);
    for (int64_t l = 0; l < q; ++l)
        for (int64_t j = 0; j < r; ++j) out[idx_k[l] + n * j] += w[l] * zhat[l + q * j];
}

/* ---- unaligned.hpp:101-115 unaligned_matvec (reference-faithful: materialised Zhat,
 * separate gather and scatter passes, single thread).
 *   xhat = K X; xbar = gather; yhat = scatter(xbar); y = K yhat + lambda xhat; y += rho x
 * work: 2*q doubles + 2*n*r doubles scratch supplied by the caller (NULL -> malloc). */
int orc_unaligned_matvec(int64_t n, int64_t r, const double* kmat, double lambda, double rho,
                         int64_t q, const double* zhat, const int32_t* idx_k, const double* x,
                         double* y, int threads) {
    double* xhat = (double*)malloc(sizeof(double) * n * r);
    double* yhat = (double*)malloc(sizeof(double) * n * r);
    double* xbar = (double*)malloc(sizeof(double) * (q > 0 ? q : 1));
    if (!xhat || !yhat || !xbar) {
        free(xhat); free(yhat); free(xbar);
        return fail(2, "orc_unaligned_matvec: out of memory");
    }
    orc_gemm(0, 0, n, r, n, 1.0, kmat, n, x, n, 0.0, xhat, n, threads);           /* :106 */
    orc_gather_rows(n, r, xhat, q, zhat, idx_k, xbar);                            /* :110 */
    orc_sampled_mttkrp(n, r, q, zhat, idx_k, xbar, yhat);                         /* :111 */
    orc_gemm(0, 0, n, r, n, 1.0, kmat, n, yhat, n, 0.0, y, n, threads);           /* :112 */
    for (int64_t t = 0; t < n * r; ++t) y[t] += lambda * xhat[t];
    for (int64_t t = 0; t < n * r; ++t) y[t] = y[t] + rho * x[t];                 /* :114 */
    free(xhat); free(yhat); free(xbar);
    return 0;
}

/* ---- Streaming variant (SURVEY §8c mode ii): fused per-observation pass without Zhat,
 * OpenMP over a deterministic contiguous partition of observations, per-thread n x r
 * accumulators merged in thread order.  Multiset semantics (duplicates are summed).
 * Computes yhat only (the scatter-gather core); the caller adds the K multiplies. */
/* Row-major copy of a column-major n x r matrix (layout only: the streaming passes below read a
 * factor / Xhat row and update an accumulator row as contiguous memory; no arithmetic changes). */
static double* to_rows(const double* a, int64_t n, int64_t r) {
    double* t = (double*)malloc(sizeof(double) * (n * r > 0 ? n * r : 1));
    if (!t) return NULL;
    for (int64_t j = 0; j < r; ++j)
        for (int64_t i = 0; i < n; ++i) t[i * r + j] = a[i + n * j];
    return t;
}

/* The per-observation pass of orc_scatter_gather_stream on observations [lo, hi): for each l in
 * storage order, z = prod of the other factors' rows (ascending mode, from ones), s = xhat(row,:) .
 * z summed j = 0..r-1, acc(row,:) += s z.  Groups of GRP observations interleave their dots (each
 * dot keeps its own ascending order) and then apply their updates in storage order, so the result
 * is bit-identical to the one-observation-at-a-time loop. */
#define GRP 4
static void stream_pass(int d, int k, int64_t q, const int32_t* idx, int64_t r, double* const* frows,
                        const double* xrows, int64_t lo, int64_t hi, double* acc) {
    const int32_t* ik = idx + (int64_t)k * q;
    double z[GRP][256];
    for (int64_t l0 = lo; l0 < hi; l0 += GRP) {
        const int g = hi - l0 < GRP ? (int)(hi - l0) : GRP;
        double s[GRP];
        for (int b = 0; b < g; ++b) {
            const int64_t l = l0 + b;
            for (int64_t j = 0; j < r; ++j) z[b][j] = 1.0;
            for (int i = 0; i < d; ++i) {
                if (i == k) continue;
                const double* a = frows[i] + (int64_t)idx[(int64_t)i * q + l] * r;
                for (int64_t j = 0; j < r; ++j) z[b][j] *= a[j];
            }
            s[b] = 0.0;
        }
        if (g == GRP) {
            const double* x0 = xrows + (int64_t)ik[l0] * r;
            const double* x1 = xrows + (int64_t)ik[l0 + 1] * r;
            const double* x2 = xrows + (int64_t)ik[l0 + 2] * r;
            const double* x3 = xrows + (int64_t)ik[l0 + 3] * r;
            for (int64_t j = 0; j < r; ++j) {
                s[0] += x0[j] * z[0][j];
                s[1] += x1[j] * z[1][j];
                s[2] += x2[j] * z[2][j];
                s[3] += x3[j] * z[3][j];
            }
        } else {
            for (int b = 0; b < g; ++b) {
                const double* xr = xrows + (int64_t)ik[l0 + b] * r;
                for (int64_t j = 0; j < r; ++j) s[b] += xr[j] * z[b][j];
            }
        }
        for (int b = 0; b < g; ++b) {
            double* ar = acc + (int64_t)ik[l0 + b] * r;
            for (int64_t j = 0; j < r; ++j) ar[j] += s[b] * z[b][j];
        }
    }
}

int orc_scatter_gather_stream(int d, const int64_t* shape, int k, int64_t q, const int32_t* idx,
                              int64_t r, const double* const* factors, int64_t n,
                              const double* xhat, double* yhat, int threads) {
    if (threads < 1) threads = 1;
    if (r > 256) return fail(1, "orc_scatter_gather_stream: rank above 256");
    double* part = (double*)calloc((size_t)threads * n * r, sizeof(double));
    double* frows[16] = {0};
    double* xrows = to_rows(xhat, n, r);
    int oom = !part || !xrows;
    for (int i = 0; i < d && !oom; ++i)
        if (i != k && !(frows[i] = to_rows(factors[i], shape[i], r))) oom = 1;
    if (!oom) {
#pragma omp parallel num_threads(threads)
        {
#ifdef _OPENMP
            const int t = omp_get_thread_num();
            const int nt = omp_get_num_threads();
#else
            const int t = 0, nt = 1;
#endif
            stream_pass(d, k, q, idx, r, frows, xrows, q * t / nt, q * (t + 1) / nt, part + (int64_t)t * n * r);
        }
        /* merge in thread order (accumulators are row-major) */
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = 0; j < r; ++j) {
                double s = 0.0;
                for (int t = 0; t < threads; ++t) s += part[(int64_t)t * n * r + i * r + j];
                yhat[i + n * j] = s;
            }
    }
    for (int i = 0; i < d; ++i) free(frows[i]);
    free(xrows);
    free(part);
    return oom ? fail(2, "orc_scatter_gather_stream: out of memory") : 0;
}

/* Streaming sampled MTTKRP with the observed values (RHS B, unaligned.hpp:44). */
int orc_sampled_mttkrp_stream(int d, const int64_t* shape, int k, int64_t q, const int32_t* idx,
                              const double* values, int64_t r, const double* const* factors,
                              int64_t n, double* b, int threads) {
    if (threads < 1) threads = 1;
    if (r > 256) return fail(1, "orc_sampled_mttkrp_stream: rank above 256");
    double* part = (double*)calloc((size_t)threads * n * r, sizeof(double));
    double* frows[16] = {0};
    int oom = !part;
    for (int i = 0; i < d && !oom; ++i)
        if (i != k && !(frows[i] = to_rows(factors[i], shape[i], r))) oom = 1;
    if (!oom) {
#pragma omp parallel num_threads(threads)
        {
#ifdef _OPENMP
            const int t = omp_get_thread_num();
            const int nt = omp_get_num_threads();
#else
            const int t = 0, nt = 1;
#endif
            const int64_t lo = q * t / nt, hi = q * (t + 1) / nt;
            double* acc = part + (int64_t)t * n * r;
            double z[256];
            const int32_t* ik = idx + (int64_t)k * q;
            for (int64_t l = lo; l < hi; ++l) {
                for (int64_t j = 0; j < r; ++j) z[j] = 1.0;
                for (int i = 0; i < d; ++i) {
                    if (i == k) continue;
                    const double* a = frows[i] + (int64_t)idx[(int64_t)i * q + l] * r;
                    for (int64_t j = 0; j < r; ++j) z[j] *= a[j];
                }
                double* ar = acc + (int64_t)ik[l] * r;
                for (int64_t j = 0; j < r; ++j) ar[j] += values[l] * z[j];
            }
        }
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = 0; j < r; ++j) {
                double s = 0.0;
                for (int t = 0; t < threads; ++t) s += part[(int64_t)t * n * r + i * r + j];
                b[i + n * j] = s;
            }
    }
    for (int i = 0; i < d; ++i) free(frows[i]);
    free(part);
    return oom ? fail(2, "orc_sampled_mttkrp_stream: out of memory") : 0;
}

/* Full streaming matvec (configs 3/4 CPU baseline): xhat = K X; yhat = stream; y = K yhat +
 * lambda xhat + rho x. */
int orc_unaligned_matvec_stream(int d, const int64_t* shape, int k, int64_t q, const int32_t* idx,
                                int64_t r, const double* const* factors, int64_t n,
                                const double* kmat, double lambda, double rho, const double* x,
                                double* y, int threads) {
    double* xhat = (double*)malloc(sizeof(double) * n * r);
    double* yhat = (double*)malloc(sizeof(double) * n * r);
    if (!xhat || !yhat) { free(xhat); free(yhat); return fail(2, "out of memory"); }
    orc_gemm(0, 0, n, r, n, 1.0, kmat, n, x, n, 0.0, xhat, n, threads);
    int rc = orc_scatter_gather_stream(d, shape, k, q, idx, r, factors, n, xhat, yhat, threads);
    if (rc == 0) {
        orc_gemm(0, 0, n, r, n, 1.0, kmat, n, yhat, n, 0.0, y, n, threads);
        for (int64_t t = 0; t < n * r; ++t) y[t] += lambda * xhat[t];
        for (int64_t t = 0; t < n * r; ++t) y[t] = y[t] + rho * x[t];
    }
    free(xhat); free(yhat);
    return rc;
}

/* ---- unaligned.hpp:120-133 build_preconditioner's D ---------------------------------
 * D(i,j) = 1 / (gamma sigma_j mu_i^2 + lambda mu_i + rho); throws runtime_error on <= 0. */
int orc_precond_diag(int64_t n, int64_t r, const double* mu_k, const double* sigma_v,
                     double gamma, double lambda, double rho, double* dmat) {
    for (int64_t j = 0; j < r; ++j)
        for (int64_t i = 0; i < n; ++i) {
            const double denom = gamma * sigma_v[j] * mu_k[i] * mu_k[i] + lambda * mu_k[i] + rho;
            if (denom <= 0.0) return fail(2, "build_preconditioner: nonpositive denominator");
            dmat[i + n * j] = 1.0 / denom;
        }
    return 0;
}

/* ---- unaligned.hpp:135-139 M^-1 x = U_K ((U_K' X U_V) .* D) U_V', left-to-right. ---- */
int orc_precond_apply(int64_t n, int64_t r, const double* uk, const double* uv, const double* dmat,
                      const double* x, double* y, int threads) {
    double* t1 = (double*)malloc(sizeof(double) * n * r);
    double* t2 = (double*)malloc(sizeof(double) * n * r);
    if (!t1 || !t2) { free(t1); free(t2); return fail(2, "out of memory"); }
    orc_gemm(1, 0, n, r, n, 1.0, uk, n, x, n, 0.0, t1, n, threads);      /* U_K' X      */
    orc_gemm(0, 0, n, r, r, 1.0, t1, n, uv, r, 0.0, t2, n, threads);     /* (.) U_V     */
    for (int64_t t = 0; t < n * r; ++t) t2[t] *= dmat[t];                 /* .* D        */
    orc_gemm(0, 0, n, r, n, 1.0, uk, n, t2, n, 0.0, t1, n, threads);     /* U_K (.)     */
    orc_gemm(0, 1, n, r, r, 1.0, t1, n, uv, r, 0.0, y, n, threads);      /* (.) U_V'    */
    free(t1); free(t2);
    return 0;
}

/* ---- tensor.hpp:158-165 + matrix_ops.hpp:24-42: Z_k = A_d (.) ... (.) A_1 without A_k,
 * last factor's row index fastest.  z is (prod_{i!=k} n_i) x r column-major. ---------- */
void orc_khatri_rao_excluding(int d, const int64_t* shape, int k, int64_t r,
                              const double* const* factors, double* z) {
    /* row index of Z = sum over remaining modes ascending, lower modes fastest */
    int64_t rows = 1;
    for (int i = 0; i < d; ++i) if (i != k) rows *= shape[i];
    for (int64_t j = 0; j < r; ++j) {
        for (int64_t row = 0; row < rows; ++row) {
            /* khatri_rao multiplies out = A_d first, then successive lower modes:
             * value = A_d(i_d) * A_{d-1}(i_{d-1}) * ... (left to right, descending mode) */
            int64_t rem = row;
            int64_t sub[16];
            for (int i = 0; i < d; ++i) {
                if (i == k) continue;
                sub[i] = rem % shape[i];
                rem /= shape[i];
            }
            double v = 0.0;
            int first = 1;
            for (int i = d - 1; i >= 0; --i) {
                if (i == k) continue;
                const double a = factors[i][sub[i] + shape[i] * j];
                v = first ? a : v * a;
                first = 0;
            }
            z[row + rows * j] = v;
        }
    }
}

/* ---- tensor.hpp:74-104 unfold + :174-182 mttkrp = unfold(t,k) * Z_k -------------- */
int orc_mttkrp(int d, const int64_t* shape, const double* t, int k, int64_t r,
               const double* const* factors, double* b, int threads) {
    if (k < 0 || k >= d) return fail(1, "unfold: mode out of range");
    int64_t ntot = 1;
    for (int i = 0; i < d; ++i) ntot *= shape[i];
    const int64_t n = shape[k], m = ntot / n;
    double* unf = (double*)malloc(sizeof(double) * ntot);
    double* z = (double*)malloc(sizeof(double) * m * r);
    if (!unf || !z) { free(unf); free(z); return fail(2, "orc_mttkrp: out of memory"); }
    int64_t stride_k = 1;
    for (int i = 0; i < k; ++i) stride_k *= shape[i];
    int64_t idx[16] = {0};
    for (int64_t col = 0; col < m; ++col) {
        int64_t base = 0, stride = 1;
        for (int i = 0; i < d; ++i) {
            if (i == k) { stride *= shape[i]; continue; }
            base += idx[i] * stride;
            stride *= shape[i];
        }
        for (int64_t row = 0; row < n; ++row) unf[row + n * col] = t[base + row * stride_k];
        for (int i = 0; i < d; ++i) {
            if (i == k) continue;
            if (++idx[i] < shape[i]) break;
            idx[i] = 0;
        }
    }
    orc_khatri_rao_excluding(d, shape, k, r, factors, z);
    orc_gemm(0, 0, n, r, m, 1.0, unf, n, z, m, 0.0, b, n, threads);
    free(unf); free(z);
    return 0;
}

/* ---- tensor.hpp:186-194 gram_khatri_rao: V = ones; V .*= A_i' A_i, ascending i != k - */
void orc_gram_khatri_rao(int d, const int64_t* shape, int64_t r, const double* const* factors,
                         int k, double* v) {
    for (int64_t t = 0; t < r * r; ++t) v[t] = 1.0;
    for (int i = 0; i < d; ++i) {
        if (i == k) continue;
        const double* a = factors[i];
        const int64_t ni = shape[i];
        for (int64_t c = 0; c < r; ++c)
            for (int64_t e = 0; e < r; ++e) {
                double s = 0.0;
                for (int64_t row = 0; row < ni; ++row) s += a[row + ni * e] * a[row + ni * c];
                v[e + r * c] *= s;
            }
    }
}

/* ---- aligned.hpp:41-54 solve_aligned_decoupled with a given (shared) eig ----------
 * core = (U_K' B) U_V; core(i,j) /= sigma_j mu_i + lambda (throw if == 0);
 * W = (U_K core) U_V'. */
int orc_solve_aligned_decoupled(int64_t n, int64_t r, const double* uk, const double* mu_k,
                                const double* uv, const double* sigma_v, double lambda,
                                const double* b, double* w, int threads) {
    double* t1 = (double*)malloc(sizeof(double) * n * r);
    double* core = (double*)malloc(sizeof(double) * n * r);
    if (!t1 || !core) { free(t1); free(core); return fail(2, "out of memory"); }
    orc_gemm(1, 0, n, r, n, 1.0, uk, n, b, n, 0.0, t1, n, threads);
    orc_gemm(0, 0, n, r, r, 1.0, t1, n, uv, r, 0.0, core, n, threads);
    for (int64_t j = 0; j < r; ++j)
        for (int64_t i = 0; i < n; ++i) {
            const double denom = sigma_v[j] * mu_k[i] + lambda;
            if (denom == 0.0) {
                free(t1); free(core);
                return fail(2, "solve_aligned_decoupled: zero eigenvalue pair; use lambda > 0");
            }
            core[i + n * j] /= denom;
        }
    orc_gemm(0, 0, n, r, n, 1.0, uk, n, core, n, 0.0, t1, n, threads);
    orc_gemm(0, 1, n, r, r, 1.0, t1, n, uv, r, 0.0, w, n, threads);
    free(t1); free(core);
    return 0;
}
