/*
 * logmpoly_b200.h -- C ABI of the B200-native batched FP64 matrix logarithm.
 *
 * Drop-in boundary for the reference's Python hot path.  The
 * reference exposes no FFI; each entry point below replaces one reference function
 * (cited file:line, relative to /root/reference/pkg/src/logmpoly/):
 *
 *   lgm_logm_f64              <- logm(A, opts) -> (L, LogmReport)       (missing driver.py,
 *                                 imported at __init__.py:55)
 *   lgm_sqrt_db_f64           <- sqrt_db(A, tol, maxiter, counter)      (sqrtm.py:27-78)
 *   lgm_est_power_norm_f64    <- est_power_norm(B, p, counter, itmax)   (matcore.py:300-311)
 *   lgm_est_product_norm_f64  <- est_product_norm([(M1,p1),(M2,1)], ...) (matcore.py:234-297)
 *   lgm_balance_f64           <- balance(A, max_sweeps)                 (matcore.py:180-215)
 *   lgm_eval_degopt_f64       <- eval_degopt(builtin_scheme(k), A, counter, first_product)
 *   lgm_eval_degopt_scheme_f64 <- eval_degopt(scheme, A, counter, first_product) for any
 *                                 GraphScheme with k <= 9 products (schemes.py:50-126)
 *                                                                       (schemes.py:104-126, 337-350)
 *
 * Conventions: every matrix pointer is a DEVICE pointer to `batch` row-major n x n
 * float64 matrices with row stride `ld` >= n and matrix stride n*ld elements;
 * inputs are never written; outputs never alias inputs.  All calls are
 * stream-ordered on `stream` (a cudaStream_t; NULL = legacy default stream): they
 * never block the host (n > 64 runs as one CUDA graph whose loops are device-side
 * conditional nodes).  No hidden device allocation: scratch comes from the caller's
 * `workspace` (lgm_workspace_bytes / lgm_block_workspace_bytes; the n <= 64 building
 * blocks other than lgm_eval_degopt_f64 with k > 5 and lgm_expm_ref_f64 ignore it).  Argument / launch errors are returned synchronously
 * (< 0).  Per-matrix numerical outcomes are reported per matrix through status
 * codes (LGM_OK ... LGM_NONFINITE), which the Python layer maps onto the
 * reference's exceptions (exceptions.py:6-18); a failed matrix's L is all NaN.
 *
 * Threading: reentrant.  Calls on different workspaces may run concurrently on any
 * streams / devices; calls sharing one workspace must be ordered by the caller (as any
 * two users of one buffer).  Process-wide state: a mutex-guarded cache of instantiated
 * CUDA graphs keyed by (device, workspace address, n, batch, entry point), and the
 * monotonic launch counters behind lgm_launch_count.
 */
#ifndef LOGMPOLY_B200_H
#define LOGMPOLY_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* lgm_stream_t; /* identical to cudaStream_t */

/* per-matrix status (lgm_report.status and the building blocks' status arrays) */
enum {
  LGM_OK = 0,
  LGM_SINGULAR = 1,        /* exact zero pivot          -> SingularMatrixError (matcore.py:124-125) */
  LGM_DB_NOCONV = 2,       /* DB maxiter / collapse     -> ConvergenceError   (sqrtm.py:69-78)    */
  LGM_SCALING_MAXITER = 3, /* s reached opts.maxiter_s  -> ConvergenceError       */
  LGM_NONFINITE = 4,       /* NaN/Inf input or iterate  -> ValueError         (matcore.py:64-65)  */
  LGM_SPECTRUM = 5         /* set by the eig_small pre-check (lgm_spectrum_check_f64) when enabled */
};

/* call-level errors (return values) */
enum {
  LGM_ERR_ARG = -1,
  LGM_ERR_CUDA = -2,
  LGM_ERR_UNSUPPORTED = -3,
  LGM_ERR_WORKSPACE = -4
};

typedef struct lgm_opts {
  int32_t max_k;      /* highest scheme index: 1..5 shipped, 6..9 generated      default 5  */
  int32_t maxiter_s;  /* square-root cap (LogmOptions.maxiter)       default 40 */
  int32_t db_maxiter; /* sqrt_db maxiter (sqrtm.py:27)                            default 50 */
  int32_t est_itmax;  /* est_power_norm itmax (matcore.py:300)                    default 5  */
  int32_t balance;    /* LogmOptions.balance                                      default 1  */
  int32_t embedded_complex; /* 1: A holds the real 2m x 2m embeddings [[X, -Y], [Y, X]] of
                       * m x m complex matrices Z = X + iY (n = 2m); every norm, estimate,
                       * balancing and stop test is taken on Z as the reference's complex128
                       * path does (matcore.py:60-61, 226-231); L is the embedding of log Z.
                       * Always the graph engine; workspace from lgm_block_workspace_bytes. 0 */
  double db_tol;      /* sqrt_db tol; 0 -> 10 n u (sqrtm.py:44-45)                default 0  */
  const double* theta;/* HOST pointer to max_k thresholds; NULL -> frozen table             */
} lgm_opts;

typedef struct lgm_report { /* per matrix, written to device memory */
  int32_t status;
  int32_t s;                 /* square roots taken                                  */
  int32_t k;                 /* scheme index selected                               */
  int32_t db_iters;          /* DB iterations summed over roots                     */
  int32_t products;          /* OpCounter.products                                  */
  int32_t divisions;         /* OpCounter.divisions (2 per DB iteration)            */
  int32_t estimation_passes; /* OpCounter.estimation_passes                         */
  int32_t norm_estimations;  /* est_* calls performed                               */
  int32_t balanced;          /* balancing applied                                   */
  int32_t balance_sweeps;
  int32_t db_plateau;        /* DB stop tests taken with rel in [tol/10, 10 tol]: the    */
                             /* iteration count is rounding-noise dependent */
  int32_t inv_skipped;       /* DB X-inversions not executed: a root's last iteration needs */
                             /* only Y^-1 (its Y' is discarded), taken when predicted       */
  double alpha_used;         /* alpha certifying k (<= Theta_k on success)          */
  double min_margin;         /* min |x - thr| / |thr| over every discrete decision  */
} lgm_report;

void lgm_default_opts(lgm_opts* opts);

/* Workspace the caller must provide to lgm_logm_f64: 8 n^2 doubles per matrix for the
 * fused n <= 64 path (polynomial nodes P4..P10, A_prev / A_I2), the Engine G slots and
 * tables beyond (both + guard bands under LGM_WS_GUARD=1, see lgm_debug_ws_guard). */
int lgm_workspace_bytes(int64_t n, int64_t batch, size_t* bytes);

/* Workspace of the building blocks below (sized for the graph path at every n). */
int lgm_block_workspace_bytes(int64_t n, int64_t batch, size_t* bytes);

/* Largest n handled by the fused one-CTA-per-matrix engine. */
int lgm_max_fused_n(void);

int lgm_logm_f64(const double* A, double* L, int64_t n, int64_t batch, int64_t ld,
                 const lgm_opts* opts, lgm_report* rep_dev, void* workspace,
                 size_t workspace_bytes, lgm_stream_t stream);

/* X = A^(1/2) by the scaled coupled DB iteration; iters/status: int32[batch] device. */
int lgm_sqrt_db_f64(const double* A, double* X, int64_t n, int64_t batch, int64_t ld,
                    double tol, int32_t maxiter, int32_t* iters_dev, int32_t* status_dev,
                    void* workspace, size_t workspace_bytes, lgm_stream_t stream);

/* est = lower bound of ||M^p||_1; passes = estimation_passes; double/int32[batch] device. */
int lgm_est_power_norm_f64(const double* M, int64_t n, int64_t batch, int64_t ld, int32_t p,
                           int32_t itmax, double* est_dev, int32_t* passes_dev,
                           void* workspace, size_t workspace_bytes, lgm_stream_t stream);

/* est = lower bound of ||M1^p1 M2||_1 (M2 may be NULL: ||M1^p1||_1 without the zero shortcut). */
int lgm_est_product_norm_f64(const double* M1, int32_t p1, const double* M2, int64_t n,
                             int64_t batch, int64_t ld, int32_t itmax, double* est_dev,
                             int32_t* passes_dev, void* workspace, size_t workspace_bytes,
                             lgm_stream_t stream);

/* B = T^-1 A T with radix-2 scales; scale: double[batch*n] device; sweeps: int32[batch]. */
int lgm_balance_f64(const double* A, double* B, double* scale, int64_t n, int64_t batch,
                    int64_t ld, int32_t max_sweeps, int32_t* sweeps_dev, void* workspace,
                    size_t workspace_bytes, lgm_stream_t stream);

/* Z = z(X) for shipped scheme k; first_product (X^2, may be NULL) saves one product. */
int lgm_eval_degopt_f64(const double* X, const double* first_product, double* Z, int64_t n,
                        int64_t batch, int64_t ld, int32_t k, int32_t* products_dev,
                        void* workspace, size_t workspace_bytes, lgm_stream_t stream);

/* The same for a caller's scheme (GraphScheme: P1 = I, P2 = X, P_{j+2} = (sum_i lhs[j][i] P_i)
 * (sum_i rhs[j][i] P_i), z = sum_i out[i] P_i) with k = 1..9 products; coef (HOST) holds the
 * k lhs rows (row j has j + 2 entries), then the k rhs rows, then the k + 2 out entries.
 * first_product (X^2) requires lhs[0] == rhs[0] == (0, 1) (the caller checks, as schemes.py
 * does); non-finite coefficients -> LGM_ERR_ARG. */
int lgm_eval_degopt_scheme_f64(const double* X, const double* first_product, double* Z, int64_t n,
                               int64_t batch, int64_t ld, int32_t k, const double* coef,
                               int32_t* products_dev, void* workspace, size_t workspace_bytes,
                               lgm_stream_t stream);

/* E = expm(A) by the reference's test-oracle recipe (matcore.py:318-336 expm_ref): scale to
 * ||A||_1 <= 1/2, degree-20 Taylor in Horner form, square back.  Validation helper (round
 * trips of logm results on the device); workspace from lgm_block_workspace_bytes. */
int lgm_expm_ref_f64(const double* A, double* E, int64_t n, int64_t batch, int64_t ld,
                     void* workspace, size_t workspace_bytes, lgm_stream_t stream);

/* eig_small pre-check (matcore.py:343-355) on the device: flags[b] = 1 when
 * matrix b has an eigenvalue on the closed negative real axis, 0 when not, 2 when the QR
 * iteration did not converge.  Hessenberg reduction + Francis double-shift QR per matrix;
 * workspace >= batch * n * n doubles (lgm_block_workspace_bytes suffices). */
int lgm_spectrum_check_f64(const double* A, int32_t* flags_dev, int64_t n, int64_t batch, int64_t ld,
                           void* workspace, size_t workspace_bytes, lgm_stream_t stream);

const char* lgm_status_string(int code);

/* Diagnostics, not part of the reference interface.  With LGM_WS_GUARD=1 in the environment
 * (read once per process) every workspace region and n x n slot is followed by a guard band;
 * check = 0 fills the bands of `workspace` (layout 1: lgm_logm_f64 with n <= 64, 0: every
 * other workspace), check = 1 adds the number of changed guard bytes to *bad_dev (device
 * uint64).  Returns 1 if done, 0 if guards are off, < 0 on error. */
int lgm_debug_ws_guard(int64_t n, int64_t batch, int layout, void* workspace, int check,
                       unsigned long long* bad_dev, lgm_stream_t stream);

/* Number of CUDA kernels this library has launched so far (process-wide, monotonic):
 * direct launches plus the kernels executed inside Engine G graphs (counted on the device;
 * reading them synchronises, so call it outside timed regions).  bench.py reports the
 * difference across its timed region as gpu_launches. */
long long lgm_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* LOGMPOLY_B200_H */
