/*
 * gapsafe_b200 -- C ABI of the B200-native Gap Safe Lasso hot path.
 *
 * This is the drop-in boundary.  The reference package
 * (/root/reference/pkg/src/gapsafe) has no FFI layer of its own; its
 * "operator API" for the path is (1) the in-place numba kernels of
 * _kernels.py, (2) the DesignMatrix method set and (3) the public solver
 * entry points.  Each entry point below names the reference interface it
 * replaces.  Plain pointers and sizes only: every host pointer is borrowed for
 * the duration of the call; device buffers are owned by the handles.
 *
 * Errors: functions return GS_OK (0) or a negative code; gs_last_error()
 * gives a thread-local message.  The codes map onto the reference's Python
 * exceptions (problem.py:12, regions.py:19, solver.py:86-87,
 * design_matrix.py:96-98).  There is no CPU fallback: without a CUDA device
 * every call fails with GS_ERR_NODEVICE.
 */
#ifndef GAPSAFE_B200_H
#define GAPSAFE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GS_OK 0
#define GS_ERR_CUDA (-1)        /* CUDA runtime failure                        */
#define GS_ERR_VALUE (-2)       /* ValueError                                  */
#define GS_ERR_INDEX (-3)       /* IndexError (design_matrix.py:96-98)         */
#define GS_ERR_RUNTIME (-4)     /* RuntimeError: zero-norm active column       */
#define GS_ERR_INFEASIBLE (-5)  /* InfeasibleDualError (problem.py:12,74-76)   */
#define GS_ERR_NUMERICAL (-6)   /* NumericalInconsistencyError (regions.py:19) */
#define GS_ERR_NODEVICE (-7)    /* no CUDA device: fail loudly, never fall back */

#define GS_DTYPE_F64 0
#define GS_DTYPE_F32 1

#define GS_RULE_NONE 0          /* solver.py:27 Rule.NONE       */
#define GS_RULE_GAP_SPHERE 1    /* solver.py:31 Rule.GAP_SPHERE */
#define GS_RULE_STATIC 2        /* solver.py:28 Rule.STATIC, regions.py:162-165  */
#define GS_RULE_DYNAMIC 3       /* solver.py:29 Rule.DYNAMIC, regions.py:168-174 */
#define GS_RULE_ST3 4           /* solver.py:30 Rule.ST3, regions.py:177-197     */
#define GS_RULE_GAP_DOME 5      /* solver.py:32 Rule.GAP_DOME, regions.py:235-273 */

typedef struct gs_matrix gs_matrix;
typedef struct gs_solver gs_solver;

/* ---- runtime ------------------------------------------------------------ */
int gs_init(int device);
int gs_device_count(int *count);
const char *gs_last_error(void);
const char *gs_version(void);
/* number of kernels this library has launched so far in this process */
int64_t gs_launch_count(void);

/* ---- DesignMatrix storage (design_matrix.py:34-57) ----------------------- */
/* Dense column-major design, column j at X + j*ld_host (F-order numpy array).
 * dtype GS_DTYPE_F64 or GS_DTYPE_F32 (fp32 storage, fp64 arithmetic).
 * norms_sq: optional host column norms^2 (else computed on the device). */
int gs_matrix_dense(const void *X, int dtype, int64_t n, int64_t p, int64_t ld_host,
                    const double *norms_sq, gs_matrix **out);
/* The same from a DEVICE buffer (column j at X_dev + j*ld_dev): device-to-device
 * copy into owned storage.  The column-sharded path builds
 * the survivors' sub-design X_A from columns received over NCCL without a
 * host round trip.  The caller synchronises the producer of X_dev first. */
int gs_matrix_dense_dev(const void *X_dev, int dtype, int64_t n, int64_t p, int64_t ld_dev, gs_matrix **out);
/* A dense design built block by block (designs too large for one host array,
 * e.g. configs[2] at 40 GB): allocate zeroed device storage, upload column
 * blocks [j0, j0+k) from a host buffer (column-major, ld_host rows; reusable
 * on return), then finalize (column norms).  No other call is valid on the
 * matrix before gs_matrix_dense_finalize. */
int gs_matrix_dense_alloc(int dtype, int64_t n, int64_t p, gs_matrix **out);
int gs_matrix_dense_set_columns(gs_matrix *M, int64_t j0, int64_t k, const void *X, int64_t ld_host);
int gs_matrix_dense_finalize(gs_matrix *M);
/* Columns idx[0..k) of a dense design into a DEVICE buffer (ld_dst rows per
 * column, rows past n zeroed): the send buffer of that gather.  Returns after
 * the copy completed. */
int gs_matrix_gather_columns_dev(const gs_matrix *M, const int64_t *idx, int64_t k, void *dst_dev, int64_t ld_dst);
/* Canonical CSC (sorted, deduplicated), design_matrix.py:37-43. */
int gs_matrix_csc(const double *data, const int32_t *indices, const int64_t *indptr,
                  int64_t n, int64_t p, const double *norms_sq, gs_matrix **out);
int gs_matrix_norms_sq(const gs_matrix *M, double *out);              /* col_norms_sq */
int64_t gs_matrix_device_bytes(const gs_matrix *M);
void gs_matrix_free(gs_matrix *M);

/* ---- DesignMatrix primitives ---------------------------------------------- */
/* X^T v (cols == NULL: all p columns, design_matrix.py:144-149) or restricted
 * to cols (_kernels.py:14-36 tdot_dense/tdot_csc).  exact_order = 1 uses the
 * reference's sequential non-FMA order (bit-exact with _kernels.py). */
int gs_tdot(const gs_matrix *M, const double *v, const int64_t *cols, int64_t k,
            double tail_scale, double *out, int exact_order);
/* X @ beta (design_matrix.py:130-137). */
int gs_matvec(const gs_matrix *M, const double *beta, double *out);
/* (max_j |x_j^T v|, argmax), smallest index on ties (design_matrix.py:160-174). */
int gs_max_abs_correlation(const gs_matrix *M, const double *v, const int64_t *restrict_cols,
                           int64_t k, double *val, int64_t *arg);
/* v += a * x_j (design_matrix.py:115-128). */
int gs_axpy_col(const gs_matrix *M, int64_t j, double a, double *v);

/* ---- kernel twin of the CD epoch (_kernels.py:39-92, solver.py:82-101) --- */
/* beta, rho updated in place.  norms_sq NULL: the matrix's own.  exact_order = 1
 * reproduces the reference arithmetic bit for bit; 0 runs the production
 * kernel (CTA-parallel dot, certified-zero skipping). */
int gs_cd_pass(const gs_matrix *M, double *beta, double *rho, const int64_t *active, int64_t k,
               double lam, const double *norms_sq, double tail_scale, int exact_order);

/* ---- sphere screening (regions.py:75-79,129-139) --------------------------- */
/* mu_j = |x_j^T center| + radius*||x_j||, active = {mu >= 1 - tol} ascending.
 * cols NULL: all p.  mu (len k or p) may be NULL. */
int gs_screen_sphere(const gs_matrix *M, const double *center, double radius, const int64_t *cols,
                     int64_t k, double tol, double *mu, int64_t *active_out, int64_t *n_active);

/* device reductions for the problem.py scalar algebra: dot = a.b (b may be
 * NULL), asum = sum |a|. */
int gs_vec_stats(const double *a, const double *b, int64_t n, double *dot, double *asum);

/* ---- solver (solver.py:149-246) and path driver support (path.py:52-105) - */
typedef void (*gs_ckpt_cb)(const int64_t *active, int64_t n_active, void *user);

typedef struct {
    double epsilon;          /* absolute gap tolerance (solver.py:37)   */
    int64_t max_passes;      /* solver.py:38                            */
    int64_t screen_every;    /* solver.py:39                            */
    int32_t rule;            /* GS_RULE_*                               */
    int32_t certify;         /* 1: certified-zero skipping in CD (exact) */
    gs_ckpt_cb on_checkpoint;/* solver.py:41-45 hook (NULL: none)      */
    void *user;
} gs_solve_config;

typedef struct {
    /* caller-provided host buffers (NULL: not copied) */
    double *beta;            /* [p] */
    double *residual;        /* [n] */
    double *theta;           /* [n] */
    int64_t *active;         /* [p] */
    int64_t *trace_passes;   /* [trace_cap] */
    int64_t *trace_active;
    double *trace_gap;
    double *trace_radius;
    int64_t trace_cap;
    /* outputs */
    int64_t n_active, n_trace, passes_done;
    int32_t converged, interpolating, lambda_max_shortcut, pad_;
    double margin, primal, dual, gap;
    uint64_t cd_visits, cd_uncertified, cd_nonzero;
    int64_t checkpoints;
    double device_ms;
    /* in-kernel phase times (device %globaltimer, ms) and counts */
    double screen_ms, ckpt_ms, refresh_ms, cd_ms;
    int64_t n_screen, n_refresh, launches;
    /* CD pipeline: candidates fetched, skipped as certified, queue rebuilds */
    int64_t cd_candidates, cd_skipped, cd_requeues;
} gs_solve_result;

/* y is uploaded once; lambda_max = |X^T y|_inf is computed once and cached
 * (problem.py:50 recomputes it per LassoProblem; the value is identical). */
int gs_solver_create(const gs_matrix *M, const double *y, gs_solver **out);
int gs_solver_lambda_max(gs_solver *S, double *lambda_max, int64_t *j_star, double *y_norm_sq);
/* Override lambda_max (LassoProblem(X, y, lam, lambda_max=...) of the oracle;
 * problem.py:50): a solver over a gathered column subset X_A of a sharded
 * design takes the full design's lambda_max, so the lambda >= lambda_max
 * shortcut (solver.py:160-161) is decided on the whole problem. */
int gs_solver_set_lambda_max(gs_solver *S, double lambda_max);
/* warm start (solver.py:164-169): beta == NULL -> zeros */
int gs_solver_set_beta(gs_solver *S, const double *beta);
/* Sequential gap-sphere screen at lam from the previous solve's (beta, theta,
 * residual) (path.py:82-91): leaves active0 on the device for the next solve. */
int gs_solver_seq_screen(gs_solver *S, double lam, int64_t *n_active);
/* active0_mode: 0 none (all nonzero-norm columns), 1 host array active0[n0],
 * 2 the device set left by gs_solver_seq_screen. */
int gs_solver_solve(gs_solver *S, double lam, const gs_solve_config *cfg, const int64_t *active0,
                    int64_t n0, int active0_mode, gs_solve_result *res);
void gs_solver_free(gs_solver *S);

/* ---- batched independent problems (BASELINE configs[4]) ---- */
/* B problems on row-resampled copies of one dense design: problem b uses rows
 * rows[b*n .. b*n+n) of X0 (with repetition) and the same entries of y0.  Each
 * problem runs its whole warm-started path in one CTA (device-side lambda loop). */
typedef struct gs_batch gs_batch;
int gs_batch_create(const gs_matrix *X0, const double *y0, const int32_t *rows, int64_t B, int64_t n,
                    gs_batch **out);
int gs_batch_lambda_max(gs_batch *Bt, double *lambda_max);      /* [B] */
/* grids: [B*T] (each non-increasing).  eps: per-problem gap tolerances [B]
 * (the reference takes epsilon per solve, solver.py:37,226; configs[4] uses
 * 1e-8 ||y_b||^2), or NULL for cfg->epsilon everywhere.  Outputs [B*T] (betas
 * [B*T*p], may be NULL). */
int gs_batch_run_paths(gs_batch *Bt, const double *grids, int64_t T, const gs_solve_config *cfg, const double *eps,
                       double *betas, int64_t *passes, double *gaps, int32_t *converged, int64_t *n_active,
                       double *device_ms);
void gs_batch_free(gs_batch *Bt);

/* ---- measurement support ---------------------------------------------------- */
/* CUDA events on the solver's stream: op 0 records the start, op 1 records the
 * stop, synchronizes and returns the elapsed milliseconds in *ms. */
int gs_solver_timer(gs_solver *S, int op, double *ms);
/* The full-p sphere screening pass: one warm-up pass (fused GEMV + test, then
 * stable compaction), then the fused GEMV+test kernel launched `reps` times on
 * the matrix stream and timed with CUDA events; *ms is the average per launch,
 * *n_active the survivors. */
int gs_screen_timed(const gs_matrix *M, const double *center, double radius, int reps, double *ms,
                    int64_t *n_active, int32_t *active_out /* [p] or NULL: the survivors, ascending */);
/* pinned (page-locked) host memory for H2D/D2H at full PCIe rate */
int gs_host_alloc(int64_t bytes, void **out);
void gs_host_free(void *ptr);

#ifdef __cplusplus
}
#endif
#endif /* GAPSAFE_B200_H */
