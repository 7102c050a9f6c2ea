/* sqp.h — C ABI of the closed-loop SQP driver in libipm.so.
 *
 * Solves the smooth NLP (eq:nlp_general, with linear constraints)
 *
 *     min f(x)   s.t.   l <= A x <= u,   xl <= x <= xu
 *
 * by sequential quadratic programming: every iteration builds the QP
 * subproblem eq:qp_subproblem (reading R17) with a quasi-Newton BFGS Hessian
 * and solves it with the GPU interior point method of ipm.h.  The subproblem is
 * written in x-space, y = x_k + d:
 *
 *     min 1/2 y^T B_k y + (grad f(x_k) - B_k x_k)^T y   s.t. the constant constraints above,
 *
 * so A and the bounds never change and only g (ipm_set_linear_term) and B (two-column
 * update, ipm_update_hessian_rank2) move between subproblems.  Globalisation:
 * Armijo backtracking on f (R21); BFGS with Powell damping.  B_0 = diag(h0),
 * h0 = diag(D^T W D) + h0_floor (R20).  Every step runs in this library's kernels (the
 * objective/gradient kernels below and the IPM); the host only takes the scalar decisions.
 *
 * Built-in objective (R20): the dose-like
 *     f(x) = sum_i 1/2 w_i (d_i - p_i)^2 + kappa_i / beta * exp(beta (d_i - dmax_i)),  d = D x
 * with D a sparse non-negative voxels x variables matrix (CSR).
 *
 * Conventions: all array pointers are DEVICE pointers unless named *_host; "BORROWED" arrays
 * must stay alive and unchanged until ipm_sqp_destroy.  Errors return a status from ipm.h
 * and leave a message for ipm_sqp_last_error.
 */
#ifndef IPM_SQP_H
#define IPM_SQP_H

#include "ipm.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ipm_sqp ipm_sqp;

/* The dose-like objective.  D: nd x n CSR, int64 row offsets, int32 columns strictly
 * increasing within a row, finite values.  All BORROWED. */
typedef struct {
    int64_t nd;                 /* rows of D (voxels), >= 1 */
    int64_t nnz;                /* nonzeros of D */
    const int64_t *D_rowptr;    /* nd + 1 */
    const int32_t *D_col;       /* nnz */
    const double *D_val;        /* nnz */
    const double *w;            /* nd, weights > 0 */
    const double *p;            /* nd, prescriptions */
    const double *dmax;         /* nd, over-dose thresholds */
    const double *kappa;        /* nd, >= 0, exponential penalty weights */
    double beta;                /* > 0 */
} ipm_dose_nlp;

typedef struct {
    int32_t size;               /* = sizeof(ipm_sqp_options) */
    int32_t max_iter;           /* 50   SQP iterations (= QP subproblems) */
    double tol_d;               /* 1e-6 stop when ||d||_inf <= tol_d * max(1, ||x||_inf) */
    double armijo_c1;           /* 1e-4 */
    int32_t max_backtrack;      /* 30   halvings of t per line search */
    double powell;              /* 0.2  Powell damping threshold */
    int32_t warm_start;         /* 0    1: warm-start each QP from the previous one (R15) */
    int32_t hess_kind;          /* 0: dense n x n B in the workspace (rank-2 update in place);
                                   1: compact B = diag(h0) + U diag(w) U^T (NEXT-1) */
    int32_t max_cols;           /* compact: capacity of U; 0 => 2 * max_iter.  When full, further
                                   updates are skipped (counted in updates_skipped). */
    double h0_floor;            /* 1e-3 (R20) */
} ipm_sqp_options;

typedef struct {
    int32_t status;             /* IPM_OK = converged, IPM_NOT_CONVERGED = max_iter reached,
                                   else the failing QP's status */
    int32_t iters;              /* QP subproblems solved */
    double f;                   /* objective at the returned x */
    double d_inf;               /* ||d||_inf of the last subproblem */
    int64_t ipm_iters_total;
    int64_t pcg_iters_total;
    int32_t updates_skipped;    /* BFGS updates skipped (s^T B s <= 0, y~^T s <= 0, U full) */
    int32_t backtracks;         /* total step halvings */
    double t_total_ms;          /* device time of ipm_sqp_solve (CUDA events) */
    double t_qp_ms;             /* sum of the QP solves' device time */
} ipm_sqp_stats;

typedef struct {
    int32_t it;                 /* 0-based SQP iteration */
    int32_t ipm_iters;
    int64_t pcg_iters;
    double f;                   /* f(x_k) before the step */
    double d_inf;
    double step;                /* accepted t (0 on the converged iteration) */
    double theta;               /* Powell damping factor (1 = undamped) */
    double qp_ms;               /* device time of this QP solve */
    int32_t updated;            /* 1: BFGS columns appended */
    int32_t ncols;              /* compact: columns of U in use after this iteration */
} ipm_sqp_trace_rec;

void ipm_sqp_options_default(ipm_sqp_options *opt);

/* Workspace bytes for ipm_sqp_create (host arithmetic).  cons: n, m, nnz, A, l, u, xl, xu of
 * the constraints (H, g, sharding and Hessian fields ignored; unsharded only). */
ipm_status ipm_sqp_workspace_size(const ipm_problem *cons, const ipm_dose_nlp *nlp, const ipm_sqp_options *sopt,
                                  const ipm_options *qopt, size_t *bytes);

/* Create: validates the objective data, builds D^T on the device (deterministic counting
 * sort), h0, B_0 and the inner IPM context (qopt: options of every QP solve, NULL =
 * defaults).  workspace: >= ipm_sqp_workspace_size() bytes, 256-byte aligned, caller-owned. */
ipm_status ipm_sqp_create(ipm_sqp **sqp, const ipm_problem *cons, const ipm_dose_nlp *nlp,
                          const ipm_sqp_options *sopt, const ipm_options *qopt, void *workspace,
                          size_t workspace_bytes, ipm_stream_t stream);

/* Run SQP from x0 (device, n; must satisfy xl <= x0 <= xu and l <= A x0 <= u — R21 keeps
 * every iterate feasible).  Restarts from B_0. */
ipm_status ipm_sqp_solve(ipm_sqp *sqp, const double *x0);

ipm_status ipm_sqp_get_x(ipm_sqp *sqp, double *x);
ipm_status ipm_sqp_get_stats(ipm_sqp *sqp, ipm_sqp_stats *stats);
ipm_status ipm_sqp_get_trace(ipm_sqp *sqp, ipm_sqp_trace_rec *recs, int32_t cap, int32_t *count);

/* Test hook: f(x) (host double) and grad f(x) (device, n; NULL = skip) with the kernels the
 * driver uses. */
ipm_status ipm_sqp_eval(ipm_sqp *sqp, const double *x, double *f_host, double *grad);

/* The inner IPM context (for ipm_get_info / ipm_kernel_launches); owned by sqp. */
ipm_ctx *ipm_sqp_qp(ipm_sqp *sqp);
int64_t ipm_sqp_kernel_launches(const ipm_sqp *sqp);
const char *ipm_sqp_last_error(const ipm_sqp *sqp);   /* NULL sqp: last create error */
void ipm_sqp_destroy(ipm_sqp *sqp);

#ifdef __cplusplus
}
#endif
#endif /* IPM_SQP_H */
