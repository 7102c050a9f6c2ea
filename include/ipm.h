/*
 * ipm.h — C ABI of libipm.so, the B200-native (sm_100a) data-parallel hot path of the
 * GPU interior point method of arxiv 2405.03584 (Liu, Fredriksson, Markidis).
 *
 * The library solves the convex QP (eq:qp, bounds split out as in P:176)
 *
 *     min 1/2 x^T H x + g^T x    s.t.   l <= A x <= u ,   xl <= x <= xu
 *
 * with Algorithm 1: every search direction is a Jacobi-preconditioned CG
 * solve of the condensed Newton system
 *
 *     K dx = rhs ,   K = H + Sigma_b + A^T Sigma_c A                                  (1)
 *
 * which is the Schur complement of the reduced system eq:2x2_reduced:
 * Sigma_b = S_lx^-1 Lam_lx + S_ux^-1 Lam_ux (the diagonal part of Q) and
 * Sigma_c = Lam_lA S_lA^-1 + Lam_uA S_uA^-1 (B^T D^-1 B with B = [A_l; -A_u]).
 *
 * Conventions (all calls):
 *   - Values fp64 (IEEE binary64), CSR row offsets int64, CSR column indices int32.
 *   - Every pointer argument is DEVICE memory on the context's device unless the
 *     parameter name ends in _host.  Vectors are dense, unit stride.
 *   - Absent bounds are +-INFINITY.  Bound families are masked full-length vectors:
 *     entry i of an m-vector belongs to row i of A, entry j of an n-vector to x_j.
 *     Entries of slack/multiplier vectors whose bound is absent are 0.
 *   - All work is stream-ordered on the cudaStream_t given to ipm_create.  Calls that
 *     return host values (stats, traces, objective) synchronise that stream.
 *   - No call throws across the ABI; every failure returns a status and sets a
 *     message readable with ipm_last_error(ctx) (or ipm_last_error(NULL) when no
 *     context exists yet).
 *   - Results are bitwise reproducible run to run on the same device and shapes: no
 *     floating-point atomics, fixed-order reductions, stored A^T.
 */
#ifndef IPM_B200_IPM_H
#define IPM_B200_IPM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IPM_ABI_VERSION 1

typedef struct ipm_ctx ipm_ctx;
typedef void *ipm_stream_t; /* a cudaStream_t / CUstream (NULL = legacy default stream) */

typedef enum {
    IPM_OK = 0,
    IPM_NOT_CONVERGED = 1,     /* iteration limit N reached; last iterate retrievable */
    IPM_ERR_INVALID = 2,       /* bad dims, CSR not sorted/unique/in range, l>=u, xl>=xu, NaN data */
    IPM_ERR_PCG_BREAKDOWN = 3, /* p^T K p <= 0 or non-finite inside PCG: loss of SPD */
    IPM_ERR_NONFINITE = 4,     /* non-finite residual / step; last finite iterate kept */
    IPM_ERR_CUDA = 5,          /* a CUDA runtime error (message has the CUDA error string) */
    IPM_ERR_OOM = 6,           /* workspace smaller than ipm_workspace_size() */
    IPM_ERR_NCCL = 7,          /* NCCL failure in the row-sharded path */
    IPM_ERR_STATE = 8          /* call not valid in this state (e.g. solution before solve) */
} ipm_status;

/* Options.  Fill with ipm_options_default() and then override fields. */
typedef struct {
    int32_t size;               /* = sizeof(ipm_options); ABI versioning */
    double mu_tol;              /* 1e-8   Alg. 1 line 11 mu_tol (reading R6) */
    double mu0_scale;           /* 0.1    mu0 = mu0_scale * sum(lam s) / #bounds (R5) */
    double mu_divisor;          /* 10     Alg. 1 line 14 "mu <- mu/10" */
    double tau;                 /* 0.995  fraction to the boundary (R6) */
    int32_t max_ipm_iter;       /* 100    Alg. 1 "for i <- 1 to N" */
    int32_t pcg_schedule;       /* 0: rtol = max(floor, min(rtol_max, factor*mu))  (D6)
                                   1: SPEC S:238 rtol = max(1e-10, min(1e-2, 0.1 mu)) */
    double pcg_rtol_max;        /* 1e-6 */
    double pcg_rtol_mu_factor;  /* 1e-3 */
    double pcg_rtol_floor;      /* 1e-12 */
    double pcg_atol;            /* 1e-13  absolute floor on ||r||_2 */
    int32_t pcg_max_iter;       /* 0 => 10*n */
    int32_t predictor_corrector;/* 0: Alg. 1 verbatim (default); 1: Mehrotra (R18, option) */
    int32_t trace;              /* 1: record one ipm_trace_rec per IPM iteration */
    int32_t use_graph;          /* 1: PCG loop as a CUDA graph with a device-side WHILE node */
    double warm_shift;          /* 0.1    theta of the warm-start rule (R15; R15) */
    int32_t gemv_kernel;        /* 0 auto: 3 when H == H^T bitwise — unsharded by a device compare at create,
                                   row-sharded by the allgathered hash certificate, and then only with an
                                   even chunk = ceil(n / nranks) — else 2.  1 LDG.128 register tiles,
                                   2 TMA-bulk mbarrier pipeline, 3 symmetric upper-triangle TMA-bulk */
    int32_t pcg_warm_start;     /* 0: each PCG starts from x0 = 0 (default, R11); 1: from the previous
                                   search direction (S:248 option) */
    int32_t pcg_system;         /* 0: PCG on the condensed system K dx = rhs (D1, default);
                                   1: PCG on the doubly augmented system eq:2x2_augmented,
                                   unknowns (dx, dlam_lA, dlam_uA), Jacobi preconditioner on its diagonal;
                                   unsharded only, and ipm_pcg() is then rejected (IPM_ERR_STATE) */
    int32_t a_row_split;        /* 1 (default): row-sharded with the peer data plane, the PCG's SpMV t = Sigma_c o
                                   (A p) runs on each rank's own m / nranks rows of A and the slices are
                                   allgathered over peer memory (north_star "A rows partitioned"); 0: every
                                   rank forms the whole t (A replicated).  No effect unsharded. */
    int32_t pcg_single_reduction; /* row-sharded only.  0 (default): Jacobi PCG with two scalar exchanges per
                                   iteration (p^T K p, then r^T z / ||r||^2).  1: the Chronopoulos-Gear
                                   single-reduction form — the operator is applied to u = M^-1 r and one
                                   exchange carries u^T K u, r^T u and ||r||^2 (same iterates in exact
                                   arithmetic; one extra operator apply at the end of each solve) */
    int32_t kernel_timer;       /* 0 (default): off.  1: the PCG operator kernel (GEMV / SYMV, PCG mode)
                                   times its own launches on the device for ipm_kernel_timer (two
                                   atomics per CTA per launch; used by bench.py's live roofline) */
} ipm_options;

/* Problem description for ipm_create.  Large arrays are BORROWED (the caller keeps them
 * alive and unchanged until ipm_destroy); small ones are copied at create. */
typedef struct {
    int64_t n;                  /* variables, >= 1 */
    int64_t m;                  /* rows of A, >= 0 */
    int64_t nnz;                /* nonzeros of A, >= 0 */
    const double *H;            /* BORROWED. Row-major SPD Hessian; element (i,j) at H[i*ldh + j].
                                   Sharded (nranks>1): only rows [row_begin,row_end), i.e. H points
                                   at the local block, element (i,j) at H[(i-row_begin)*ldh + j].
                                   Written only by ipm_update_hessian_rank2. */
    int64_t ldh;                /* >= n.  ldh even and H 16-byte aligned enable 128-bit loads. */
    const double *g;            /* n, copied */
    const int64_t *A_rowptr;    /* m+1, BORROWED; A_rowptr[0]=0, A_rowptr[m]=nnz, non-decreasing */
    const int32_t *A_col;       /* nnz, BORROWED; strictly increasing within each row, in [0,n) */
    const double *A_val;        /* nnz, BORROWED; finite */
    const double *l, *u;        /* m each, copied; -INF / +INF = absent; l < u where both finite */
    const double *xl, *xu;      /* n each, copied; xl < xu where both finite */
    /* Row sharding.  With chunk = ceil(n / nranks), rank r must own rows
     * [r*chunk, min(n, (r+1)*chunk)) of H and the same slice of every x-space vector; A (and
     * all m-space vectors) are replicated on every rank.  g, xl, xu are passed FULL length
     * (each rank copies its slice).  comm_kind: 0 = none (nranks must be 1); 1 = NCCL,
     * comm_handle_host -> ncclUniqueId (128 bytes, from ipm_nccl_unique_id on rank 0,
     * broadcast by the caller); 2 = in-process group, comm_handle_host = ipm_group* (one host
     * thread per rank must drive its context); 3 = caller-provided host allgather,
     * comm_handle_host = ipm_host_comm* (any transport: e.g. a gloo process group).
     * comm_kind 2 with nranks 1 runs the sharded code path on one context (testing).
     * DATA PLANE: with 2 <= nranks <= 8 every per-iteration exchange runs over peer memory
     * (each rank stores into the others' workspace regions over NVLink / NVSwitch; the regions'
     * addresses are exchanged once at create over the comm — CUDA IPC between processes, so the
     * workspace must be cudaMalloc memory, not a VMM/expandable-segment allocation); the comm
     * itself (NCCL, group or host callback) is then used only at create.  comm_kind 3 requires
     * this peer plane.  The environment switch IPM_PEER=0 keeps the comm allgathers instead
     * (comm_kind 1 / 2 only).  ipm_create is COLLECTIVE when sharded: all ranks
     * must call it concurrently (communicator setup and the exchange of the H-symmetry
     * certificate that selects the sharded symmetric GEMV for an exactly symmetric H with an
     * even chunk; every rank takes the same decision). */
    int64_t row_begin, row_end;
    int32_t rank, nranks;
    int32_t comm_kind;
    const void *comm_handle_host;
    /* Hessian representation.  hess_kind 0: the dense H above.  hess_kind 1:
     * compact quasi-Newton H = diag(h0) + U diag(w) U^T (eq:bfgs_hessian), applied
     * matrix-free as h0 o p + U (w o (U^T p)); H and ldh are ignored.  U is BORROWED,
     * n x ldu row-major, the first k columns in use; ipm_update_hessian_rank2 APPENDS (u, v) as
     * columns k, k+1 with weights (alpha, beta) — the paper's SQP adds two columns per iteration
     * — while k + 2 <= ldu.  h0 (n) and w (k) are copied.  Unsharded only. */
    int32_t hess_kind;
    int32_t k;
    int64_t ldu;
    const double *h0;
    double *U;
    const double *w;
} ipm_problem;

typedef struct ipm_group ipm_group;  /* in-process rank group (comm_kind 2) */

/* comm_kind 3: the caller's host allgather.  allgather(send, recv, bytes, user) must gather
 * `bytes` from every rank into recv (rank r's block at offset r * bytes) and return 0; it is
 * called only inside ipm_create (collective), never during a solve. */
typedef int32_t (*ipm_host_allgather_fn)(const void *send_host, void *recv_host, size_t bytes, void *user);
typedef struct {
    int32_t rank, nranks;
    ipm_host_allgather_fn allgather;
    void *user;
} ipm_host_comm;

typedef struct {
    int32_t status;             /* final ipm_status of the last ipm_solve */
    int32_t ipm_iters;
    int64_t pcg_iters_total;
    int32_t pcg_iters_max;
    int32_t pcg_stalls;         /* PCG solves that hit pcg_max_iter without reaching rtol */
    int32_t pcg_restarts;       /* true-residual restarts */
    double mu_final;
    double kkt_inf;             /* ||r||_inf over the nine residual families (R4) */
    double obj;                 /* 1/2 x^T H x + g^T x at the returned iterate */
    double t_solve_ms;          /* device time of the last ipm_solve (CUDA events) */
    double t_pcg_ms;            /* device time spent inside PCG solves */
} ipm_stats;

typedef struct {
    int32_t it;
    int32_t pcg_iters;
    double mu;
    double kkt_inf;
    double alpha_x, alpha_lam;
    double pcg_relres;          /* final true relative residual of the PCG solve */
    double obj;
} ipm_trace_rec;

/* Static facts about a created context (which kernels were selected, the partition). */
typedef struct {
    int32_t gemv_kernel;        /* 1 LDG tiles, 2 TMA-bulk, 3 symmetric upper-triangle TMA */
    int32_t ncb;                /* column blocks of the GEMV tile-partial layout */
    int32_t group_lanes;        /* lanes per A^T row in the fused SpMV^T kernels */
    int32_t sharded;            /* 1 when the row-sharded code path is active */
    int32_t rank, nranks;
    int64_t row_begin, row_end; /* rows of H owned by this context */
} ipm_info;

/* Fill defaults (documented per field above). */
void ipm_options_default(ipm_options *opt);

/* Sharding helpers.  ipm_nccl_unique_id writes an ncclUniqueId (needs >= 128 bytes) for
 * rank 0 to broadcast; ipm_group_create/destroy manage an in-process group of nranks
 * contexts (destroy only after every member context is destroyed). */
ipm_status ipm_nccl_unique_id(void *id_out_host, size_t bytes);
ipm_status ipm_group_create(int32_t nranks, ipm_group **group);
void ipm_group_destroy(ipm_group *group);

/* Bytes of device workspace ipm_create needs for this problem (host-only arithmetic). */
ipm_status ipm_workspace_size(const ipm_problem *prob, const ipm_options *opt, size_t *bytes);

/* Create a context: validates the problem (host copies of the O(n+m+nnz) data; H is checked
 * for non-finite entries on the device), copies g and the bounds, builds the stored
 * transpose A^T on the device (deterministic counting sort), caches diag(H).
 * workspace: device buffer of >= ipm_workspace_size() bytes, 256-byte aligned, owned by the
 * caller, not touched by anyone else until ipm_destroy.  The context's device is the
 * current CUDA device at the time of the call. */
ipm_status ipm_create(ipm_ctx **ctx, const ipm_problem *prob, const ipm_options *opt,
                      void *workspace, size_t workspace_bytes, ipm_stream_t stream);

/* Run Algorithm 1 to convergence (IPM_OK), to the iteration limit (IPM_NOT_CONVERGED) or
 * to an error.  Cold start from the S:290 initial point unless ipm_set_iterate /
 * ipm_warm_start was called since the last solve. */
ipm_status ipm_solve(ipm_ctx *ctx);

/* Copy the current iterate out (device pointers; NULL = skip).  obj_host: host double.
 * Sharded: x, lam_lx, lam_ux are this rank's row slice; lam_lA, lam_uA are full (replicated). */
ipm_status ipm_get_solution(ipm_ctx *ctx, double *x, double *lam_lA, double *lam_uA,
                            double *lam_lx, double *lam_ux, double *obj_host);

ipm_status ipm_get_stats(ipm_ctx *ctx, ipm_stats *stats);
ipm_status ipm_get_info(const ipm_ctx *ctx, ipm_info *info);
/* Copy up to cap trace records of the last solve (requires opt.trace = 1). */
ipm_status ipm_get_trace(ipm_ctx *ctx, ipm_trace_rec *recs_host, int32_t cap, int32_t *count_host);

/* C4 (SQP sequence): replace g (device, n); modify the borrowed H in place:
 * H <- H + alpha u u^T + beta v v^T (u, v device n-vectors, full length even when sharded);
 * diag(H) cache is updated; then ipm_warm_start makes the next solve start from the
 * current solution by the R15 rule. */
ipm_status ipm_set_linear_term(ipm_ctx *ctx, const double *g);
ipm_status ipm_update_hessian_rank2(ipm_ctx *ctx, const double *u, double alpha,
                                    const double *v, double beta);
ipm_status ipm_warm_start(ipm_ctx *ctx);
/* Replace the QP's bounds (device, FULL length even when sharded; copied).  In the paper's SQP
 * every sub-problem's linearised constraints g(x_k) + grad g(x_k)^T d <= 0 shift with the iterate
 * (P:140-146), so a sequence of QPs changes its bounds as well as g and H.  Validated like
 * ipm_create (NaN, l < u); which entries are finite may not change (it fixes the bound families),
 * else IPM_ERR_INVALID and nothing is changed.  Synchronises the context stream. */
ipm_status ipm_set_bounds(ipm_ctx *ctx, const double *l, const double *u, const double *xl, const double *xu);

/* Replace / read the iterate (masked full-length layout; order lA, uA, lx, ux). */
ipm_status ipm_set_iterate(ipm_ctx *ctx, const double *x, const double *const s4[4],
                           const double *const lam4[4], double mu);
ipm_status ipm_get_iterate(ipm_ctx *ctx, double *x, double *const s4[4], double *const lam4[4],
                           double *mu_host);

/* Test hooks — one stage of the hot path on caller-supplied diagonals (device):
 *   ipm_op_apply: y = K v with K of (1), Sigma_b = sig_b (n), Sigma_c = sig_c (m)
 *   ipm_op_diag : d = diag(K) = diag(H) + sig_b + colsq(A, sig_c)
 *   ipm_pcg     : Jacobi-PCG on K x = rhs from x = 0 to ||r|| <= rtol ||rhs|| (true residual
 *                 confirmed); iters_host gets the iteration count.
 * Sharded contexts: v is FULL length (n); sig_b, d, y, rhs and x are this rank's row slice;
 * sig_c is full (m). */
ipm_status ipm_op_apply(ipm_ctx *ctx, const double *sig_b, const double *sig_c, const double *v,
                        double *y);
ipm_status ipm_op_diag(ipm_ctx *ctx, const double *sig_b, const double *sig_c, double *d);
ipm_status ipm_pcg(ipm_ctx *ctx, const double *sig_b, const double *sig_c, const double *rhs,
                   double *x, double rtol, int32_t *iters_host);

/* Test hook (PCG-mode operator parity): exactly k >= 1 iterations of the PCG
 * recurrence ipm_solve runs (Jacobi PCG) on K x = rhs from x0 = 0, with
 * Sigma_b = sig_b, Sigma_c = sig_c — the same kernels and launch path (single-CTA loop for small
 * n; otherwise the CUDA graph: symmetric GEMV in PCG mode with p^T (H + Sigma_b) p fused, the
 * SpMV / SpMV^T branch, the fused cooperative update), but no stopping test, no true-residual
 * confirmation and no restart.  Outputs (device, this rank's rows; NULL = skip): x_k, r_k,
 * z_k = M^-1 r_k, and p = the search direction used by iteration k.  scal_host (NULL = skip)
 * receives 4 doubles {rho_k = r_k^T z_k, p^T K p of iteration k, alpha_k, ||r_k||^2}.
 * IPM_ERR_PCG_BREAKDOWN if p^T K p <= 0 or a non-finite value occurs. */
ipm_status ipm_pcg_iterate(ipm_ctx *ctx, const double *sig_b, const double *sig_c, const double *rhs, int32_t k,
                           double *x, double *r, double *z, double *p, double *scal_host);

/* Measurement hook (bench.py roofline): launch one hot-path stage `reps` times back to back
 * on the context's stream, bracketed by CUDA events recorded on that stream, with the
 * current PCG vectors as operands; *ms_host = average device time per launch.
 *   what = 0: the PCG GEMV kernel (y-tiles of H p + p^T H p), 1: the PCG SpMV (A p),
 *   what = 2: one full PCG iteration (all four kernels).  Clobbers PCG scratch state. */
ipm_status ipm_profile(ipm_ctx *ctx, int32_t what, int32_t reps, double *ms_host);

/* Host-only test hook (no device work): the work plan of the symmetric GEMV for global size
 * ncols split over nranks (equal chunks, rank's view) and `grid` CTAs.  Tiles are reported as
 * 8 int32 each {r0 (local), rows, c0 (global), cols, rslot, cmode, cbase, cslot}, ranges as 5
 * int32 per CTA {t0, s0, t1, s1, carry}; NULL outputs are skipped, at most cap tiles are
 * copied, *ntiles is always the full count.  *ldy / *ldz: ypart / remote-part strides.
 * Every ordered entry (i, j) of H must be used exactly once across ranks (tests/test_abi.py). */
ipm_status ipm_sym_plan(int32_t ncols, int32_t nranks, int32_t rank, int32_t grid, int32_t *tiles_host,
                        int32_t cap, int32_t *ntiles_host, int32_t *ranges_host, int32_t *ldy_host,
                        int32_t *ldz_host);

/* Number of kernel launches the library issued since create (graph nodes count once per
 * executed node); used by bench.py's gpu_launches. */
int64_t ipm_kernel_launches(const ipm_ctx *ctx);

/* Live device-side timing of the PCG operator kernel (the dominant GEMV / SYMV in PCG
 * mode): cumulative duration in ms (first CTA start to last CTA end, %globaltimer) and
 * number of timed launches since create, read on ctx's stream (synchronises it).
 * Counts only with opt.kernel_timer = 1 (else both stay 0).
 * bench.py differences two reads around its timed region.  Host pointers. */
ipm_status ipm_kernel_timer(ipm_ctx *ctx, double *ms_total_host, int64_t *launches_host);

/* Context-local message of the last failure (or the last create failure for NULL). */
const char *ipm_last_error(const ipm_ctx *ctx);
void ipm_destroy(ipm_ctx *ctx);
int32_t ipm_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* IPM_B200_IPM_H */
