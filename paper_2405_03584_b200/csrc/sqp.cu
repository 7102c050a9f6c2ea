// sqp.cu — closed-loop SQP driver (§2.3).
//
// Kernels for the dose-like objective (R20) and the SQP vector steps, plus the host loop of
// include/sqp.h.  The QP subproblems go through the public IPM entry points of ipm.h (one
// inner context, created once: A and the bounds are constant in the x-space formulation).
//
// Deterministic: every reduction is a fixed-order block reduction + last-block combine; the
// trial point of the line search and the accepted iterate use the same fma(t, d_j, x_j), so
// the accepted f is bitwise the trial f.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "ipm.h"
#include "kernels.h"
#include "sqp.h"
#include "state.h"

#define IPM_EXPORT extern "C" __attribute__((visibility("default")))

namespace {
using namespace ipm;

constexpr int kPart = 2048;    // partial slots per reduction
constexpr int kSqpGrid = 148 * 8;

struct SqpScal {               // device scalars of the SQP kernels
    double red[4];
    unsigned long long bad;
    unsigned int cnt[4];
};

inline int sgrid(int64_t units, int per_block) {
    int64_t g = (units + per_block - 1) / per_block;
    if (g < 1) g = 1;
    if (g > kSqpGrid) g = kSqpGrid;
    return (int)g;
}

// Fixed-order combine of up to three per-block values (kind 0 = sum, 1 = max) into sc->red.
__device__ void publish(int ns, double v0, double v1, double v2, int k0, int k1, int k2, double *part, SqpScal *sc,
                        int cnt) {
    __shared__ double red[kBlock / 32];
    const double v[3] = {v0, v1, v2};
    const int k[3] = {k0, k1, k2};
    for (int q = 0; q < ns; ++q) {
        const double b = k[q] ? block_max(v[q], red) : block_sum(v[q], red);
        if (threadIdx.x == 0) part[q * kPart + blockIdx.x] = b;
    }
    if (last_block(&sc->cnt[cnt])) {
        for (int q = 0; q < ns; ++q) {
            const double t = k[q] ? max_partials(part + q * kPart, gridDim.x, red)
                                  : sum_partials(part + q * kPart, gridDim.x, red);
            if (threadIdx.x == 0) sc->red[q] = t;
        }
        if (threadIdx.x == 0) sc->cnt[cnt] = 0;
    }
}

// ------------------------------------------------------------------ objective (R20)
// f at z = x + t dir (dir == nullptr: z = x), warp per voxel row of D:
//   d_i = D_i: z,  f = sum 1/2 w (d - p)^2 + kappa/beta exp(beta (d - dmax)),
//   GRAD: e_i = w (d - p) + kappa exp(beta (d - dmax))   (grad f = D^T e, next kernel)
template <int GRAD>
__global__ void __launch_bounds__(kBlock)
k_dose_f(int nd, const int64_t *__restrict__ rp, const int *__restrict__ col, const double *__restrict__ val,
         const double *__restrict__ x, const double *__restrict__ dir, double t, const double *__restrict__ w,
         const double *__restrict__ p, const double *__restrict__ dmax, const double *__restrict__ kappa,
         double beta, double *__restrict__ e, double *__restrict__ part, SqpScal *sc) {
    const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    double facc = 0.0;
    for (int i = blockIdx.x * wpb + (threadIdx.x >> 5); i < nd; i += gridDim.x * wpb) {
        const int64_t s0 = rp[i], s1 = rp[i + 1];
        double a = 0.0;
        if (dir) {
            for (int64_t k = s0 + lane; k < s1; k += 32) {
                const int c = __ldg(col + k);
                a = fma(__ldg(val + k), fma(t, __ldg(dir + c), __ldg(x + c)), a);
            }
        } else {
            for (int64_t k = s0 + lane; k < s1; k += 32) a = fma(__ldg(val + k), __ldg(x + __ldg(col + k)), a);
        }
        a = warp_sum(a);
        if (lane == 0) {
            const double r = a - p[i];
            const double ex = exp(beta * (a - dmax[i]));
            facc += 0.5 * w[i] * r * r + kappa[i] / beta * ex;
            if (GRAD) e[i] = fma(w[i], r, kappa[i] * ex);
        }
    }
    publish(1, facc, 0, 0, 0, 0, 0, part, sc, 0);
}

// grad_j = (D^T e)_j, warp per row of the stored transpose; h0 mode: sum w D_ij^2 + floor.
template <int H0>
__global__ void __launch_bounds__(kBlock)
k_dose_t(int n, const int64_t *__restrict__ trp, const int *__restrict__ tcol, const double *__restrict__ tval,
         const double *__restrict__ e, double floor_, double *__restrict__ out) {
    const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    for (int j = blockIdx.x * wpb + (threadIdx.x >> 5); j < n; j += gridDim.x * wpb) {
        double a = 0.0;
        for (int64_t k = trp[j] + lane; k < trp[j + 1]; k += 32) {
            const double v = __ldg(tval + k);
            a = H0 ? fma(__ldg(e + __ldg(tcol + k)) * v, v, a) : fma(v, __ldg(e + __ldg(tcol + k)), a);
        }
        a = warp_sum(a);
        if (lane == 0) out[j] = H0 ? a + floor_ : a;
    }
}

// ------------------------------------------------------------------ SQP vector steps
enum VecOp { V_GQ = 0, V_DIR, V_STEP, V_CURV, V_DAMP };

// V_GQ  : o1 = a - b                                  (g - B x_k)
// V_DIR : o1 = a - b (d = y - x);  max|d|, g.d (c = g), max|x|
// V_STEP: o1 = fma(t, a, b) (x_{k+1}),  o2 = t a (s)   (a = d, b = x)
// V_CURV: o1 = a - b (y = g_new - g);  s.Bs, s.y       (c = s, e = Bs)
// V_DAMP: o1 = theta a + (1 - theta) b (y~; a = y, b = Bs);  y~.s (c = s)
__global__ void __launch_bounds__(kBlock)
k_sqp_vec(int op, int n, const double *__restrict__ a, const double *__restrict__ b, const double *__restrict__ c,
          const double *__restrict__ e, double t, double *__restrict__ o1, double *__restrict__ o2,
          double *__restrict__ part, SqpScal *sc) {
    double r0 = 0.0, r1 = 0.0, r2 = 0.0;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        switch (op) {
            case V_GQ: o1[j] = a[j] - b[j]; break;
            case V_DIR: {
                const double d = a[j] - b[j];
                o1[j] = d;
                r0 = fmax(r0, fabs(d));
                r1 = fma(c[j], d, r1);
                r2 = fmax(r2, fabs(b[j]));
            } break;
            case V_STEP: {
                o1[j] = fma(t, a[j], b[j]);
                o2[j] = t * a[j];
            } break;
            case V_CURV: {
                const double y = a[j] - b[j];
                o1[j] = y;
                r0 = fma(c[j], e[j], r0);
                r1 = fma(c[j], y, r1);
            } break;
            default: {
                const double y = fma(t, a[j], (1.0 - t) * b[j]);
                o1[j] = y;
                r0 = fma(y, c[j], r0);
            }
        }
    }
    if (op == V_DIR) publish(3, r0, r1, r2, 1, 0, 1, part, sc, 1);
    else if (op == V_CURV) publish(2, r0, r1, 0, 0, 0, 0, part, sc, 1);
    else if (op == V_DAMP) publish(1, r0, 0, 0, 0, 0, 0, part, sc, 1);
}

__global__ void k_diag_set(int n, int64_t ldh, const double *__restrict__ h0, double *__restrict__ H) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) H[(int64_t)j * ldh + j] = h0[j];
}

// x0 feasibility: bounds and l <= A x0 <= u (counts violations)
__global__ void k_feasible(int n, int m, const double *__restrict__ x, const double *__restrict__ xl,
                           const double *__restrict__ xu, const int64_t *__restrict__ rp, const int *__restrict__ col,
                           const double *__restrict__ val, const double *__restrict__ l, const double *__restrict__ u,
                           SqpScal *sc) {
    const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    int bad = 0;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        bad += !(x[j] >= xl[j] && x[j] <= xu[j]);
    for (int i = blockIdx.x * wpb + (threadIdx.x >> 5); i < m; i += gridDim.x * wpb) {
        double a = 0.0;
        for (int64_t k = rp[i] + lane; k < rp[i + 1]; k += 32) a = fma(val[k], x[col[k]], a);
        a = warp_sum(a);
        if (lane == 0) bad += !(a >= l[i] && a <= u[i]);
    }
    if (bad) atomicAdd(&sc->bad, (unsigned long long)bad);
}

thread_local std::string g_sqp_create_error;

struct Lay {
    size_t total = 0;
    size_t take(size_t b) {
        const size_t o = total;
        total += (b + 255) & ~size_t(255);
        return o;
    }
};

struct SqpPlan {
    size_t sc, vec[12], nd_e, part, h0, trp, tcol, tval, cnt, B, wq, zero, qp;
    int nchunk;
    int64_t ldh, ldu;
    size_t qp_bytes, total;
};

}  // namespace

struct ipm_sqp {
    cudaStream_t st = nullptr;
    ipm_sqp_options so{};
    ipm_options qo{};
    int64_t n = 0, m = 0, nd = 0, dnnz = 0;
    ipm_dose_nlp nlp{};
    ipm_problem cons{};
    char *ws = nullptr;
    SqpScal *sc = nullptr, *hsc = nullptr;
    double *x, *g, *gq, *d, *gn, *s, *y, *Bs, *yt, *Bx, *tmp, *e, *part, *h0, *B, *wq, *zero;
    int64_t *trp;
    int *tcol;
    double *tval;
    int64_t ldh = 0, ldu = 0;
    int ncols = 0;
    ipm_ctx *qp = nullptr;
    ipm_sqp_stats stats{};
    std::vector<ipm_sqp_trace_rec> trace;
    std::string err;
    int64_t launches = 0;
    bool have_x = false;
    bool dirty = false;          // a solve ran: B and the inner context must be reset
    char *qp_ws = nullptr;
    size_t qp_bytes = 0;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
};

namespace {

ipm_status sfail(ipm_sqp *c, ipm_status s, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    else g_sqp_create_error = buf;
    return s;
}

#define SCK(call)                                                                                     \
    do {                                                                                              \
        cudaError_t e_ = (call);                                                                      \
        if (e_ != cudaSuccess) return sfail(S, IPM_ERR_CUDA, "%s: %s (%s:%d)", #call,                 \
                                            cudaGetErrorString(e_), __FILE__, __LINE__);             \
    } while (0)
#define SCKL() SCK(cudaGetLastError())
#define QP(call)                                                                                      \
    do {                                                                                              \
        ipm_status s_ = (call);                                                                       \
        if (s_ != IPM_OK) return sfail(S, s_, "%s: %s", #call, ipm_last_error(S->qp));               \
    } while (0)

int64_t eff_cols(const ipm_sqp_options &o) { return o.max_cols > 0 ? o.max_cols : 2 * (int64_t)o.max_iter; }

ipm_problem qp_problem(const ipm_problem *c, const ipm_sqp_options &o) {
    ipm_problem q = *c;
    q.comm_kind = 0;
    q.nranks = 1;
    q.rank = 0;
    q.row_begin = 0;
    q.row_end = c->n;
    q.hess_kind = o.hess_kind;
    q.k = 0;
    q.ldh = c->n + (c->n & 1);
    q.ldu = o.hess_kind == 1 ? std::max<int64_t>(2, eff_cols(o)) : 0;
    return q;
}

SqpPlan plan(const ipm_problem *c, const ipm_dose_nlp *nlp, const ipm_sqp_options &o, const ipm_options *qo,
             ipm_status &st) {
    SqpPlan p{};
    Lay L;
    const int64_t n = c->n, nd = nlp->nd;
    p.sc = L.take(sizeof(SqpScal));
    for (auto &v : p.vec) v = L.take(sizeof(double) * (n + 2));
    p.nd_e = L.take(sizeof(double) * nd);
    p.part = L.take(sizeof(double) * 3 * kPart);
    p.h0 = L.take(sizeof(double) * n);
    p.trp = L.take(sizeof(int64_t) * (n + 1));
    p.tcol = L.take(sizeof(int) * std::max<int64_t>(1, nlp->nnz));
    p.tval = L.take(sizeof(double) * std::max<int64_t>(1, nlp->nnz));
    p.nchunk = (int)std::max<int64_t>(1, std::min<int64_t>(128, nd));
    p.cnt = L.take(sizeof(int) * (size_t)p.nchunk * n);
    p.ldh = n + (n & 1);
    p.ldu = o.hess_kind == 1 ? std::max<int64_t>(2, eff_cols(o)) : 0;
    p.B = (o.hess_kind == 1) ? L.take(sizeof(double) * n * p.ldu) : L.take(sizeof(double) * n * p.ldh);
    p.wq = L.take(sizeof(double) * std::max<int64_t>(2, p.ldu));
    p.zero = L.take(sizeof(double) * std::max<int64_t>(n, c->m) + 16);
    const ipm_problem q = qp_problem(c, o);
    size_t qb = 0;
    st = ipm_workspace_size(&q, qo, &qb);
    p.qp_bytes = qb;
    p.qp = L.take(qb);   // 256-aligned offset
    p.total = L.total;
    return p;
}

// f (and e, for the gradient) at x + t dir; result in S->sc->red[0] after a sync
void launch_f(ipm_sqp *S, const double *x, const double *dir, double t, int grad) {
    const int grid = sgrid(S->nd, kBlock / 32);
    const ipm_dose_nlp &N = S->nlp;
    if (grad)
        k_dose_f<1><<<grid, kBlock, 0, S->st>>>((int)S->nd, N.D_rowptr, N.D_col, N.D_val, x, dir, t, N.w, N.p, N.dmax,
                                               N.kappa, N.beta, S->e, S->part, S->sc);
    else
        k_dose_f<0><<<grid, kBlock, 0, S->st>>>((int)S->nd, N.D_rowptr, N.D_col, N.D_val, x, dir, t, N.w, N.p, N.dmax,
                                               N.kappa, N.beta, S->e, S->part, S->sc);
    S->launches += 1;
}

void launch_grad(ipm_sqp *S, double *out) {
    k_dose_t<0><<<sgrid(S->n, kBlock / 32), kBlock, 0, S->st>>>((int)S->n, S->trp, S->tcol, S->tval, S->e, 0.0, out);
    S->launches += 1;
}

void launch_vec(ipm_sqp *S, int op, const double *a, const double *b, const double *c, const double *e, double t,
                double *o1, double *o2) {
    k_sqp_vec<<<sgrid(S->n, kBlock), kBlock, 0, S->st>>>(op, (int)S->n, a, b, c, e, t, o1, o2, S->part, S->sc);
    S->launches += 1;
}

ipm_status sync(ipm_sqp *S) {
    SCKL();
    SCK(cudaMemcpyAsync(S->hsc, S->sc, sizeof(SqpScal), cudaMemcpyDeviceToHost, S->st));
    SCK(cudaStreamSynchronize(S->st));
    return IPM_OK;
}

// out = B v (the inner context's Hessian; Sigma = 0 makes its operator exactly H)
ipm_status apply_B(ipm_sqp *S, const double *v, double *out) {
    QP(ipm_op_apply(S->qp, S->zero, S->zero, v, out));
    return IPM_OK;
}

ipm_status eval_fg(ipm_sqp *S, const double *x, double *f, double *grad) {
    launch_f(S, x, nullptr, 0.0, grad != nullptr);
    if (grad) launch_grad(S, grad);
    if (sync(S) != IPM_OK) return IPM_ERR_CUDA;
    *f = S->hsc->red[0];
    return IPM_OK;
}

// the inner IPM context over the current B (g = S->gq, zero until the first subproblem)
ipm_status create_qp(ipm_sqp *S) {
    ipm_problem q = qp_problem(&S->cons, S->so);
    q.g = S->gq;
    if (S->so.hess_kind == 0) {
        q.H = S->B;
        q.ldh = S->ldh;
    } else {
        q.H = nullptr;
        q.h0 = S->h0;
        q.U = S->B;
        q.w = S->wq;
        q.k = 0;
    }
    const ipm_status s = ipm_create(&S->qp, &q, &S->qo, S->qp_ws, S->qp_bytes, S->st);
    if (s != IPM_OK) return sfail(S, s, "inner QP create: %s", ipm_last_error(nullptr));
    return IPM_OK;
}

ipm_status solve_impl(ipm_sqp *S, const double *x0) {
    const ipm_sqp_options &o = S->so;
    S->trace.clear();
    S->stats = ipm_sqp_stats{};
    ipm_sqp_stats &st = S->stats;
    SCK(cudaEventRecord(S->ev[0], S->st));
    // feasibility of x0 (R21: the line search keeps every iterate feasible)
    SCK(cudaMemsetAsync(&S->sc->bad, 0, sizeof(unsigned long long), S->st));
    k_feasible<<<sgrid(std::max(S->n, S->m * 32), kBlock), kBlock, 0, S->st>>>(
        (int)S->n, (int)S->m, x0, S->cons.xl, S->cons.xu, S->cons.A_rowptr, S->cons.A_col, S->cons.A_val, S->cons.l,
        S->cons.u, S->sc);
    S->launches += 1;
    if (sync(S) != IPM_OK) return IPM_ERR_CUDA;
    if (S->hsc->bad) return sfail(S, IPM_ERR_INVALID, "x0 violates %llu bounds / constraint rows", S->hsc->bad);
    SCK(cudaMemcpyAsync(S->x, x0, sizeof(double) * S->n, cudaMemcpyDeviceToDevice, S->st));
    S->have_x = true;
    double f = 0.0;
    if (eval_fg(S, S->x, &f, S->g) != IPM_OK) return IPM_ERR_CUDA;
    ipm_status status = IPM_NOT_CONVERGED;
    int k = 0;
    for (k = 0; k < o.max_iter; ++k) {
        // QP subproblem in x-space: linear term g_k - B_k x_k
        if (apply_B(S, S->x, S->Bx) != IPM_OK) return IPM_ERR_CUDA;
        launch_vec(S, V_GQ, S->g, S->Bx, nullptr, nullptr, 0.0, S->gq, nullptr);
        QP(ipm_set_linear_term(S->qp, S->gq));
        if (o.warm_start && k > 0) QP(ipm_warm_start(S->qp));
        const ipm_status qs = ipm_solve(S->qp);
        ipm_stats qst{};
        ipm_get_stats(S->qp, &qst);
        st.ipm_iters_total += qst.ipm_iters;
        st.pcg_iters_total += qst.pcg_iters_total;
        st.t_qp_ms += qst.t_solve_ms;
        if (qs != IPM_OK) {
            status = qs;
            sfail(S, qs, "QP subproblem %d: %s", k, ipm_last_error(S->qp));
            break;
        }
        QP(ipm_get_solution(S->qp, S->tmp, nullptr, nullptr, nullptr, nullptr, nullptr));
        launch_vec(S, V_DIR, S->tmp, S->x, S->g, nullptr, 0.0, S->d, nullptr);
        if (sync(S) != IPM_OK) return IPM_ERR_CUDA;
        const double dinf = S->hsc->red[0], gd = S->hsc->red[1], xinf = S->hsc->red[2];
        ipm_sqp_trace_rec rec{};
        rec.it = k;
        rec.ipm_iters = qst.ipm_iters;
        rec.pcg_iters = qst.pcg_iters_total;
        rec.f = f;
        rec.d_inf = dinf;
        rec.qp_ms = qst.t_solve_ms;
        rec.theta = 1.0;
        rec.ncols = S->ncols;
        st.d_inf = dinf;
        if (dinf <= o.tol_d * std::max(1.0, xinf)) {
            S->trace.push_back(rec);
            status = IPM_OK;
            break;
        }
        // Armijo backtracking on f along d (R21)
        double t = 1.0, ft = 0.0;
        int nb = 0;
        launch_f(S, S->x, S->d, t, 0);
        if (sync(S) != IPM_OK) return IPM_ERR_CUDA;
        ft = S->hsc->red[0];
        // written as !(ft <= ...) so a NaN trial value keeps backtracking instead of being accepted
        while (!(ft <= f + o.armijo_c1 * t * gd) && nb < o.max_backtrack) {
            t *= 0.5;
            ++nb;
            launch_f(S, S->x, S->d, t, 0);
            if (sync(S) != IPM_OK) return IPM_ERR_CUDA;
            ft = S->hsc->red[0];
        }
        st.backtracks += nb;
        if (!(ft <= f + o.armijo_c1 * t * gd)) {
            // no sufficient decrease within max_backtrack halvings: the step is NOT taken (the
            // merit function must not increase across accepted steps)
            status = std::isfinite(ft) ? IPM_NOT_CONVERGED : IPM_ERR_NONFINITE;
            sfail(S, status, "line search failed at SQP iteration %d (f(x + t d) = %g after %d halvings)", k, ft, nb);
            rec.step = 0.0;
            S->trace.push_back(rec);
            break;
        }
        // x_{k+1} = x + t d (same fma as the trial), s = t d; gradient at x_{k+1}
        launch_vec(S, V_STEP, S->d, S->x, nullptr, nullptr, t, S->tmp, S->s);
        std::swap(S->x, S->tmp);
        double fn = 0.0;
        if (eval_fg(S, S->x, &fn, S->gn) != IPM_OK) return IPM_ERR_CUDA;
        // BFGS with Powell damping
        if (apply_B(S, S->s, S->Bs) != IPM_OK) return IPM_ERR_CUDA;
        launch_vec(S, V_CURV, S->gn, S->g, S->s, S->Bs, 0.0, S->y, nullptr);
        if (sync(S) != IPM_OK) return IPM_ERR_CUDA;
        const double sBs = S->hsc->red[0], sy = S->hsc->red[1];
        bool updated = false;
        double theta = 1.0;
        if (sBs > 0.0) {
            theta = (sy >= o.powell * sBs) ? 1.0 : (1.0 - o.powell) * sBs / (sBs - sy);
            launch_vec(S, V_DAMP, S->y, S->Bs, S->s, nullptr, theta, S->yt, nullptr);
            if (sync(S) != IPM_OK) return IPM_ERR_CUDA;
            const double ys = S->hsc->red[0];
            const bool room = o.hess_kind == 0 || S->ncols + 2 <= S->ldu;
            if (ys > 0.0 && room) {
                QP(ipm_update_hessian_rank2(S->qp, S->Bs, -1.0 / sBs, S->yt, 1.0 / ys));
                S->ncols += 2;
                updated = true;
            }
        }
        if (!updated) st.updates_skipped += 1;
        rec.step = t;
        rec.theta = theta;
        rec.updated = updated ? 1 : 0;
        rec.ncols = S->ncols;
        S->trace.push_back(rec);
        std::swap(S->g, S->gn);
        f = fn;
    }
    st.status = status;
    st.iters = std::min(k + 1, o.max_iter);
    st.f = f;
    SCK(cudaEventRecord(S->ev[1], S->st));
    SCK(cudaEventSynchronize(S->ev[1]));
    float ms = 0.f;
    SCK(cudaEventElapsedTime(&ms, S->ev[0], S->ev[1]));
    st.t_total_ms = ms;
    return status;
}

}  // namespace

// ================================================================================= C ABI
IPM_EXPORT void ipm_sqp_options_default(ipm_sqp_options *o) {
    if (!o) return;
    std::memset(o, 0, sizeof *o);
    o->size = (int32_t)sizeof(ipm_sqp_options);
    o->max_iter = 50;
    o->tol_d = 1e-6;
    o->armijo_c1 = 1e-4;
    o->max_backtrack = 30;
    o->powell = 0.2;
    o->warm_start = 0;
    o->hess_kind = 0;
    o->max_cols = 0;
    o->h0_floor = 1e-3;
}

static ipm_status check_args(const ipm_problem *c, const ipm_dose_nlp *nlp, const ipm_sqp_options *so) {
    if (!c || !nlp || !so) return sfail(nullptr, IPM_ERR_INVALID, "null argument");
    if (so->size != (int32_t)sizeof(ipm_sqp_options)) return sfail(nullptr, IPM_ERR_INVALID, "ipm_sqp_options.size mismatch (ABI)");
    if (c->n < 1 || c->m < 0 || c->nnz < 0) return sfail(nullptr, IPM_ERR_INVALID, "bad constraint dimensions");
    if (c->comm_kind != 0 || c->nranks > 1) return sfail(nullptr, IPM_ERR_INVALID, "SQP driver is unsharded");
    if (nlp->nd < 1 || nlp->nnz < 0 || nlp->nd > INT32_MAX || nlp->nnz >= INT32_MAX)
        return sfail(nullptr, IPM_ERR_INVALID, "bad objective dimensions");
    if (!(nlp->beta > 0.0)) return sfail(nullptr, IPM_ERR_INVALID, "beta must be > 0");
    if (so->max_iter < 1 || so->hess_kind < 0 || so->hess_kind > 1 || so->max_cols < 0 || !(so->tol_d >= 0.0) ||
        !(so->powell >= 0.0 && so->powell < 1.0) || !(so->h0_floor > 0.0))
        return sfail(nullptr, IPM_ERR_INVALID, "bad SQP options");
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_sqp_workspace_size(const ipm_problem *c, const ipm_dose_nlp *nlp,
                                             const ipm_sqp_options *so, const ipm_options *qo, size_t *bytes) {
    ipm_sqp_options d;
    ipm_sqp_options_default(&d);
    if (!so) so = &d;
    if (!bytes) return sfail(nullptr, IPM_ERR_INVALID, "null argument");
    if (check_args(c, nlp, so) != IPM_OK) return IPM_ERR_INVALID;
    ipm_status st = IPM_OK;
    const SqpPlan p = plan(c, nlp, *so, qo, st);
    if (st != IPM_OK) return sfail(nullptr, st, "inner QP: %s", ipm_last_error(nullptr));
    *bytes = p.total;
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_sqp_create(ipm_sqp **out, const ipm_problem *c, const ipm_dose_nlp *nlp,
                                     const ipm_sqp_options *so_in, const ipm_options *qo, void *workspace,
                                     size_t workspace_bytes, ipm_stream_t stream) {
    if (!out) return sfail(nullptr, IPM_ERR_INVALID, "null argument");
    *out = nullptr;
    ipm_sqp_options so;
    ipm_sqp_options_default(&so);
    if (so_in) so = *so_in;
    if (check_args(c, nlp, &so) != IPM_OK) return IPM_ERR_INVALID;
    if (!nlp->D_rowptr || (nlp->nnz > 0 && (!nlp->D_col || !nlp->D_val)) || !nlp->w || !nlp->p || !nlp->dmax ||
        !nlp->kappa)
        return sfail(nullptr, IPM_ERR_INVALID, "null objective pointer");
    ipm_status pst = IPM_OK;
    const SqpPlan pl = plan(c, nlp, so, qo, pst);
    if (pst != IPM_OK) return sfail(nullptr, pst, "inner QP: %s", ipm_last_error(nullptr));
    if (!workspace || workspace_bytes < pl.total)
        return sfail(nullptr, IPM_ERR_OOM, "workspace too small: %zu < %zu bytes", workspace_bytes, pl.total);
    if (reinterpret_cast<uintptr_t>(workspace) & 255) return sfail(nullptr, IPM_ERR_INVALID, "workspace not 256-byte aligned");
    ipm_sqp *S = new ipm_sqp();
    S->st = reinterpret_cast<cudaStream_t>(stream);
    S->so = so;
    ipm_options_default(&S->qo);
    if (qo) S->qo = *qo;
    S->n = c->n;
    S->m = c->m;
    S->nd = nlp->nd;
    S->dnnz = nlp->nnz;
    S->nlp = *nlp;
    S->cons = *c;
    S->ws = reinterpret_cast<char *>(workspace);
    S->ldh = pl.ldh;
    S->ldu = pl.ldu;
    auto fin = [&](ipm_status s) {
        if (s != IPM_OK) {
            g_sqp_create_error = S->err;
            ipm_sqp_destroy(S);
            return s;
        }
        *out = S;
        return IPM_OK;
    };
    auto body = [&]() -> ipm_status {
        for (auto &e : S->ev) SCK(cudaEventCreate(&e));
        SCK(cudaMallocHost(&S->hsc, sizeof(SqpScal)));
        // host validation of D (O(nd + nnz) copies, once)
        std::vector<int64_t> rp(S->nd + 1);
        std::vector<int> col(S->dnnz);
        std::vector<double> val(S->dnnz), w(S->nd), kap(S->nd);
        SCK(cudaMemcpy(rp.data(), nlp->D_rowptr, sizeof(int64_t) * (S->nd + 1), cudaMemcpyDeviceToHost));
        if (S->dnnz) {
            SCK(cudaMemcpy(col.data(), nlp->D_col, sizeof(int) * S->dnnz, cudaMemcpyDeviceToHost));
            SCK(cudaMemcpy(val.data(), nlp->D_val, sizeof(double) * S->dnnz, cudaMemcpyDeviceToHost));
        }
        SCK(cudaMemcpy(w.data(), nlp->w, sizeof(double) * S->nd, cudaMemcpyDeviceToHost));
        SCK(cudaMemcpy(kap.data(), nlp->kappa, sizeof(double) * S->nd, cudaMemcpyDeviceToHost));
        if (rp[0] != 0 || rp[S->nd] != S->dnnz) return sfail(S, IPM_ERR_INVALID, "D_rowptr[0] must be 0 and D_rowptr[nd] == nnz");
        for (int64_t i = 0; i < S->nd; ++i) {
            if (rp[i + 1] < rp[i]) return sfail(S, IPM_ERR_INVALID, "D_rowptr decreasing at row %lld", (long long)i);
            for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
                if (col[k] < 0 || col[k] >= S->n || (k > rp[i] && col[k] <= col[k - 1]))
                    return sfail(S, IPM_ERR_INVALID, "D_col out of range or not increasing in row %lld", (long long)i);
            if (!(w[i] > 0.0) || !(kap[i] >= 0.0) || !std::isfinite(w[i]) || !std::isfinite(kap[i]))
                return sfail(S, IPM_ERR_INVALID, "w must be > 0 and kappa >= 0 (row %lld)", (long long)i);
        }
        for (double v : val)
            if (!std::isfinite(v)) return sfail(S, IPM_ERR_INVALID, "D_val has a non-finite entry");
        char *b = S->ws;
        SCK(cudaMemsetAsync(b, 0, pl.qp, S->st));
        S->sc = reinterpret_cast<SqpScal *>(b + pl.sc);
        double *v[12];
        for (int i = 0; i < 12; ++i) v[i] = reinterpret_cast<double *>(b + pl.vec[i]);
        S->x = v[0]; S->g = v[1]; S->gq = v[2]; S->d = v[3]; S->gn = v[4]; S->s = v[5];
        S->y = v[6]; S->Bs = v[7]; S->yt = v[8]; S->Bx = v[9]; S->tmp = v[10];
        S->e = reinterpret_cast<double *>(b + pl.nd_e);
        S->part = reinterpret_cast<double *>(b + pl.part);
        S->h0 = reinterpret_cast<double *>(b + pl.h0);
        S->trp = reinterpret_cast<int64_t *>(b + pl.trp);
        S->tcol = reinterpret_cast<int *>(b + pl.tcol);
        S->tval = reinterpret_cast<double *>(b + pl.tval);
        S->B = reinterpret_cast<double *>(b + pl.B);
        S->wq = reinterpret_cast<double *>(b + pl.wq);
        S->zero = reinterpret_cast<double *>(b + pl.zero);
        // D^T by the IPM's deterministic counting sort (rows of D^T = variables)
        Prob Q{};
        Q.n = (int)S->n;
        Q.m = (int)S->nd;
        Q.ncols = (int)S->n;
        Q.nnz = S->dnnz;
        Q.Arp = nlp->D_rowptr;
        Q.Acol = nlp->D_col;
        Q.Aval = nlp->D_val;
        launch_transpose(Q, 0, pl.nchunk, reinterpret_cast<int *>(b + pl.cnt), S->trp, S->tcol, S->tval, S->st);
        // h0 = diag(D^T W D) + floor (R20); B_0 = diag(h0)
        k_dose_t<1><<<sgrid(S->n, kBlock / 32), kBlock, 0, S->st>>>((int)S->n, S->trp, S->tcol, S->tval, nlp->w,
                                                                    so.h0_floor, S->h0);
        if (so.hess_kind == 0)
            k_diag_set<<<sgrid(S->n, kBlock), kBlock, 0, S->st>>>((int)S->n, S->ldh, S->h0, S->B);
        S->launches += 5;
        SCKL();
        S->qp_ws = b + pl.qp;
        S->qp_bytes = pl.qp_bytes;
        SCK(cudaStreamSynchronize(S->st));
        return create_qp(S);
    };
    return fin(body());
}

IPM_EXPORT ipm_status ipm_sqp_solve(ipm_sqp *S, const double *x0) {
    if (!S || !x0) return sfail(S, IPM_ERR_INVALID, "null argument");
    S->err.clear();
    if (S->dirty) {
        // restart from B_0: dense B back to diag(h0) / compact columns dropped, and a fresh
        // inner context (its cached diag(H), column count and graphs restart with it)
        ipm_destroy(S->qp);
        S->qp = nullptr;
        S->ncols = 0;
        if (S->so.hess_kind == 0) {
            SCK(cudaMemsetAsync(S->B, 0, sizeof(double) * S->n * S->ldh, S->st));
            k_diag_set<<<sgrid(S->n, kBlock), kBlock, 0, S->st>>>((int)S->n, S->ldh, S->h0, S->B);
            S->launches += 1;
            SCKL();
        }
        SCK(cudaMemsetAsync(S->gq, 0, sizeof(double) * S->n, S->st));
        SCK(cudaStreamSynchronize(S->st));
        const ipm_status s = create_qp(S);
        if (s != IPM_OK) return s;
    }
    S->dirty = true;
    return solve_impl(S, x0);
}

IPM_EXPORT ipm_status ipm_sqp_get_x(ipm_sqp *S, double *x) {
    if (!S || !x) return sfail(S, IPM_ERR_INVALID, "null argument");
    if (!S->have_x) return sfail(S, IPM_ERR_STATE, "no iterate: call ipm_sqp_solve first");
    SCK(cudaMemcpyAsync(x, S->x, sizeof(double) * S->n, cudaMemcpyDeviceToDevice, S->st));
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_sqp_get_stats(ipm_sqp *S, ipm_sqp_stats *st) {
    if (!S || !st) return sfail(S, IPM_ERR_INVALID, "null argument");
    *st = S->stats;
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_sqp_get_trace(ipm_sqp *S, ipm_sqp_trace_rec *recs, int32_t cap, int32_t *count) {
    if (!S || !count) return sfail(S, IPM_ERR_INVALID, "null argument");
    const int32_t nrec = (int32_t)S->trace.size();
    *count = nrec;
    if (recs)
        for (int32_t i = 0; i < std::min(cap, nrec); ++i) recs[i] = S->trace[i];
    return IPM_OK;
}

IPM_EXPORT ipm_status ipm_sqp_eval(ipm_sqp *S, const double *x, double *f_host, double *grad) {
    if (!S || !x || !f_host) return sfail(S, IPM_ERR_INVALID, "null argument");
    return eval_fg(S, x, f_host, grad);
}

IPM_EXPORT ipm_ctx *ipm_sqp_qp(ipm_sqp *S) { return S ? S->qp : nullptr; }

IPM_EXPORT int64_t ipm_sqp_kernel_launches(const ipm_sqp *S) {
    return S ? S->launches + (S->qp ? ipm_kernel_launches(S->qp) : 0) : 0;
}

IPM_EXPORT const char *ipm_sqp_last_error(const ipm_sqp *S) { return S ? S->err.c_str() : g_sqp_create_error.c_str(); }

IPM_EXPORT void ipm_sqp_destroy(ipm_sqp *S) {
    if (!S) return;
    if (S->st) cudaStreamSynchronize(S->st);
    if (S->qp) ipm_destroy(S->qp);
    for (auto &e : S->ev)
        if (e) cudaEventDestroy(e);
    if (S->hsc) cudaFreeHost(S->hsc);
    delete S;
}
