// ipmops.cu — per-IPM-iteration kernels around the PCG solve (Alg. 1 lines 3-9).
//
// Layout: masked full-length families.  m-vectors carry the row families lA
// (l finite) and uA (u finite), n-vectors the variable families lx (xl finite) and ux
// (xu finite); entries of an absent family are kept at exactly 0 and never enter a sum,
// a min or a max.  Formulas:
//   residuals (eq:perturbed_KKT, reading R1 for the r_u sign)
//     r_H  = H x + g - A^T (lam_lA - lam_uA) - lam_lx + lam_ux
//     r_lA = A x - s_lA - l,  r_uA = u - A x - s_uA,  r_lx = x - s_lx - xl,  r_ux = xu - x - s_ux
//     r_c  = lam o s - mu
//   diagonals   Sigma_b = lam_lx/s_lx + lam_ux/s_ux,  Sigma_c = lam_lA/s_lA + lam_uA/s_uA
//   condensed rhs (eq:2x2_reduced + Schur complement)
//     r1 = -r_H - (r_c,lx + lam_lx r_lx)/s_lx + (r_c,ux + lam_ux r_ux)/s_ux
//     r2_l = -r_lA - r_c,lA/lam_lA,  r2_u = -r_uA - r_c,uA/lam_uA,  w = r2_l/D_l - r2_u/D_u
//     rhs = r1 + A^T w
//   recovery (Alg. 1 line 3): dlam_A = D^-1 (r2 - B dx), ds_lA = A dx + r_lA, ds_uA = -A dx + r_uA,
//     ds_lx = dx + r_lx, ds_ux = -dx + r_ux, dlam_x = -(r_c + lam ds)/s
//   step lengths (Alg. 1 line 4): alpha = min(1, tau * min{-v/dv : dv < 0})
//   update (Alg. 1 lines 5-7): x, s += alpha_x d;  lam += alpha_lam d
#include "common.cuh"
#include "kernels.h"
#include "state.h"
#include "finalize.cuh"

namespace ipm {

__device__ __forceinline__ bool has(double b) { return fabs(b) < INFINITY; }

static int grid_for(int64_t units, int per_block) {
    int64_t g = (units + per_block - 1) / per_block;
    if (g < 1) g = 1;
    if (g > kMaxGrid) g = kMaxGrid;
    return (int)g;
}

// ------------------------------------------------------------------ initial point (R5 / R15)
__global__ void k_init_x(int n, const double *__restrict__ xl, const double *__restrict__ xu, double *__restrict__ x,
                         int warm, double theta) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const double lo = xl[j], hi = xu[j];
        const bool hl = has(lo), hu = has(hi);
        double v;
        if (!warm) {
            if (hl && hu) {
                const double delta = fmin(1.0, (hi - lo) / 4.0);
                v = fmin(fmax(0.0, lo + delta), hi - delta);
            } else if (hl) {
                v = fmax(0.0, lo + 1.0);
            } else if (hu) {
                v = fmin(0.0, hi - 1.0);
            } else {
                v = 0.0;
            }
        } else {
            v = x[j];
            const double mlo = (hl && hu) ? fmin(theta, (hi - lo) / 4.0) : theta;
            if (hl) v = fmax(v, lo + mlo);
            if (hu) v = fmin(v, hi - mlo);
        }
        x[j] = v;
    }
}

void launch_init_x(const Prob &P, const Vecs &V, int warm, double theta, cudaStream_t st) {
    if (P.n == 0) return;
    k_init_x<<<grid_for(P.n, kBlock), kBlock, 0, st>>>(P.n, P.xl, P.xu, V.x, warm, theta);
}

// slacks = max(gap, floor); multipliers = 1 (cold) or max(lam_prev, theta) (warm); sum lam*s.
__global__ void __launch_bounds__(kBlock)
k_init_slacks(int len, const double *__restrict__ lo, const double *__restrict__ hi, const double *__restrict__ v,
              double *__restrict__ s_l, double *__restrict__ s_u, double *__restrict__ lam_l, double *__restrict__ lam_u,
              int warm, double theta, double *__restrict__ dpart, Scalars *sc, int cid, int final_) {
    __shared__ double red[kBlock / 32];
    const double floor_ = warm ? theta : 1.0;
    double acc = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) {
        const double vi = v[i];
        if (has(lo[i])) {
            const double s = fmax(vi - lo[i], floor_);
            const double l = warm ? fmax(lam_l[i], theta) : 1.0;
            s_l[i] = s;
            lam_l[i] = l;
            acc = fma(l, s, acc);
        } else {
            s_l[i] = 0.0;
            lam_l[i] = 0.0;
        }
        if (has(hi[i])) {
            const double s = fmax(hi[i] - vi, floor_);
            const double l = warm ? fmax(lam_u[i], theta) : 1.0;
            s_u[i] = s;
            lam_u[i] = l;
            acc = fma(l, s, acc);
        } else {
            s_u[i] = 0.0;
            lam_u[i] = 0.0;
        }
    }
    const double b = block_sum(acc, red);
    if (threadIdx.x == 0) dpart[blockIdx.x] = b;
    if (last_block(&sc->counters[cid])) {
        const double t = sum_partials(dpart, gridDim.x, red);
        if (threadIdx.x == 0) {
            sc->counters[cid] = 0;
            if (final_) { sc->sum_ls = sc->sum_ls_m + t; sc->loc[5] = t; }
            else sc->sum_ls_m = t;
        }
    }
}

void launch_init_slacks(const Prob &P, const Vecs &V, Scalars *sc, int warm, double theta, cudaStream_t st) {
    cudaMemsetAsync(&sc->sum_ls_m, 0, sizeof(double), st);
    if (P.m > 0)
        k_init_slacks<<<grid_for(P.m, kBlock), kBlock, 0, st>>>(P.m, P.l, P.u, V.Ax, V.s_lA, V.s_uA, V.lam_lA, V.lam_uA,
                                                               warm, theta, V.part[0], sc, C_INIT_M, 0);
    k_init_slacks<<<grid_for(P.n, kBlock), kBlock, 0, st>>>(P.n, P.xl, P.xu, V.x, V.s_lx, V.s_ux, V.lam_lx, V.lam_ux,
                                                           warm, theta, V.part[1], sc, C_INIT_N, 1);
}

// sum lam*s over all families (mu for Mehrotra / warm starts)
__global__ void __launch_bounds__(kBlock)
k_sum_ls(int len, const double *__restrict__ s1, const double *__restrict__ l1, const double *__restrict__ s2,
         const double *__restrict__ l2, double *__restrict__ dpart, Scalars *sc, int cid, int final_) {
    __shared__ double red[kBlock / 32];
    double acc = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) {
        acc = fma(l1[i], s1[i], acc);
        acc = fma(l2[i], s2[i], acc);
    }
    const double b = block_sum(acc, red);
    if (threadIdx.x == 0) dpart[blockIdx.x] = b;
    if (last_block(&sc->counters[cid])) {
        const double t = sum_partials(dpart, gridDim.x, red);
        if (threadIdx.x == 0) {
            sc->counters[cid] = 0;
            if (final_) { sc->sum_ls = sc->sum_ls_m + t; sc->loc[5] = t; }
            else sc->sum_ls_m = t;
        }
    }
}

void launch_sum_ls(const Prob &P, const Vecs &V, Scalars *sc, cudaStream_t st) {
    cudaMemsetAsync(&sc->sum_ls_m, 0, sizeof(double), st);
    if (P.m > 0)
        k_sum_ls<<<grid_for(P.m, kBlock), kBlock, 0, st>>>(P.m, V.s_lA, V.lam_lA, V.s_uA, V.lam_uA, V.part[0], sc, C_LS_M, 0);
    k_sum_ls<<<grid_for(P.n, kBlock), kBlock, 0, st>>>(P.n, V.s_lx, V.lam_lx, V.s_ux, V.lam_ux, V.part[1], sc, C_LS_N, 1);
}

// ------------------------------------------------------------------------------ residuals
// m-part: r_lA, r_uA, lamd = lam_lA - lam_uA; maxima of |primal|, |lam s - mu|, lam s.
__global__ void __launch_bounds__(kBlock)
k_resid_m(int m, const double *__restrict__ l, const double *__restrict__ u, const double *__restrict__ Ax,
          const double *__restrict__ s_l, const double *__restrict__ s_u, const double *__restrict__ lam_l,
          const double *__restrict__ lam_u, double *__restrict__ r_l, double *__restrict__ r_u,
          double *__restrict__ lamd, double mu, double *__restrict__ p1, double *__restrict__ p2,
          double *__restrict__ p3, Scalars *sc) {
    __shared__ double red[kBlock / 32];
    double prim = 0.0, comp = 0.0, lsm = 0.0;
    int bad = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        const double ax = Ax[i];
        double rl = 0.0, ru = 0.0;
        if (has(l[i])) {
            rl = ax - s_l[i] - l[i];
            const double ls = lam_l[i] * s_l[i];
            prim = fmax(prim, fabs(rl));
            comp = fmax(comp, fabs(ls - mu));
            lsm = fmax(lsm, ls);
            bad |= !finite_d(rl) | !finite_d(ls);
        }
        if (has(u[i])) {
            ru = u[i] - ax - s_u[i];
            const double ls = lam_u[i] * s_u[i];
            prim = fmax(prim, fabs(ru));
            comp = fmax(comp, fabs(ls - mu));
            lsm = fmax(lsm, ls);
            bad |= !finite_d(ru) | !finite_d(ls);
        }
        r_l[i] = rl;
        r_u[i] = ru;
        lamd[i] = lam_l[i] - lam_u[i];
    }
    if (bad) sc->nonfinite = 1;
    const double a = block_max(prim, red);
    const double b = block_max(comp, red);
    const double c = block_max(lsm, red);
    if (threadIdx.x == 0) {
        p1[blockIdx.x] = a;
        p2[blockIdx.x] = b;
        p3[blockIdx.x] = c;
    }
    if (last_block(&sc->counters[C_RES_M])) {
        const double ta = max_partials(p1, gridDim.x, red);
        const double tb = max_partials(p2, gridDim.x, red);
        const double tc = max_partials(p3, gridDim.x, red);
        if (threadIdx.x == 0) {
            sc->counters[C_RES_M] = 0;
            sc->prim_max_m = ta;
            sc->comp_max_m = tb;
            sc->ls_max_m = tc;
        }
    }
}

// n-part, G lanes per variable: Hx from the GEMV tile partials, A^T lamd through the stored
// transpose, then r_H, r_lx, r_ux, maxima and the objective 1/2 x^T H x + g^T x.
template <int G>
__global__ void __launch_bounds__(kBlock)
k_resid_n(int n, int ncb, const double *__restrict__ ypart, const int64_t *__restrict__ ATrp,
          const int *__restrict__ ATcol, const double *__restrict__ ATval, const double *__restrict__ lamd,
          const double *__restrict__ x, const double *__restrict__ g, const double *__restrict__ xl,
          const double *__restrict__ xu, const double *__restrict__ s_l, const double *__restrict__ s_u,
          const double *__restrict__ lam_l, const double *__restrict__ lam_u, double *__restrict__ Hx,
          double *__restrict__ rH, double *__restrict__ r_l, double *__restrict__ r_u, double mu,
          double *__restrict__ p1, double *__restrict__ p2, double *__restrict__ p3, double *__restrict__ p4,
          double *__restrict__ p5, Scalars *sc) {
    __shared__ double red[kBlock / 32];
    const int gl = threadIdx.x & (G - 1);
    const int gpb = blockDim.x / G;
    double rhm = 0.0, prim = 0.0, comp = 0.0, lsm = 0.0, obj = 0.0;
    int bad = 0;
    // warp-uniform trip count: every lane reaches the group shuffles (full-mask __shfl_sync)
    for (int gb_ = blockIdx.x * gpb + (int)(threadIdx.x & ~31u) / G; gb_ < n; gb_ += gridDim.x * gpb) {
        const bool act = gb_ + (int)(threadIdx.x & 31u) / G < n;
        const int j = act ? gb_ + (int)(threadIdx.x & 31u) / G : n - 1;   // idle lanes re-read row n-1, write nothing
        double hs = 0.0, at = 0.0;
        hs += row_part_sum<G>(ypart + (int64_t)j * ncb, gl, ncb);
        if (lamd != nullptr) {
            const int64_t e = ATrp[j + 1];
            for (int64_t k = ATrp[j] + gl; k < e; k += G) at = fma(__ldg(ATval + k), __ldg(lamd + __ldg(ATcol + k)), at);
        }
        hs = group_sum<G>(hs);
        at = group_sum<G>(at);
        if (act && gl == 0) {
            const double xj = x[j];
            Hx[j] = hs;
            const double rh = hs + g[j] - at - lam_l[j] + lam_u[j];
            rH[j] = rh;
            rhm = fmax(rhm, fabs(rh));
            bad |= !finite_d(rh);
            obj = fma(0.5 * xj, hs, obj);
            obj = fma(g[j], xj, obj);
            double rl = 0.0, ru = 0.0;
            if (has(xl[j])) {
                rl = xj - s_l[j] - xl[j];
                const double ls = lam_l[j] * s_l[j];
                prim = fmax(prim, fabs(rl));
                comp = fmax(comp, fabs(ls - mu));
                lsm = fmax(lsm, ls);
                bad |= !finite_d(rl) | !finite_d(ls);
            }
            if (has(xu[j])) {
                ru = xu[j] - xj - s_u[j];
                const double ls = lam_u[j] * s_u[j];
                prim = fmax(prim, fabs(ru));
                comp = fmax(comp, fabs(ls - mu));
                lsm = fmax(lsm, ls);
                bad |= !finite_d(ru) | !finite_d(ls);
            }
            r_l[j] = rl;
            r_u[j] = ru;
        }
    }
    if (bad) sc->nonfinite = 1;
    const double a = block_max(rhm, red);
    const double b = block_max(prim, red);
    const double c = block_max(comp, red);
    const double d = block_max(lsm, red);
    const double e = block_sum(obj, red);
    if (threadIdx.x == 0) {
        p1[blockIdx.x] = a;
        p2[blockIdx.x] = b;
        p3[blockIdx.x] = c;
        p4[blockIdx.x] = d;
        p5[blockIdx.x] = e;
    }
    if (last_block(&sc->counters[C_RES_N])) {
        const double ta = max_partials(p1, gridDim.x, red);
        const double tb = max_partials(p2, gridDim.x, red);
        const double tc = max_partials(p3, gridDim.x, red);
        const double td = max_partials(p4, gridDim.x, red);
        const double te = sum_partials(p5, gridDim.x, red);
        if (threadIdx.x == 0) {
            sc->counters[C_RES_N] = 0;
            if (sc->sharded) {
                sc->loc[0] = ta; sc->loc[1] = tb; sc->loc[2] = tc; sc->loc[3] = td; sc->loc[4] = te;
                sc->loc[6] = (double)sc->nonfinite;
            } else {
                fin_resid(sc, ta, tb, tc, td, te);
            }
        }
    }
}

#define IPM_DISPATCH_G(G, ...)                                  \
    switch (G) {                                                \
        case 4: { constexpr int GG = 4; __VA_ARGS__; } break;   \
        case 8: { constexpr int GG = 8; __VA_ARGS__; } break;   \
        case 16: { constexpr int GG = 16; __VA_ARGS__; } break; \
        default: { constexpr int GG = 32; __VA_ARGS__; } break; \
    }

// Requires: V.ypart holds the GEMV tiles of H x and V.Ax = A x (launched by the caller).
void launch_residuals(const Prob &P, const Vecs &V, int G, Scalars *sc, double mu, cudaStream_t st) {
    const int ncb = P.ncb;
    cudaMemsetAsync(&sc->prim_max_m, 0, 3 * sizeof(double) * 2, st);   // *_max_m and neighbours
    if (P.m > 0)
        k_resid_m<<<grid_for(P.m, kBlock), kBlock, 0, st>>>(P.m, P.l, P.u, V.Ax, V.s_lA, V.s_uA, V.lam_lA, V.lam_uA,
                                                           V.r_lA, V.r_uA, V.lamd, mu, V.part[0], V.part[1],
                                                           V.part[2], sc);
    const double *lamd = (P.m > 0) ? V.lamd : nullptr;
    const int grid = grid_for(P.n, kBlock / G);
    IPM_DISPATCH_G(G, (k_resid_n<GG><<<grid, kBlock, 0, st>>>(P.n, ncb, V.ypart, P.ATrp, P.ATcol, P.ATval, lamd, V.x, P.g,
                                                              P.xl, P.xu, V.s_lx, V.s_ux, V.lam_lx, V.lam_ux, V.Hx, V.rH,
                                                              V.r_lx, V.r_ux, mu, V.part[3], V.part[4], V.part[5],
                                                              V.part[6], V.part[7], sc)));
}

// ------------------------------------------------------------------ diagonals + Jacobi
__global__ void k_sigma_m(int m, const double *__restrict__ l, const double *__restrict__ u,
                          const double *__restrict__ s_l, const double *__restrict__ s_u,
                          const double *__restrict__ lam_l, const double *__restrict__ lam_u,
                          double *__restrict__ sigc, int aug, double *__restrict__ Dl, double *__restrict__ Du,
                          double *__restrict__ Ml, double *__restrict__ Mu) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        double s = 0.0;
        const bool hl = has(l[i]), hu = has(u[i]);
        if (hl) s += lam_l[i] / s_l[i];
        if (hu) s += lam_u[i] / s_u[i];
        sigc[i] = s;
        if (aug) {   // eq:2x2_augmented: D = S Lam^-1 on the middle rows, Jacobi 1/D (0 on absent rows,
                     // which keeps their z, p and dlam at exactly 0)
            Dl[i] = hl ? s_l[i] / lam_l[i] : 0.0;
            Du[i] = hu ? s_u[i] / lam_u[i] : 0.0;
            Ml[i] = hl ? lam_l[i] / s_l[i] : 0.0;
            Mu[i] = hu ? lam_u[i] / s_u[i] : 0.0;
        }
    }
}

template <int G>
__global__ void __launch_bounds__(kBlock)
k_sigma_n_jacobi(int n, const double *__restrict__ xl, const double *__restrict__ xu, const double *__restrict__ s_l,
                 const double *__restrict__ s_u, const double *__restrict__ lam_l, const double *__restrict__ lam_u,
                 const double *__restrict__ diagH, const int64_t *__restrict__ ATrp, const int *__restrict__ ATcol,
                 const double *__restrict__ ATval, const double *__restrict__ sigc, double *__restrict__ sigb,
                 double *__restrict__ Minv, double cfac) {
    const int gl = threadIdx.x & (G - 1);
    const int gpb = blockDim.x / G;
    // warp-uniform trip count: every lane reaches the group shuffles (full-mask __shfl_sync)
    for (int gb_ = blockIdx.x * gpb + (int)(threadIdx.x & ~31u) / G; gb_ < n; gb_ += gridDim.x * gpb) {
        const bool act = gb_ + (int)(threadIdx.x & 31u) / G < n;
        const int j = act ? gb_ + (int)(threadIdx.x & 31u) / G : n - 1;   // idle lanes re-read row n-1, write nothing
        double s = 0.0;
        if (sigc != nullptr) {
            const int64_t e = ATrp[j + 1];
            for (int64_t k = ATrp[j] + gl; k < e; k += G) {
                const double a = __ldg(ATval + k);
                s = fma(a * a, __ldg(sigc + __ldg(ATcol + k)), s);
            }
        }
        s = group_sum<G>(s);
        if (act && gl == 0) {
            double sb = 0.0;
            if (has(xl[j])) sb += lam_l[j] / s_l[j];
            if (has(xu[j])) sb += lam_u[j] / s_u[j];
            sigb[j] = sb;
            Minv[j] = 1.0 / (diagH[j] + sb + cfac * s);   // cfac = 2 on the augmented top block
        }
    }
}

void launch_sigma(const Prob &P, const Vecs &V, int G, cudaStream_t st) {
    if (P.m > 0)
        k_sigma_m<<<grid_for(P.m, kBlock), kBlock, 0, st>>>(P.m, P.l, P.u, V.s_lA, V.s_uA, V.lam_lA, V.lam_uA, V.sig_c,
                                                           P.aug, V.ag.Dl, V.ag.Du, V.ag.Ml, V.ag.Mu);
    const double *sigc = (P.m > 0) ? V.sig_c : nullptr;
    const int grid = grid_for(P.n, kBlock / G);
    IPM_DISPATCH_G(G, (k_sigma_n_jacobi<GG><<<grid, kBlock, 0, st>>>(P.n, P.xl, P.xu, V.s_lx, V.s_ux, V.lam_lx, V.lam_ux,
                                                                     P.diagH, P.ATrp, P.ATcol, P.ATval, sigc, V.sig_b,
                                                                     V.Minv, P.aug ? 2.0 : 1.0)));
}

// ------------------------------------------------------------------------------ RHS
// mode 0: r_c = lam s - mu (Alg. 1);  1: r_c = lam s (Mehrotra affine);
// mode 2: r_c = lam s + dlam_aff ds_aff - sigma_mu (Mehrotra corrector).
__device__ __forceinline__ double rc_of(double lam, double s, double adl, double ads, double mu, int mode,
                                        double smu) {
    if (mode == 0) return lam * s - mu;
    if (mode == 1) return lam * s;
    return fma(adl, ads, lam * s) - smu;
}

__global__ void k_rhs_m(int m, const double *__restrict__ l, const double *__restrict__ u, const double *__restrict__ s_l,
                        const double *__restrict__ s_u, const double *__restrict__ lam_l, const double *__restrict__ lam_u,
                        const double *__restrict__ r_l, const double *__restrict__ r_u, const double *__restrict__ adl_l,
                        const double *__restrict__ ads_l, const double *__restrict__ adl_u, const double *__restrict__ ads_u,
                        double *__restrict__ rc_l, double *__restrict__ rc_u, double *__restrict__ r2_l,
                        double *__restrict__ r2_u, double *__restrict__ w, double mu, int mode, double smu) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        double wi = 0.0, a = 0.0, b = 0.0, ca = 0.0, cb = 0.0;
        if (has(l[i])) {
            const double lam = lam_l[i], s = s_l[i];
            ca = rc_of(lam, s, mode == 2 ? adl_l[i] : 0.0, mode == 2 ? ads_l[i] : 0.0, mu, mode, smu);
            a = -r_l[i] - ca / lam;
            wi += a / (s / lam);
        }
        if (has(u[i])) {
            const double lam = lam_u[i], s = s_u[i];
            cb = rc_of(lam, s, mode == 2 ? adl_u[i] : 0.0, mode == 2 ? ads_u[i] : 0.0, mu, mode, smu);
            b = -r_u[i] - cb / lam;
            wi -= b / (s / lam);
        }
        rc_l[i] = ca;
        rc_u[i] = cb;
        r2_l[i] = a;
        r2_u[i] = b;
        w[i] = wi;
    }
}

template <int G>
__global__ void __launch_bounds__(kBlock)
k_rhs_n(int n, const double *__restrict__ xl, const double *__restrict__ xu, const double *__restrict__ s_l,
        const double *__restrict__ s_u, const double *__restrict__ lam_l, const double *__restrict__ lam_u,
        const double *__restrict__ r_l, const double *__restrict__ r_u, const double *__restrict__ rH,
        const double *__restrict__ adl_l, const double *__restrict__ ads_l, const double *__restrict__ adl_u,
        const double *__restrict__ ads_u, double *__restrict__ rc_l, double *__restrict__ rc_u,
        const int64_t *__restrict__ ATrp, const int *__restrict__ ATcol, const double *__restrict__ ATval,
        const double *__restrict__ w, double *__restrict__ rhs, double mu, int mode, double smu, double wfac) {
    const int gl = threadIdx.x & (G - 1);
    const int gpb = blockDim.x / G;
    // warp-uniform trip count: every lane reaches the group shuffles (full-mask __shfl_sync)
    for (int gb_ = blockIdx.x * gpb + (int)(threadIdx.x & ~31u) / G; gb_ < n; gb_ += gridDim.x * gpb) {
        const bool act = gb_ + (int)(threadIdx.x & 31u) / G < n;
        const int j = act ? gb_ + (int)(threadIdx.x & 31u) / G : n - 1;   // idle lanes re-read row n-1, write nothing
        double at = 0.0;
        if (w != nullptr) {
            const int64_t e = ATrp[j + 1];
            for (int64_t k = ATrp[j] + gl; k < e; k += G) at = fma(__ldg(ATval + k), __ldg(w + __ldg(ATcol + k)), at);
        }
        at = group_sum<G>(at);
        if (act && gl == 0) {
            double r1 = -rH[j];
            double ca = 0.0, cb = 0.0;
            if (has(xl[j])) {
                const double lam = lam_l[j], s = s_l[j];
                ca = rc_of(lam, s, mode == 2 ? adl_l[j] : 0.0, mode == 2 ? ads_l[j] : 0.0, mu, mode, smu);
                r1 -= fma(lam, r_l[j], ca) / s;
            }
            if (has(xu[j])) {
                const double lam = lam_u[j], s = s_u[j];
                cb = rc_of(lam, s, mode == 2 ? adl_u[j] : 0.0, mode == 2 ? ads_u[j] : 0.0, mu, mode, smu);
                r1 += fma(lam, r_u[j], cb) / s;
            }
            rc_l[j] = ca;
            rc_u[j] = cb;
            rhs[j] = fma(wfac, at, r1);   // wfac = 2: top block r1 + 2 B^T D^-1 r2 of eq:2x2_augmented
        }
    }
}

void launch_rhs(const Prob &P, const Vecs &V, int G, double mu, int mode, double sigma_mu, cudaStream_t st) {
    if (P.m > 0)
        k_rhs_m<<<grid_for(P.m, kBlock), kBlock, 0, st>>>(P.m, P.l, P.u, V.s_lA, V.s_uA, V.lam_lA, V.lam_uA, V.r_lA,
                                                         V.r_uA, V.adl_lA, V.ads_lA, V.adl_uA, V.ads_uA, V.rc_lA,
                                                         V.rc_uA, V.r2_l, V.r2_u, V.w, mu, mode, sigma_mu);
    const double *w = (P.m > 0) ? V.w : nullptr;
    const int grid = grid_for(P.n, kBlock / G);
    IPM_DISPATCH_G(G, (k_rhs_n<GG><<<grid, kBlock, 0, st>>>(P.n, P.xl, P.xu, V.s_lx, V.s_ux, V.lam_lx, V.lam_ux, V.r_lx,
                                                            V.r_ux, V.rH, V.adl_lx, V.ads_lx, V.adl_ux, V.ads_ux,
                                                            V.rc_lx, V.rc_ux, P.ATrp, P.ATcol, P.ATval, w, V.rhs, mu,
                                                            mode, sigma_mu, P.aug ? 2.0 : 1.0)));
}

// ------------------------------------------------------------- recovery + step lengths
__device__ __forceinline__ void ratio_min(double v, double dv, double &mn) {
    if (dv < 0.0) mn = fmin(mn, -v / dv);
}

__global__ void __launch_bounds__(kBlock)
k_recover_m(int m, const double *__restrict__ l, const double *__restrict__ u, const double *__restrict__ Adx,
            const double *__restrict__ r_l, const double *__restrict__ r_u, const double *__restrict__ r2_l,
            const double *__restrict__ r2_u, const double *__restrict__ s_l, const double *__restrict__ s_u,
            const double *__restrict__ lam_l, const double *__restrict__ lam_u, double *__restrict__ ds_l,
            double *__restrict__ ds_u, double *__restrict__ dl_l, double *__restrict__ dl_u,
            double *__restrict__ p1, double *__restrict__ p2, Scalars *sc, const double *__restrict__ aug_dl,
            const double *__restrict__ aug_du) {
    __shared__ double red[kBlock / 32];
    double mx = INFINITY, ml = INFINITY;
    int bad = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        const double a = Adx[i];
        double dsl = 0.0, dll = 0.0, dsu = 0.0, dlu = 0.0;
        if (has(l[i])) {
            dsl = a + r_l[i];
            dll = aug_dl ? aug_dl[i] : (r2_l[i] - a) / (s_l[i] / lam_l[i]);   // augmented: PCG's dlam
            ratio_min(s_l[i], dsl, mx);
            ratio_min(lam_l[i], dll, ml);
            bad |= !finite_d(dsl) | !finite_d(dll);
        }
        if (has(u[i])) {
            dsu = -a + r_u[i];
            dlu = aug_du ? aug_du[i] : (r2_u[i] + a) / (s_u[i] / lam_u[i]);
            ratio_min(s_u[i], dsu, mx);
            ratio_min(lam_u[i], dlu, ml);
            bad |= !finite_d(dsu) | !finite_d(dlu);
        }
        ds_l[i] = dsl;
        ds_u[i] = dsu;
        dl_l[i] = dll;
        dl_u[i] = dlu;
    }
    if (bad) sc->nonfinite = 1;
    const double a = block_min(mx, red);
    const double b = block_min(ml, red);
    if (threadIdx.x == 0) {
        p1[blockIdx.x] = a;
        p2[blockIdx.x] = b;
    }
    if (last_block(&sc->counters[C_REC_M])) {
        const double ta = min_partials(p1, gridDim.x, red);
        const double tb = min_partials(p2, gridDim.x, red);
        if (threadIdx.x == 0) {
            sc->counters[C_REC_M] = 0;
            sc->minx_m = ta;
            sc->minl_m = tb;
        }
    }
}

__global__ void __launch_bounds__(kBlock)
k_recover_n(int n, const double *__restrict__ xl, const double *__restrict__ xu, const double *__restrict__ dx,
            const double *__restrict__ r_l, const double *__restrict__ r_u, const double *__restrict__ rc_l,
            const double *__restrict__ rc_u, const double *__restrict__ s_l, const double *__restrict__ s_u,
            const double *__restrict__ lam_l, const double *__restrict__ lam_u, double *__restrict__ ds_l,
            double *__restrict__ ds_u, double *__restrict__ dl_l, double *__restrict__ dl_u,
            double *__restrict__ p1, double *__restrict__ p2, Scalars *sc, double tau) {
    __shared__ double red[kBlock / 32];
    double mx = INFINITY, ml = INFINITY;
    int bad = 0;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const double d = dx[j];
        double dsl = 0.0, dll = 0.0, dsu = 0.0, dlu = 0.0;
        bad |= !finite_d(d);
        if (has(xl[j])) {
            dsl = d + r_l[j];
            dll = -fma(lam_l[j], dsl, rc_l[j]) / s_l[j];
            ratio_min(s_l[j], dsl, mx);
            ratio_min(lam_l[j], dll, ml);
            bad |= !finite_d(dsl) | !finite_d(dll);
        }
        if (has(xu[j])) {
            dsu = -d + r_u[j];
            dlu = -fma(lam_u[j], dsu, rc_u[j]) / s_u[j];
            ratio_min(s_u[j], dsu, mx);
            ratio_min(lam_u[j], dlu, ml);
            bad |= !finite_d(dsu) | !finite_d(dlu);
        }
        ds_l[j] = dsl;
        ds_u[j] = dsu;
        dl_l[j] = dll;
        dl_u[j] = dlu;
    }
    if (bad) sc->nonfinite = 1;
    const double a = block_min(mx, red);
    const double b = block_min(ml, red);
    if (threadIdx.x == 0) {
        p1[blockIdx.x] = a;
        p2[blockIdx.x] = b;
    }
    if (last_block(&sc->counters[C_REC_N])) {
        const double ta = min_partials(p1, gridDim.x, red);
        const double tb = min_partials(p2, gridDim.x, red);
        if (threadIdx.x == 0) {
            sc->counters[C_REC_N] = 0;
            if (sc->sharded) {
                sc->loc[0] = ta;
                sc->loc[1] = tb;
            } else {
                fin_recover(sc, ta, tb, tau);
            }
        }
    }
}

// Requires V.dx (PCG solution) and V.Adx = A dx.  aff=1 writes the affine-step arrays.
void launch_recover(const Prob &P, const Vecs &V, Scalars *sc, double tau, int aff, cudaStream_t st) {
    double *dsA_l = aff ? V.ads_lA : V.ds_lA, *dsA_u = aff ? V.ads_uA : V.ds_uA;
    double *dlA_l = aff ? V.adl_lA : V.dl_lA, *dlA_u = aff ? V.adl_uA : V.dl_uA;
    double *dsx_l = aff ? V.ads_lx : V.ds_lx, *dsx_u = aff ? V.ads_ux : V.ds_ux;
    double *dlx_l = aff ? V.adl_lx : V.dl_lx, *dlx_u = aff ? V.adl_ux : V.dl_ux;
    const double inf = INFINITY;
    cudaMemcpyAsync(&sc->minx_m, &inf, sizeof(double), cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(&sc->minl_m, &inf, sizeof(double), cudaMemcpyHostToDevice, st);
    if (P.m > 0)
        k_recover_m<<<grid_for(P.m, kBlock), kBlock, 0, st>>>(P.m, P.l, P.u, V.Adx, V.r_lA, V.r_uA, V.r2_l, V.r2_u,
                                                             V.s_lA, V.s_uA, V.lam_lA, V.lam_uA, dsA_l, dsA_u, dlA_l,
                                                             dlA_u, V.part[0], V.part[1], sc, P.aug ? V.ag.xl : nullptr,
                                                             P.aug ? V.ag.xu : nullptr);
    k_recover_n<<<grid_for(P.n, kBlock), kBlock, 0, st>>>(P.n, P.xl, P.xu, V.dx, V.r_lx, V.r_ux, V.rc_lx, V.rc_ux,
                                                         V.s_lx, V.s_ux, V.lam_lx, V.lam_ux, dsx_l, dsx_u, dlx_l, dlx_u,
                                                         V.part[2], V.part[3], sc, tau);
}

// ------------------------------------------------------------------------------ update
__global__ void k_update(int len, double ax, double al, const double *__restrict__ axp, const double *__restrict__ alp,
                         double *__restrict__ v, const double *__restrict__ dv, double *__restrict__ s1,
                         const double *__restrict__ ds1, double *__restrict__ s2, const double *__restrict__ ds2,
                         double *__restrict__ l1, const double *__restrict__ dl1, double *__restrict__ l2,
                         const double *__restrict__ dl2) {
    if (axp) { ax = *axp; al = *alp; }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) {
        if (v) v[i] = fma(ax, dv[i], v[i]);
        s1[i] = fma(ax, ds1[i], s1[i]);
        s2[i] = fma(ax, ds2[i], s2[i]);
        l1[i] = fma(al, dl1[i], l1[i]);
        l2[i] = fma(al, dl2[i], l2[i]);
    }
}

void launch_update(const Prob &P, const Vecs &V, Scalars *sc, cudaStream_t st) {
    if (P.m > 0)
        k_update<<<grid_for(P.m, kBlock), kBlock, 0, st>>>(P.m, 0.0, 0.0, &sc->alpha_x, &sc->alpha_l, nullptr, nullptr,
                                                          V.s_lA, V.ds_lA, V.s_uA, V.ds_uA, V.lam_lA, V.dl_lA, V.lam_uA,
                                                          V.dl_uA);
    k_update<<<grid_for(P.n, kBlock), kBlock, 0, st>>>(P.n, 0.0, 0.0, &sc->alpha_x, &sc->alpha_l, V.x, V.dx, V.s_lx,
                                                      V.ds_lx, V.s_ux, V.ds_ux, V.lam_lx, V.dl_lx, V.lam_ux, V.dl_ux);
}

// ---------------------------------------------------------------- Mehrotra mu_aff (R18)
__global__ void __launch_bounds__(kBlock)
k_muaff(int len, const double *__restrict__ s1, const double *__restrict__ ds1, const double *__restrict__ l1,
        const double *__restrict__ dl1, const double *__restrict__ s2, const double *__restrict__ ds2,
        const double *__restrict__ l2, const double *__restrict__ dl2, double *__restrict__ dpart, Scalars *sc,
        int cid, int final_) {
    __shared__ double red[kBlock / 32];
    const double ax = sc->alpha_x, al = sc->alpha_l;
    double acc = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) {
        acc = fma(fma(al, dl1[i], l1[i]), fma(ax, ds1[i], s1[i]), acc);
        acc = fma(fma(al, dl2[i], l2[i]), fma(ax, ds2[i], s2[i]), acc);
    }
    const double b = block_sum(acc, red);
    if (threadIdx.x == 0) dpart[blockIdx.x] = b;
    if (last_block(&sc->counters[cid])) {
        const double t = sum_partials(dpart, gridDim.x, red);
        if (threadIdx.x == 0) {
            sc->counters[cid] = 0;
            if (final_) { sc->muaff = sc->muaff_m + t; sc->loc[5] = t; }
            else sc->muaff_m = t;
        }
    }
}

void launch_muaff(const Prob &P, const Vecs &V, Scalars *sc, cudaStream_t st) {
    cudaMemsetAsync(&sc->muaff_m, 0, sizeof(double), st);
    if (P.m > 0)
        k_muaff<<<grid_for(P.m, kBlock), kBlock, 0, st>>>(P.m, V.s_lA, V.ads_lA, V.lam_lA, V.adl_lA, V.s_uA, V.ads_uA,
                                                         V.lam_uA, V.adl_uA, V.part[0], sc, C_MUAFF_M, 0);
    k_muaff<<<grid_for(P.n, kBlock), kBlock, 0, st>>>(P.n, V.s_lx, V.ads_lx, V.lam_lx, V.adl_lx, V.s_ux, V.ads_ux,
                                                     V.lam_ux, V.adl_ux, V.part[1], sc, C_MUAFF_N, 1);
}


// Touch every kernel once (cudaFuncGetAttributes) so that CUDA's lazy module loading never
// has to load one while a peer-exchange wait kernel spins on the device (kernels.h).
template <class F>
static void touch_kernel(F f) {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(f));
}

void preload_ipmops() {
    touch_kernel(k_init_x); touch_kernel(k_init_slacks); touch_kernel(k_sum_ls); touch_kernel(k_resid_m);
    touch_kernel(k_sigma_m); touch_kernel(k_rhs_m); touch_kernel(k_recover_m); touch_kernel(k_recover_n);
    touch_kernel(k_update); touch_kernel(k_muaff);
#define IPM_TOUCH_G(GG) touch_kernel(k_resid_n<GG>); touch_kernel(k_sigma_n_jacobi<GG>); touch_kernel(k_rhs_n<GG>);
    IPM_TOUCH_G(4) IPM_TOUCH_G(8) IPM_TOUCH_G(16) IPM_TOUCH_G(32)
#undef IPM_TOUCH_G
}

}  // namespace ipm
