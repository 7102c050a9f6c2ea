// finalize.cuh — the scalar "epilogues" of the reductions, shared by the kernels' last
// blocks (one GPU) and by k_xcombine (row-sharded: applied to the rank-ordered combination
// of every rank's partials, so all ranks take bit-identical decisions).
#pragma once

#include "common.cuh"
#include "state.h"

namespace ipm {

// PCG start (S:225 stopping rule ||r||_2 <= max(rtol ||rhs||_2, atol)).
__device__ __forceinline__ void fin_pcg_init(Scalars *sc, double trz, double trr, double rtol, double atol,
                                             int64_t maxit) {
    sc->rho = trz;
    sc->rho_old = trz;
    sc->rr = trr;
    sc->rhs2 = trr;
    const double t1 = rtol * rtol * trr, t2 = atol * atol;
    sc->tol2 = t1 > t2 ? t1 : t2;
    sc->it = 0;
    sc->it_rs = 0;
    sc->maxit = maxit;
    sc->breakdown = 0;
    sc->S_b = sc->S_c = sc->S_H = 0.0;
    sc->done = (trr <= sc->tol2) ? 1 : 0;
    if (!finite_d(trr) || !finite_d(trz)) {
        sc->done = 1;
        sc->breakdown = 1;
    }
}

__device__ __forceinline__ void fin_pcg_restart(Scalars *sc, double trz, double trr) {
    sc->rho = trz;
    sc->rho_old = trz;
    sc->rr = trr;
    sc->it_rs = 0;
    sc->done = (trr <= sc->tol2 || sc->it >= sc->maxit) ? 1 : 0;
}

// alpha = rho / p^T K p; p^T K p <= 0 is a breakdown.
__device__ __forceinline__ void fin_pcg_alpha(Scalars *sc, double pkp) {
    sc->pKp = pkp;
    if (!(pkp > 0.0) || !finite_d(pkp)) {
        sc->breakdown = 1;
        sc->done = 1;
        sc->alpha = 0.0;
    } else {
        sc->alpha = sc->rho / pkp;
    }
}

// end of a PCG iteration: rho, ||r||^2, iteration count and the stop decision.
__device__ __forceinline__ int fin_pcg_update(Scalars *sc, double trz, double trr) {
    sc->rho_old = sc->rho;
    sc->rho = trz;
    sc->rr = trr;
    sc->it += 1;
    sc->it_rs += 1;
    int stop = 0;
    if (trr <= sc->tol2 || sc->it >= sc->maxit) stop = 1;
    if (!finite_d(trr) || !finite_d(trz)) {
        stop = 1;
        sc->breakdown = 1;
    }
    sc->done = stop;
    return stop;
}

// fraction to the boundary: alpha = min(1, tau * min ratio); empty set -> 1.
__device__ __forceinline__ void fin_recover(Scalars *sc, double minx, double minl, double tau) {
    sc->alpha_x = fmin(1.0, tau * fmin(minx, sc->minx_m));
    sc->alpha_l = fmin(1.0, tau * fmin(minl, sc->minl_m));
}

__device__ __forceinline__ void fin_resid(Scalars *sc, double rh, double prim, double comp, double lsm, double obj) {
    sc->rH_max = rh;
    sc->prim_max = fmax(prim, sc->prim_max_m);
    sc->comp_max = fmax(comp, sc->comp_max_m);
    sc->ls_max = fmax(lsm, sc->ls_max_m);
    sc->obj = obj;
    if (!finite_d(obj)) sc->nonfinite = 1;
}

// Rank-ordered combination of every rank's partials of one XStage (row-sharded mode; one
// thread): the same epilogue the single-GPU last blocks apply, so every rank takes
// bit-identical decisions.  xa[r * 8 + k] = rank r's Scalars::loc[k].  Used by k_xcombine
// (allgather data plane) and by the peer-memory wait kernel (peer.cu).
__device__ __forceinline__ void xcombine_apply(Scalars *sc, const double *xa, int P, int stage, double p0, double p1,
                                               int64_t p2) {
    auto sum = [&](int k) {
        double s = 0.0;
        for (int r = 0; r < P; ++r) s += xa[r * 8 + k];
        return s;
    };
    auto mx = [&](int k) {
        double s = xa[k];
        for (int r = 1; r < P; ++r) s = fmax(s, xa[r * 8 + k]);
        return s;
    };
    auto mn = [&](int k) {
        double s = xa[k];
        for (int r = 1; r < P; ++r) s = fmin(s, xa[r * 8 + k]);
        return s;
    };
    switch (stage) {
        case X_PCG_INIT:
            fin_pcg_init(sc, sum(2), sum(3), p0, p1, p2);
            break;
        case X_PCG_ALPHA: {
            if (sc->done) return;
            double s = 0.0, sb = 0.0, sh = 0.0;
            for (int r = 0; r < P; ++r) {
                s += xa[r * 8 + 0] + xa[r * 8 + 1];
                sb += xa[r * 8 + 0];
                sh += xa[r * 8 + 1];
            }
            sc->S_b = sb;
            sc->S_H = sh;
            if (sc->spmv_split) {              // every rank formed S_c over its own rows of A
                double scs = 0.0;
                for (int r = 0; r < P; ++r) scs += xa[r * 8 + 2];
                sc->S_c = scs;
            }
            fin_pcg_alpha(sc, s + sc->S_c);
            break;
        }
        case X_PCG_UPDATE:
            if (sc->done) return;
            fin_pcg_update(sc, sum(2), sum(3));
            break;
        case X_PCG_RESTART:
            fin_pcg_restart(sc, sum(2), sum(3));
            break;
        case X_RES2:
            sc->res2 = sum(4);
            break;
        case X_SUMLS:
            sc->sum_ls = sc->sum_ls_m + sum(5);
            break;
        case X_RESID:
            if (mx(6) > 0.0) sc->nonfinite = 1;
            fin_resid(sc, mx(0), mx(1), mx(2), mx(3), sum(4));
            break;
        case X_RECOVER:
            fin_recover(sc, mn(0), mn(1), p0);
            break;
        case X_MUAFF:
            sc->muaff = sc->muaff_m + sum(5);
            break;
        case X_CG: {
            // Chronopoulos-Gear PCG (one reduction per iteration): loc = {S_b, S_H, S_c part,
            // gamma = r^T u, ||r||^2} of the current u = M^-1 r and w = K u.  Stop before the
            // update when ||r||^2 <= tol^2 or the cap is reached; else
            //   beta = gamma / gamma_prev,  alpha = gamma / (delta - beta gamma / alpha_prev),
            // delta = u^T K u (first step of a (re)start: beta = 0, alpha = gamma / delta).
            if (sc->done) return;
            double sb = 0.0, sh = 0.0, scs = 0.0;
            for (int r = 0; r < P; ++r) {
                sb += xa[r * 8 + 0];
                sh += xa[r * 8 + 1];
                scs += xa[r * 8 + 2];
            }
            const double gam = sum(3), rr = sum(4), gam_prev = sc->rho;
            sc->S_b = sb;
            sc->S_H = sh;
            if (sc->spmv_split) sc->S_c = scs;
            sc->rr = rr;
            sc->rho_old = gam_prev;                   // rho = r^T u of the current residual, as
            sc->rho = gam;                            // fin_pcg_update leaves it
            if (!finite_d(rr) || !finite_d(gam)) {
                sc->breakdown = 1;
                sc->done = 1;
                break;
            }
            if (rr <= sc->tol2 || sc->it >= sc->maxit) {
                sc->done = 1;
                break;
            }
            const double delta = sh + sb + sc->S_c;
            const bool first = (sc->it_rs == 0);
            const double beta = first ? 0.0 : gam / gam_prev;
            const double den = first ? delta : delta - beta * gam / sc->alpha;
            sc->pKp = den;
            if (!(den > 0.0) || !finite_d(den)) {
                sc->breakdown = 1;
                sc->done = 1;
                sc->alpha = 0.0;
                break;
            }
            sc->alpha = gam / den;
            sc->cg_beta = beta;
            sc->cg_first = first ? 1 : 0;
            sc->it += 1;
            sc->it_rs += 1;
            break;
        }
        default:
            break;
    }
}


}  // namespace ipm
