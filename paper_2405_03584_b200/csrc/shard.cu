// shard.cu — deterministic cross-rank combination of reduction partials.
//
// Row-sharded mode: every reduction kernel's last block writes THIS rank's partial into
// Scalars::loc[]; the host allgathers loc[] of all ranks (P x 8 doubles) and k_xcombine —
// one thread, ranks in ascending order — applies the same epilogue the single-GPU last
// blocks apply (finalize.cuh).  Every rank computes bit-identical global scalars, so the
// host-side decisions of Algorithm 1 (PCG stop, mu/10, return) agree across ranks without
// a second collective.  Slot use:
//   X_PCG_INIT     loc[2] = r^T z, loc[3] = r^T r                     (k_pcg_init)
//   X_PCG_ALPHA    loc[0] = sum sig_b p^2 (k_pcg_p), loc[1] = p^T H_loc p (GEMV); S_c is
//                  replicated (A is replicated) and added once
//   X_PCG_UPDATE   loc[2] = r^T z, loc[3] = r^T r                     (k_pcg_update)
//   X_PCG_RESTART  loc[2], loc[3]                                     (k_pcg_restart)
//   X_RES2         loc[4] = ||rhs - K x||^2 partial                   (k_apply_reduce<.,1>)
//   X_SUMLS        loc[5] = n-space part of sum lam s (m-space part replicated)
//   X_RESID        loc[0..4] = max|r_H|, max|primal|, max|lam s - mu|, max lam s, objective
//                  part; loc[6] = non-finite flag                      (k_resid_n)
//   X_RECOVER      loc[0], loc[1] = min step ratios over the local x-space families
//   X_MUAFF        loc[5] = n-space part of the Mehrotra affine complementarity sum
#include "common.cuh"
#include "finalize.cuh"
#include "kernels.h"
#include "state.h"

namespace ipm {

__global__ void k_xcombine(Scalars *sc, const double *__restrict__ xa, int P, int stage, double p0, double p1,
                           int64_t p2) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
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
        default:
            break;
    }
}

void launch_xcombine(Scalars *sc, const double *xall, int P, int stage, double p0, double p1, int64_t p2,
                     cudaStream_t st) {
    k_xcombine<<<1, 32, 0, st>>>(sc, xall, P, stage, p0, p1, p2);
}

}  // namespace ipm
