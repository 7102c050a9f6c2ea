// state.h — device-side views shared by the kernels and the host orchestration.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace ipm {

constexpr int kMaxPartials = 4096;   // per-reduction partial slots (>= any grid we launch)
constexpr int kNumCounters = 48;

// Scalars living in device memory (one struct, 8-byte fields).  Host reads a copy after
// the per-IPM-iteration synchronisation.
struct Scalars {
    // --- PCG ---------------------------------------------------------------------------
    double rho;        // r^T z of the current iteration
    double rho_old;
    double rr;         // r^T r
    double tol2;       // squared stopping threshold on ||r||_2
    double pKp;        // p^T K p
    double alpha;      // rho / pKp
    double S_b;        // sum sig_b p^2          (diagonal part of p^T K p)
    double S_c;        // sum sig_c (A p)^2      (A^T Sigma_c A part)
    double S_H;        // p^T H p
    double rhs2;       // ||rhs||^2
    double res2;       // scratch: a squared norm (true residual)
    int64_t it;        // PCG iterations since the last init
    int64_t it_rs;     // iterations since the last (re)start (beta = 0 when 0)
    int64_t maxit;
    int64_t done;      // 1 = stop the loop (converged or limit or breakdown)
    int64_t breakdown; // 1 = p^T K p <= 0 or non-finite
    int64_t restarts;  // one-warp PCG (n <= kWarpMaxN): true-residual restarts taken in the kernel
    int64_t stalled;   // one-warp PCG: stopped at the iteration / restart limit above tolerance
    // --- IPM -----------------------------------------------------------------------------
    double sum_ls_m, sum_ls;     // sum lam*s (init / mu updates)
    double rH_max_m, rH_max;     // (m-part unused slot kept for symmetry)
    double prim_max_m, prim_max; // max |r_lA|,|r_uA|,|r_lx|,|r_ux|
    double comp_max_m, comp_max; // max |lam s - mu|
    double ls_max_m, ls_max;     // max lam s
    double obj;                  // 1/2 x^T H x + g^T x
    double minx_m, minl_m;       // min ratio over m-space families
    double alpha_x, alpha_l;
    double muaff_m, muaff;       // Mehrotra affine complementarity sums
    int64_t nonfinite;           // residual/step contained Inf/NaN
    // --- row-sharded mode ------------------------------------------------
    // sharded = 1: last blocks write this rank's partials to loc[] and skip every derived
    // quantity; an allgather of loc[] plus k_xcombine (rank-ordered, identical on all ranks)
    // produces the global values.  Slot use per stage is documented in shard.cu.
    int64_t sharded;
    double loc[8];
    // peer-memory data plane (peer.cu): sequence number of the last completed exchange, the
    // put kernels' arrival counter, and a timeout flag (a peer never arrived)
    unsigned long long peer_seq[2];      // per exchange channel (peer.h)
    unsigned int peer_ctr[2], peer_timeout;
    int64_t spmv_split;                  // 1: the PCG SpMV runs on this rank's A rows; S_c partial in loc[2]
    // Chronopoulos-Gear single-reduction PCG (sharded option): beta of the update, first-step flag
    double cg_beta;
    int64_t cg_first;
    unsigned long long peer_diag[4];     // timeout: {expected seq, sender, its flag, stage + 1000}
    unsigned int counters[kNumCounters];
    // --- live launch timing of the PCG operator kernel (bench.py roofline) ---------------
    // kt_neg = max over CTAs of ~(start %globaltimer) (so 0 = unset), reset by the last CTA,
    // which adds (its end - earliest start) to kt_ns and counts the launch.
    unsigned long long kt_neg, kt_ns, kt_count;
#ifdef IPM_TIMELINE
    // diagnostic builds only (scripts/timeline_probe.py): per-kernel first-CTA start (as ~t)
    // and last thread-0 exit of the current PCG iteration, copied into a ring by the update
    unsigned long long tl[4][2];
    unsigned long long tl_u[4];          // update: latest CTA start, latest rows-done, latest arrival
    unsigned long long tl_ring[64][16];
#endif
};

// Combine stages of k_xcombine (shard.cu).
enum XStage { X_PCG_INIT = 0, X_PCG_ALPHA, X_PCG_UPDATE, X_PCG_RESTART, X_RES2, X_SUMLS, X_RESID, X_RECOVER, X_MUAFF,
              X_CG };

enum Counter {
    C_GEMV = 0, C_GEMV_PCG, C_SPMV, C_SPMV_PCG, C_P, C_UPD, C_INIT_PCG, C_TRUE_RES, C_INIT_M, C_INIT_N,
    C_RES_M, C_RES_N, C_REC_M, C_REC_N, C_MUAFF_M, C_MUAFF_N, C_FINITE, C_LS_M, C_LS_N,
    C_UPD2, C_BAR, C_BAR_GEN, C_P2
};

// Read-only problem view.
struct Prob {
    int n, m;              // n = local rows of H / x-space length (== global n unsharded)
    int ncols;             // global n (columns of H, length of gathered vectors)
    int64_t nnz;
    int64_t ldh;
    double *H;             // local row block (writable only by the rank-2 update)
    const int64_t *Arp;
    const int *Acol;
    const double *Aval;
    const int64_t *ATrp;   // transpose, rows = local x-space rows
    const int *ATcol;
    const double *ATval;
    const double *g, *l, *u, *xl, *xu;
    double *diagH;
    int gemv_bulk;         // 1: use the TMA-bulk GEMV (k_gemv_bulk) with grid gemv_bulk_grid
    int gemv_bulk_grid;
    int gemv_sym;          // 1: symmetric upper-triangle TMA-bulk GEMV (k_symv_bulk)
    int sym_keep;          // leading tiles of each CTA's range loaded with an L2 evict_last policy
    int ncb;               // column blocks of the ypart[row][cb] layout of the chosen GEMV
    const void *tmap_sym;  // host copy of the CUtensorMap over H (16 x 256 fp64 boxes)
    const struct SymRange *sym_ranges;   // device: per-CTA strip ranges (kernels.h SymPlan)
    const struct SymTile *sym_tiles;     // device: the tile list
    double *sym_z;                       // sharded: column parts of other ranks' rows [zrows][ldz]
    int sym_ycarry, sym_ldz, sym_zcarry; // ypart carry base (= nbg), zpart stride and carry base
    int sym_ntma, sym_ntiles;            // hybrid SYMV: tiles [ntma, ntiles) go to the LDG warps
    int64_t row_begin;                   // global index of local row 0
    // compact quasi-Newton Hessian H = diag(h0) + U diag(w) U^T (compact.cu)
    int hess_compact;
    int ck;                // columns of U in use
    int64_t ldu;           // leading dimension (= column capacity) of U
    double *U;             // borrowed, n x ldu row-major
    double *h0, *w;        // workspace copies (w has capacity ldu)
    double *cs, *cspart, *chpart;   // s = U^T p (ldu), per-CTA column partials, per-CTA h0 p^2 partials
    int aug;               // 1: PCG on the doubly augmented system eq:2x2_augmented
    int ktimer;            // 1: the PCG-mode operator kernel times its launches (opt.kernel_timer)
    double *Kd;            // n <= kWarpMaxN: the condensed K assembled densely (kWarpMaxN x kWarpMaxN)
};

// Iterate, residuals and per-IPM-iteration work vectors (masked full-length layout).
struct Vecs {
    // n-space
    double *x, *s_lx, *s_ux, *lam_lx, *lam_ux;
    double *rH, *r_lx, *r_ux, *rc_lx, *rc_ux, *Hx;
    double *sig_b, *Minv, *rhs, *dx;
    double *ds_lx, *ds_ux, *dl_lx, *dl_ux;
    double *ads_lx, *ads_ux, *adl_lx, *adl_ux;      // Mehrotra affine step
    // m-space
    double *s_lA, *s_uA, *lam_lA, *lam_uA;
    double *r_lA, *r_uA, *rc_lA, *rc_uA, *Ax;
    double *sig_c, *r2_l, *r2_u, *w, *Adx;
    double *ds_lA, *ds_uA, *dl_lA, *dl_uA;
    double *ads_lA, *ads_uA, *adl_lA, *adl_uA;
    double *lamd;                                   // lam_lA - lam_uA scratch (m)
    // PCG
    double *pr, *pz, *pp, *pt, *py;                  // r, z, p (n), t (m), y (n)
    double *pAt;                                     // A^T t (n), formed on the SpMV branch
    double *ypart;                                   // n x ncb GEMV tile partials
    double *gfull;                                   // sharded: gathered full-length vector (P*chunk)
    double *xloc_all;                                // sharded: allgathered loc[] of all ranks (8*P)
    double *part[8];                                 // reduction partials, kMaxPartials each
    struct {                                         // doubly augmented PCG (NEXT-2), m-space segments
        double *xl, *xu, *rl, *ru, *zl, *zu, *pl, *pu, *yl, *yu, *Dl, *Du, *Ml, *Mu;
    } ag;
};

// Kernel-side view of the augmented segments (on = 0: condensed system, everything ignored).
struct AugArgs {
    int on;
    int m;
    double *xl, *xu, *rl, *ru, *zl, *zu, *pl, *pu, *yl, *yu;
    const double *Ml, *Mu;
    const double *rhsl, *rhsu;   // = r2_l, r2_u (the bottom block of the eq:2x2_augmented rhs)
};

}  // namespace ipm
