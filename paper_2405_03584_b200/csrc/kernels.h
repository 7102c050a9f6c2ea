// kernels.h — launch wrappers of every kernel in libipm.so (host-callable).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "state.h"

namespace ipm {

constexpr int kBlock = 256;
constexpr int kMaxGrid = 148 * 8;   // grid-stride elementwise kernels: <= 8 CTAs per SM
constexpr int kGemvThreads = 256;   // 8 warps, 2 rows each
constexpr int kGemvRB = 16;         // rows per GEMV tile
constexpr int kGemvCW = 1024;       // columns per GEMV tile (8 KB of the vector in smem)

inline int gemv_ncb(int ncols) { return (ncols + kGemvCW - 1) / kGemvCW; }
constexpr int kSymB = 256;          // symmetric GEMV: square B x B blocks of H
inline int sym_ncb(int n) { return (n + kSymB - 1) / kSymB; }
#ifndef IPM_SYM_SR
#define IPM_SYM_SR 32
#endif
constexpr int kSymSR = IPM_SYM_SR;  // symmetric GEMV: rows per TMA strip (pipeline stage)

// Work plan of the symmetric GEMV (sym_plan_build, linalg.cu).  A tile is a kSymB x kSymB
// block of this rank's rows; its row part (H_IJ p_J) goes to ypart slot rslot of its rows, its
// column part (H_IJ^T p_I) to slot cslot of rows cbase.. of ypart (cmode 1) or of the remote
// buffer zpart (cmode 2: another rank's rows; reduced and exchanged by the caller); cmode 0 =
// diagonal tile (row part only).  The strips (kSymSR rows) of the tile list are cut into
// `grid` contiguous equal ranges, so no CTA streams more than one strip (64 KB) above the
// average.  A range that starts inside a tile writes that tile's column partial to a carry
// slot (ycarry + k / zcarry + k) instead of cslot (written by the tile's owner, the CTA
// holding its strip 0): every slot is written by exactly one CTA and the consumers' fixed-
// order row sums stay deterministic.
struct SymTile {
    int r0, rows;   // local rows
    int c0, cols;   // global columns
    int rslot;      // ypart slot of the row part
    int cmode;      // 0 diagonal tile, 1 column part to ypart, 2 column part to zpart
    int cbase;      // first row (ypart: local row, zpart: compact remote column) of the column part
    int cslot;      // its slot
};
struct SymRange {
    int t0, s0;     // first tile and first strip in it
    int t1, s1;     // end: tile t1, strip s1 (exclusive); s1 == 0 means the range ends at tile t1
    int carry;      // carry slot of the head partial tile, -1 if none
    int pad[3];
};
struct SymPlan {
    std::vector<SymTile> tiles;     // [0, ntma): streamed through the TMA ring (ranges); [ntma, size):
                                    // whole tiles for the LDG warps (hybrid build), CTA b takes
                                    // ntma + b, ntma + b + grid, ...
    std::vector<SymRange> ranges;
    std::vector<int> zcol;          // global column of each zpart row
    int nbg = 0, ycarry_n = 0, zcarry_n = 0, ldy = 0, ldz = 0, zrows = 0, ntma = 0;
};
#ifndef IPM_SYM_LDG_EVERY
#define IPM_SYM_LDG_EVERY 0
#endif
constexpr int kSymLdgEvery = IPM_SYM_LDG_EVERY;   // hybrid SYMV: every k-th off-diagonal tile to LDG warps
void sym_plan_build(int ncols, int nranks, int rank, int grid, SymPlan &plan);

// linalg.cu
// sigb_dot (symmetric GEMV only): also add sigma_b p^2 to the fused dot (p^T (H + Sigma_b) p)
void launch_gemv(const Prob &P, const double *v, const double *vdot, double *ypart, int ncb,
                 double *dpart, Scalars *sc, int grid, int mode, int cid, cudaStream_t st,
                 const double *sigb_dot = nullptr);
int gemv_max_grid();
bool gemv_bulk_ok(const Prob &P);
void launch_symv_bulk(const Prob &P, const double *v, const double *vdot, double *ypart, double *dpart, Scalars *sc,
                      int grid, int mode, int cid, cudaStream_t st, const double *sigb_dot = nullptr);
void launch_count_asym(const Prob &P, unsigned long long *bad, cudaStream_t st);
bool make_sym_tensor_map(const Prob &P, void *out128);   // CUtensorMap (128 B, 64-B aligned)
int gemv_bulk_grid();
void launch_gemv_bulk(const Prob &P, const double *v, const double *vdot, double *ypart, int ncb, double *dpart,
                      Scalars *sc, int grid, int mode, int cid, cudaStream_t st);
// max_grid: optional grid cap (the PCG side branch; see side_grid in pcg.cu)
void launch_spmv(const Prob &P, const double *v, const double *sigc, double *y, double *dpart,
                 Scalars *sc, int mode, int check_done, cudaStream_t st, int max_grid = kMaxGrid,
                 int block = kBlock);
int num_sms();
// shard.cu: exchange of the sharded symmetric GEMV's remote column parts, symmetry certificate
void launch_zreduce(int zrows, int ldz, const double *zpart, const int *zcol, double *zvec, cudaStream_t st);
void launch_zfold(int nloc, int ncols, int nranks, int64_t row_begin, const double *zall, double *ypart, int ldy,
                  cudaStream_t st);
void launch_sym_hash(int nloc, int ncols, int64_t row_begin, int chunk, int nranks, const double *H, int64_t ldh,
                     unsigned long long *out, cudaStream_t st);
int side_block();
int spmv_keep();    // IPM_SPMV_KEEP switch (1 default)
int spmv_keep_for(const Prob &P);   // 1: PCG-mode SpMV / SpMV^T load A, A^T evict_last (only when they fit L2)
void launch_spmv_rows(const Prob &P, const double *v, const double *sigc, double *y, double *dpart, Scalars *sc,
                      int64_t r0, int64_t r1, cudaStream_t st, int block);
void launch_pcg_spmvT(const Prob &P, const Vecs &V, int G, Scalars *sc, const double *t, cudaStream_t st);
void launch_pcg_update_only(const Prob &P, const Vecs &V, int G, int ncb, Scalars *sc, double *x, cudaStream_t st);
// Chronopoulos-Gear single-reduction PCG (sharded option, pcg.cu): priming after a (re)start and
// the update (operator applied to u = V.pz; p = V.pp, s = K p = V.py by recurrence)
void launch_cg_prime(const Prob &P, const Vecs &V, Scalars *sc, cudaStream_t st);
void launch_cg_update(const Prob &P, const Vecs &V, int ncb, Scalars *sc, double *x, cudaStream_t st);
void configure_linalg_carveout();   // max-shared carveout for kernels co-running with the SYMV
cudaError_t configure_linalg_attrs();   // >48 KB dynamic smem opt-ins (per device: called at every create)
cudaError_t configure_pcg_attrs();
// force-load every kernel (CUDA lazy loading must not run while a peer wait kernel spins)
void preload_linalg();
void preload_pcg();
void preload_ipmops();
void preload_shard();
void preload_peer();
void preload_compact();
void preload_tiny();
inline void preload_all_kernels() {
    preload_linalg();
    preload_pcg();
    preload_ipmops();
    preload_shard();
    preload_peer();
    preload_compact();
    preload_tiny();
}

// tiny.cu — the whole Algorithm 1 loop in one warp (n, m <= kWarpMaxN)
struct TinyOut {
    int32_t status, ipm_iters, pcg_max, stalls, restarts, ntrace;
    int64_t pcg_total, pcg_it_last;
    double mu;
    unsigned long long t_pcg_ns;
};
struct TinyArgs {
    int n, m;
    const double *H;
    int64_t ldh;
    const int64_t *Arp;
    const int *Acol;
    const double *Aval;
    const double *g, *l, *u, *xl, *xu;
    double *x, *s_lA, *s_uA, *lam_lA, *lam_uA, *s_lx, *s_ux, *lam_lx, *lam_ux, *dx, *Hx, *Ax;
    double mu0, mu_tol, mu_div, tau, rtol_floor, rtol_max, rtol_fac, atol;
    int schedule, max_ipm, trace;
    int64_t pcg_maxit;
    void *trace_buf;                       // ipm_trace_rec[max_ipm] (device)
    TinyOut *out;
    Scalars *sc;
};
bool tiny_eligible(int n, int m);
size_t tiny_smem_bytes();
void launch_ipm_tiny(const TinyArgs &a, cudaStream_t st);
cudaError_t configure_tiny_attrs();
void configure_pcg_carveout();
// NEXT-2 doubly augmented operator: t = 2 sig_c o (A px) + pl - pu, yl = A px + D_l pl,
// yu = -A px + D_u pu (masked); mode 1 (PCG): done check + S_c = a.t + pl.yl + pu.yu
void launch_spmv_aug(const Prob &P, const Vecs &V, const double *px, const double *pl, const double *pu, Scalars *sc,
                     int mode, cudaStream_t st);
AugArgs aug_args(const Prob &P, const Vecs &V);
void launch_apply_reduce(const Prob &P, int G, int ncb, const double *ypart, const double *sigb,
                         const double *v, const double *t, double *y, const double *rhs, double *dpart,
                         Scalars *sc, int mode, cudaStream_t st, const AugArgs *ag = nullptr);
void launch_jacobi(const Prob &P, int G, const double *sigb, const double *sigc, double *out, int invert,
                   cudaStream_t st);
void launch_setup_diag(const Prob &P, int row0, cudaStream_t st);
void launch_count_nonfinite(const Prob &P, unsigned long long *bad, cudaStream_t st);
void launch_transpose(const Prob &P, int col0, int nchunk, int *cnt, int64_t *ATrp, int *ATcol,
                      double *ATval, cudaStream_t st);
void launch_rank2(const Prob &P, int row0, const double *u, double a, const double *v, double b, cudaStream_t st);

// compact.cu (NEXT-1: H = diag(h0) + U diag(w) U^T, matrix-free)
constexpr int kCompactGrid = 148;   // U^T p: one 1024-thread CTA per SM
constexpr int kCompactMaxCols = 6144;   // w o s staged in 48 KB of dynamic smem (k_compact_us)
void launch_compact_apply(const Prob &P, const double *v, const double *vdot, double *ypart, Scalars *sc, int mode,
                          int cid, cudaStream_t st);
void launch_compact_diag(const Prob &P, cudaStream_t st);
void launch_compact_append(const Prob &P, double *U, int col, const double *u, const double *v, cudaStream_t st);

// pcg.cu
void launch_pcg_init(const Prob &P, const Vecs &V, Scalars *sc, const double *rhs, double *x, double rtol,
                     double atol, int64_t maxit, int keep_x, cudaStream_t st);
struct Fork {  // side stream + events for the SpMV || GEMV branch of a PCG iteration
    cudaStream_t side;
    cudaEvent_t ev_fork, ev_join;
};
void launch_pcg_iteration(const Prob &P, const Vecs &V, int G, int ncb, int gemv_grid, Scalars *sc, double *x,
                          cudaGraphConditionalHandle h, int use_cond, cudaStream_t st, const Fork *fork,
                          bool fused_p = false);
void launch_pcg_restart(const Prob &P, const Vecs &V, Scalars *sc, cudaStream_t st);
void launch_pcg_p(const Prob &P, const Vecs &V, Scalars *sc, cudaStream_t st);
constexpr int kWarpMaxN = 64;       // one-warp PCG on an assembled K at or below this size
constexpr int kSmallN = 256;        // single-CTA PCG loop below this size (launch-latency bound)
// one-warp path (n <= kWarpMaxN, K assembled): also confirms the true residual and restarts in the
// kernel when check = 1 (sc->res2 / restarts / stalled); the single-CTA path leaves that to the host
bool pcg_warp_path(const Prob &P);
int launch_pcg_small(const Prob &P, const Vecs &V, Scalars *sc, double *x, const double *rhs, int check,
                     cudaStream_t st);
void launch_pcg_update(const Prob &P, const Vecs &V, int G, int ncb, Scalars *sc, double *x, cudaStream_t st);

// shard.cu
void launch_xcombine(Scalars *sc, const double *xall, int P, int stage, double p0, double p1, int64_t p2,
                     cudaStream_t st);
void launch_dot2(int n, const double *a, double *dpart, Scalars *sc, cudaStream_t st);  // res2 = |a|^2

// ipmops.cu — per-IPM-iteration kernels (masked full-length families)
void launch_init_x(const Prob &P, const Vecs &V, int warm, double theta, cudaStream_t st);
void launch_init_slacks(const Prob &P, const Vecs &V, Scalars *sc, int warm, double theta, cudaStream_t st);
void launch_residuals(const Prob &P, const Vecs &V, int G, Scalars *sc, double mu, cudaStream_t st);
void launch_sigma(const Prob &P, const Vecs &V, int G, cudaStream_t st);
void launch_rhs(const Prob &P, const Vecs &V, int G, double mu, int mode, double sigma_mu, cudaStream_t st);
void launch_recover(const Prob &P, const Vecs &V, Scalars *sc, double tau, int aff, cudaStream_t st);
void launch_update(const Prob &P, const Vecs &V, Scalars *sc, cudaStream_t st);
void launch_muaff(const Prob &P, const Vecs &V, Scalars *sc, cudaStream_t st);
void launch_sum_ls(const Prob &P, const Vecs &V, Scalars *sc, cudaStream_t st);

}  // namespace ipm
