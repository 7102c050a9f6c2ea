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
#include <algorithm>

#include "common.cuh"
#include "finalize.cuh"
#include "kernels.h"
#include "state.h"

namespace ipm {

__global__ void k_xcombine(Scalars *sc, const double *__restrict__ xa, int P, int stage, double p0, double p1,
                           int64_t p2) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    xcombine_apply(sc, xa, P, stage, p0, p1, p2);
}

void launch_xcombine(Scalars *sc, const double *xall, int P, int stage, double p0, double p1, int64_t p2,
                     cudaStream_t st) {
    k_xcombine<<<1, 32, 0, st>>>(sc, xall, P, stage, p0, p1, p2);
}

// ---------------------------------------------------- sharded symmetric GEMV (SymPlan)
// Column parts a rank computed for other ranks' rows: zvec[col] = sum of its zpart row over the
// slots in slot order (untouched columns stay 0); after the allgather of zvec, every rank adds
// the P contributions to its own rows in rank order into the last ypart slot.
__global__ void k_zreduce(int zrows, int ldz, const double *__restrict__ zpart, const int *__restrict__ zcol,
                          double *__restrict__ zvec) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < zrows; q += gridDim.x * blockDim.x) {
        const double *z = zpart + (int64_t)q * ldz;
        double s = 0.0;
        for (int k = 0; k < ldz; ++k) s += z[k];
        zvec[zcol[q]] = s;
    }
}

__global__ void k_zfold(int nloc, int ncols, int nranks, int64_t row_begin, const double *__restrict__ zall,
                        double *__restrict__ ypart, int ldy) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nloc; i += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < nranks; ++r) s += zall[(int64_t)r * ncols + row_begin + i];
        ypart[(int64_t)i * ldy + ldy - 1] = s;
    }
}

void launch_zreduce(int zrows, int ldz, const double *zpart, const int *zcol, double *zvec, cudaStream_t st) {
    if (zrows <= 0) return;
    k_zreduce<<<std::min(kMaxGrid, (zrows + 255) / 256), 256, 0, st>>>(zrows, ldz, zpart, zcol, zvec);
}

void launch_zfold(int nloc, int ncols, int nranks, int64_t row_begin, const double *zall, double *ypart, int ldy,
                  cudaStream_t st) {
    k_zfold<<<std::min(kMaxGrid, (nloc + 255) / 256), 256, 0, st>>>(nloc, ncols, nranks, row_begin, zall, ypart, ldy);
}

// Exact symmetry certificate of a row-sharded H without moving it: every entry outside the
// rank's own column range contributes mix(min(i,j), max(i,j), bits(H_ij)) to a per-owner-rank
// sum mod 2^64 (order-independent), so rank a's sum for rank b equals rank b's sum for rank a
// iff the two off-diagonal blocks are transposes (up to a 2^-64 collision chance); the
// diagonal block is compared entry by entry (k_count_asym on the shifted block).
__device__ __forceinline__ unsigned long long smix(unsigned long long z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__global__ void k_sym_hash(int nloc, int ncols, int64_t row_begin, int chunk, int nranks, const double *__restrict__ H,
                           int64_t ldh, unsigned long long *__restrict__ out) {
    const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    for (int i = blockIdx.x * wpb + (threadIdx.x >> 5); i < nloc; i += gridDim.x * wpb) {
        const unsigned long long gi = (unsigned long long)(row_begin + i);
        const double *h = H + (int64_t)i * ldh;
        for (int b = 0; b < nranks; ++b) {
            const int64_t c0 = (int64_t)b * chunk, c1 = min((int64_t)ncols, c0 + chunk);
            if (c0 == row_begin) continue;
            unsigned long long acc = 0ull;
            for (int64_t j = c0 + lane; j < c1; j += 32) {
                const unsigned long long lo = gi < (unsigned long long)j ? gi : (unsigned long long)j;
                const unsigned long long hi = gi < (unsigned long long)j ? (unsigned long long)j : gi;
                acc += smix(smix(lo * 0x100000001b3ull + hi) ^ (unsigned long long)__double_as_longlong(h[j]));
            }
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0 && c0 < c1) atomicAdd(out + b, acc);
        }
    }
}

void launch_sym_hash(int nloc, int ncols, int64_t row_begin, int chunk, int nranks, const double *H, int64_t ldh,
                     unsigned long long *out, cudaStream_t st) {
    k_sym_hash<<<std::min(kMaxGrid, (nloc + 7) / 8), 256, 0, st>>>(nloc, ncols, row_begin, chunk, nranks, H, ldh, out);
}


// Touch every kernel once (cudaFuncGetAttributes) so that CUDA's lazy module loading never
// has to load one while a peer-exchange wait kernel spins on the device (kernels.h).
template <class F>
static void touch_kernel(F f) {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(f));
}

void preload_shard() {
    touch_kernel(k_xcombine); touch_kernel(k_zreduce); touch_kernel(k_zfold); touch_kernel(k_sym_hash);
}

}  // namespace ipm
