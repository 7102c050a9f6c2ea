// compact.cu — matrix-free compact quasi-Newton Hessian (eq:bfgs_hessian,
// PAPER.md P:240-245):  H = diag(h0) + U diag(w) U^T,  U n x k row-major (leading dim ldu),
// applied as  H p = h0 o p + U (w o (U^T p))  without ever assembling H.
//
// These are the paper's hottest kernels for the proton case (Table 2: "gemv" = U v and
// "gemv transpose" = U^T x).  Both passes stream U once (8 n k bytes each):
//   k_compact_ut : s = U^T p.  Each CTA owns a contiguous row range and thread c a column;
//                  per-CTA partial column sums go to spart[cta][c] and the last CTA reduces
//                  them in CTA order (deterministic), then forms p^T H p = sum h0 p^2 +
//                  sum w s^2 (the fused dot of north_star (b)).
//   k_compact_us : y_i = h0_i p_i + U_i: . (w o s), one warp per row, written as the single
//                  column-block partial ypart[i][0] (ncb = 1) that the PCG update / residual
//                  kernels already consume.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "state.h"

namespace ipm {

constexpr int kCompactThreads = 256;   // warp-per-row CTAs of k_compact_us; ldu <= kCompactMaxCols checked at create

constexpr int kUtThreads = 1024;       // 4 row groups x 256 column slots
constexpr int kUtGroups = kUtThreads / 256;

__global__ void __launch_bounds__(kUtThreads, 1)
k_compact_ut(int n, int k, const double *__restrict__ U, int64_t ldu, const double *__restrict__ p,
             double *__restrict__ spart, double *__restrict__ hpart, double *__restrict__ s,
             const double *__restrict__ h0, const double *__restrict__ w, const double *__restrict__ pdot_vec,
             Scalars *sc, int cid, int mode) {
    __shared__ double red[kUtThreads / 32];
    __shared__ double grp[kUtGroups][256];
    if (mode == 1 && sc->done) return;
    const int64_t r0 = (int64_t)n * blockIdx.x / gridDim.x, r1 = (int64_t)n * (blockIdx.x + 1) / gridDim.x;
    const int slot = threadIdx.x & 255, gq = threadIdx.x >> 8;
    // column slices of 256: thread (gq, slot) sums column cs + slot over rows r0 + gq + 4 t of
    // this CTA's range with eight independent chains (~50 KB of U in flight per SM); the four
    // row groups are then added in group order — a fixed association, deterministic
    for (int cs = 0; cs < k; cs += 256) {
        const int c = cs + slot;
        double part = 0.0;
        if (c < k) {
            double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            int64_t i = r0 + gq;
            for (; i + 7 * kUtGroups < r1; i += 8 * kUtGroups) {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    acc[j] = fma(__ldcs(U + (i + j * kUtGroups) * ldu + c), __ldg(p + i + j * kUtGroups), acc[j]);
            }
            for (int j = 0; i < r1; i += kUtGroups, ++j) acc[j] = fma(__ldcs(U + i * ldu + c), __ldg(p + i), acc[j]);
            part = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
        }
        grp[gq][slot] = part;
        __syncthreads();
        if (gq == 0 && c < k)
            spart[(int64_t)blockIdx.x * k + c] = (grp[0][slot] + grp[1][slot]) + (grp[2][slot] + grp[3][slot]);
        __syncthreads();
    }
    if (pdot_vec) {                              // this CTA's part of sum_i h0_i p_i^2
        double hp = 0.0;
        for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) hp = fma(h0[i] * pdot_vec[i], pdot_vec[i], hp);
        const double b = block_sum(hp, red);
        if (threadIdx.x == 0) hpart[blockIdx.x] = b;
    }
    if (last_block(&sc->counters[cid])) {
        // s_c = sum over CTAs (eight interleaved chains b = j mod 8, then a fixed tree);
        // p^T H p = sum h0 p^2 + sum_c w_c s_c^2
        double wss = 0.0;
        for (int c = threadIdx.x; c < k; c += blockDim.x) {
            double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            const int G = (int)gridDim.x;
            int b = 0;
            for (; b + 7 < G; b += 8) {
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[j] += __ldcg(spart + (int64_t)(b + j) * k + c);
            }
            for (int j = 0; b < G; ++b, ++j) acc[j] += __ldcg(spart + (int64_t)b * k + c);
            const double t = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
            s[c] = t;
            wss = fma(w[c] * t, t, wss);
        }
        const double a = block_sum(wss, red);
        const double b = pdot_vec ? sum_partials(hpart, gridDim.x, red) : 0.0;
        if (threadIdx.x == 0) {
            sc->counters[cid] = 0;
            sc->S_H = b + a;
            if (sc->sharded) sc->loc[1] = b + a;
        }
    }
}

__global__ void __launch_bounds__(kCompactThreads)
k_compact_us(int n, int k, const double *__restrict__ U, int64_t ldu, const double *__restrict__ s,
             const double *__restrict__ w, const double *__restrict__ h0, const double *__restrict__ p,
             double *__restrict__ y, Scalars *sc, int mode) {
    extern __shared__ double ws[];               // k doubles: w o s
    if (mode == 1 && sc->done) return;
    for (int c = threadIdx.x; c < k; c += blockDim.x) ws[c] = w[c] * s[c];
    __syncthreads();
    const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    for (int i = blockIdx.x * wpb + (threadIdx.x >> 5); i < n; i += gridDim.x * wpb) {
        const double *u = U + (int64_t)i * ldu;
        double a = 0.0;
        for (int c = lane; c < k; c += 32) a = fma(__ldcs(u + c), ws[c], a);
        a = warp_sum(a);
        if (lane == 0) y[i] = fma(h0[i], p[i], a);
    }
}

// y-partials (ncb = 1) of H v; mode 1 (PCG): early exit on done and S_H = p^T H p.
void launch_compact_apply(const Prob &P, const double *v, const double *vdot, double *ypart, Scalars *sc, int mode,
                          int cid, cudaStream_t st) {
    if (P.n == 0) return;
    k_compact_ut<<<kCompactGrid, kUtThreads, 0, st>>>(P.n, P.ck, P.U, P.ldu, v, P.cspart, P.chpart, P.cs, P.h0,
                                                         P.w, vdot, sc, cid, mode);
    const int g2 = (int)std::min<int64_t>(kMaxGrid, (P.n + 7) / 8);
    k_compact_us<<<g2, kCompactThreads, sizeof(double) * (P.ck > 0 ? P.ck : 1), st>>>(P.n, P.ck, P.U, P.ldu, P.cs, P.w,
                                                                                     P.h0, v, ypart, sc, mode);
}

// diag(H)_j = h0_j + sum_c w_c U_jc^2   (cached once)
__global__ void k_compact_diag(int n, int k, const double *__restrict__ U, int64_t ldu, const double *__restrict__ h0,
                               const double *__restrict__ w, double *__restrict__ d) {
    const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
    for (int i = blockIdx.x * wpb + (threadIdx.x >> 5); i < n; i += gridDim.x * wpb) {
        double a = 0.0;
        for (int c = lane; c < k; c += 32) {
            const double u = U[(int64_t)i * ldu + c];
            a = fma(w[c] * u, u, a);
        }
        a = warp_sum(a);
        if (lane == 0) d[i] = h0[i] + a;
    }
}

void launch_compact_diag(const Prob &P, cudaStream_t st) {
    if (P.n == 0) return;
    k_compact_diag<<<(int)std::min<int64_t>(kMaxGrid, (P.n + 7) / 8), kBlock, 0, st>>>(P.n, P.ck, P.U, P.ldu, P.h0,
                                                                                      P.w, P.diagH);
}

// Rank-2 quasi-Newton update in compact form: append columns u, v with weights a, b (P:304:
// "each iteration adds two terms to the BFGS Hessian approximation").
__global__ void k_compact_append(int n, double *__restrict__ U, int64_t ldu, int col, const double *__restrict__ u,
                                 const double *__restrict__ v) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        U[(int64_t)i * ldu + col] = u[i];
        U[(int64_t)i * ldu + col + 1] = v[i];
    }
}

void launch_compact_append(const Prob &P, double *U, int col, const double *u, const double *v, cudaStream_t st) {
    k_compact_append<<<(int)std::min<int64_t>(kMaxGrid, (P.n + kBlock - 1) / kBlock), kBlock, 0, st>>>(P.n, U, P.ldu,
                                                                                                     col, u, v);
}


// Touch every kernel once (cudaFuncGetAttributes) so that CUDA's lazy module loading never
// has to load one while a peer-exchange wait kernel spins on the device (kernels.h).
template <class F>
static void touch_kernel(F f) {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(f));
}

void preload_compact() {
    touch_kernel(k_compact_ut); touch_kernel(k_compact_us); touch_kernel(k_compact_diag);
    touch_kernel(k_compact_append);
}

}  // namespace ipm
