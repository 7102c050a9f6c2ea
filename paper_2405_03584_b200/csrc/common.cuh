// common.cuh — shared device helpers of libipm.so (sm_100a).
//
// Determinism contract ("bitwise reproducible"): every floating-point
// reduction below has a fixed association order that depends only on the launch shape
// (grid/block size, which are functions of the problem dimensions), never on timing:
// lane-strided partial sums -> xor-shuffle tree -> per-warp slots in shared memory summed
// in warp order -> per-block partials summed in block order by the last block to finish.
// No floating-point atomics anywhere.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace ipm {

constexpr int kWarp = 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Sum over a group of G consecutive lanes (G power of two <= 32); all lanes get the result.
template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Lane gl's part of a GEMV tile-partial row sum: row[gl] + row[gl + G] + ... added in that
// order, with four loads in flight per trip (bitwise the plain strided loop).
template <int G>
__device__ __forceinline__ double row_part_sum(const double *__restrict__ row, int gl, int ncb) {
    double s = 0.0;
    int c = gl;
    for (; c + 3 * G < ncb; c += 4 * G) {
        const double a0 = row[c], a1 = row[c + G], a2 = row[c + 2 * G], a3 = row[c + 3 * G];
        s += a0;
        s += a1;
        s += a2;
        s += a3;
    }
    for (; c < ncb; c += G) s += row[c];
    return s;
}

// Block-wide sum; result valid in ALL threads.  `sh` needs blockDim/32 doubles.
__device__ __forceinline__ double block_sum(double v, double *sh) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncwarp();                             // reconverged warp at the barrier (synccheck)
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double t = 0.0;
    for (int i = 0; i < nw; ++i) t += sh[i];  // fixed order, every thread
    return t;
}

__device__ __forceinline__ double block_min(double v, double *sh) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_min(v);
    __syncwarp();
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double t = sh[0];
    for (int i = 1; i < nw; ++i) t = fmin(t, sh[i]);
    return t;
}

__device__ __forceinline__ double block_max(double v, double *sh) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_max(v);
    __syncwarp();
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double t = sh[0];
    for (int i = 1; i < nw; ++i) t = fmax(t, sh[i]);
    return t;
}

// "Last block done" election (threadfence-reduction pattern).  Every block calls it after
// writing its partials; exactly one block (the last to arrive) gets true and must reset the
// counter.  The reduction order over partials is then fixed (block order), so which block
// happens to be last does not change the bits.
__device__ __forceinline__ bool last_block(unsigned int *counter) {
    __shared__ bool am_last;
    __threadfence();
    __syncwarp();
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int prev = atomicAdd(counter, 1u);
        am_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (am_last) __threadfence();
    return am_last;
}

// Read-only loads with an L2 evict_last priority: the PCG's sparse matrices (A, A^T: 24 MB at
// C3) are re-read every iteration while the symmetric GEMV streams H evict_first past them.
__device__ __forceinline__ uint64_t keep_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ double ld_keep(const double *p, uint64_t pol) {
    double v;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int ld_keep(const int *p, uint64_t pol) {
    int v;
    asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

__device__ __forceinline__ double2 ld_keep2(const double *p, uint64_t pol) {     // 16-B aligned
    double2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int2 ld_keep2(const int *p, uint64_t pol) {           // 8-B aligned
    int2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
    return v;
}

// Dot of one CSR row with a dense vector x by one group of G lanes, 16-B column-pair loads
// (experiment IPM_SPMV_VEC): an odd leading entry is taken by lane 0 first, then lane l folds the
// pairs starting at a + 2l, a + 2l + 2G, ... (four in flight per trip), then an odd trailing
// entry — a fixed order for a given row and G.
template <int G>
__device__ __forceinline__ double row_dot_pairs(const int *__restrict__ col, const double *__restrict__ val,
                                                const double *__restrict__ x, int64_t s, int64_t e, int gl,
                                                uint64_t pol) {
    double acc = 0.0;
    if ((s & 1) && s < e) {
        if (gl == 0) acc = ld_keep(val + s, pol) * __ldg(x + ld_keep(col + s, pol));
        ++s;
    }
    int64_t k = s + 2 * gl;
    for (; k + 1 + 6 * G < e; k += 8 * G) {
        const int2 c0 = ld_keep2(col + k, pol), c1 = ld_keep2(col + k + 2 * G, pol);
        const int2 c2 = ld_keep2(col + k + 4 * G, pol), c3 = ld_keep2(col + k + 6 * G, pol);
        const double2 w0 = ld_keep2(val + k, pol), w1 = ld_keep2(val + k + 2 * G, pol);
        const double2 w2 = ld_keep2(val + k + 4 * G, pol), w3 = ld_keep2(val + k + 6 * G, pol);
        const double x0 = __ldg(x + c0.x), y0 = __ldg(x + c0.y), x1 = __ldg(x + c1.x), y1 = __ldg(x + c1.y);
        const double x2 = __ldg(x + c2.x), y2 = __ldg(x + c2.y), x3 = __ldg(x + c3.x), y3 = __ldg(x + c3.y);
        acc = fma(w0.x, x0, acc);
        acc = fma(w0.y, y0, acc);
        acc = fma(w1.x, x1, acc);
        acc = fma(w1.y, y1, acc);
        acc = fma(w2.x, x2, acc);
        acc = fma(w2.y, y2, acc);
        acc = fma(w3.x, x3, acc);
        acc = fma(w3.y, y3, acc);
    }
    for (; k + 1 < e; k += 2 * G) {
        const int2 c = ld_keep2(col + k, pol);
        const double2 w = ld_keep2(val + k, pol);
        acc = fma(w.x, __ldg(x + c.x), acc);
        acc = fma(w.y, __ldg(x + c.y), acc);
    }
    if (k < e) acc = fma(ld_keep(val + k, pol), __ldg(x + ld_keep(col + k, pol)), acc);
    return acc;
}

// Device-side launch timer (ns, %globaltimer): the PCG's dominant kernel records the
// earliest CTA start and, in its last CTA, adds (end - start) to a running sum, so bench.py
// reads the kernel's average launch duration over the timed region without splitting the
// captured graph (CUDA events cannot bracket a node inside a conditional WHILE body).
__device__ __forceinline__ unsigned long long gtimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void ktimer_start(unsigned long long *neg) {
    if (threadIdx.x == 0) atomicMax(neg, ~gtimer_ns());
}
__device__ __forceinline__ void ktimer_stop(unsigned long long *neg, unsigned long long *ns, unsigned long long *cnt) {
    const unsigned long long e = gtimer_ns();
    const unsigned long long s = ~atomicExch(neg, 0ull);
    if (e > s) *ns += e - s;
    *cnt += 1;
}

#ifdef IPM_TIMELINE
#define TL_BEGIN(sc, k) do { if (threadIdx.x == 0) atomicMax(&(sc)->tl[k][0], ~gtimer_ns()); } while (0)
#define TL_END(sc, k) do { if (threadIdx.x == 0) atomicMax(&(sc)->tl[k][1], gtimer_ns()); } while (0)
#else
#define TL_BEGIN(sc, k) do { } while (0)
#define TL_END(sc, k) do { } while (0)
#endif

// Grid-wide barrier for cooperatively launched kernels (all CTAs co-resident): arrival
// counter + generation word.  The generation is read BEFORE arriving, so the last arrival's
// increment cannot be missed; fences order every CTA's prior global writes before release.
__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int *p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void grid_barrier(unsigned int *count, unsigned int *gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int g = ld_acquire_u32(gen);
        __threadfence();
        if (atomicAdd(count, 1u) == gridDim.x - 1) {
            *(volatile unsigned int *)count = 0u;
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (ld_acquire_u32(gen) == g) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// Fixed-order sum of `cnt` partials by one block (all threads get it).
__device__ __forceinline__ double sum_partials(const double *part, int cnt, double *sh) {
    double v = 0.0;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) v += ((volatile const double *)part)[i];
    return block_sum(v, sh);
}

// Two fixed-order sums in one pass (one round of loads, one block reduction): bitwise equal to
// two sum_partials calls (same per-thread order, same shuffle tree, same warp order).
// sh2 holds 2 * (blockDim.x / 32) doubles.
__device__ __forceinline__ void sum_partials2(const double *p, const double *q, int cnt, double *sh2, double &a,
                                              double &b) {
    double u = 0.0, v = 0.0;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
        u += ((volatile const double *)p)[i];
        v += ((volatile const double *)q)[i];
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        u += __shfl_xor_sync(0xffffffffu, u, o);
        v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    __syncthreads();
    if (lane == 0) {
        sh2[wid] = u;
        sh2[nw + wid] = v;
    }
    __syncthreads();
    double x = 0.0, y = 0.0;
    for (int i = 0; i < nw; ++i) {
        x += sh2[i];
        y += sh2[nw + i];
    }
    a = x;
    b = y;
}

__device__ __forceinline__ double min_partials(const double *part, int cnt, double *sh) {
    double v = INFINITY;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) v = fmin(v, ((volatile const double *)part)[i]);
    return block_min(v, sh);
}

__device__ __forceinline__ double max_partials(const double *part, int cnt, double *sh) {
    double v = 0.0;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) v = fmax(v, ((volatile const double *)part)[i]);
    return block_max(v, sh);
}

__device__ __forceinline__ bool finite_d(double v) { return fabs(v) <= 1.7976931348623157e308; }

}  // namespace ipm
