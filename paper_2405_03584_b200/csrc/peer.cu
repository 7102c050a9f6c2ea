// peer.cu — the peer-memory data plane of the row-sharded path (see peer.h).
#include <algorithm>

#include "common.cuh"
#include "finalize.cuh"
#include "kernels.h"
#include "peer.h"
#include "state.h"

namespace ipm {

PeerLayout peer_layout(int64_t ncols, int64_t m, int nranks) {
    const int64_t chunk = (ncols + nranks - 1) / nranks;
    auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
    PeerLayout L;
    size_t off = 0;
    L.gfull = off;
    off += up(sizeof(double) * ((size_t)chunk * nranks + 2));
    L.zall = off;
    off += up(sizeof(double) * (size_t)chunk * nranks);
    L.xall = off;
    off += up(sizeof(double) * 8 * (size_t)nranks * kPeerX);
    L.tall = off;
    off += up(sizeof(double) * (size_t)std::max<int64_t>(m, 1));
    L.flags = off;
    off += up(sizeof(unsigned long long) * kPeerMax * kPeerCh);
    L.bytes = off;
    return L;
}

namespace {

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// End of a put kernel: every CTA's stores are fenced at system scope; the last CTA to arrive
// raises this rank's flag in every peer's region to the exchange's sequence number.
__device__ __forceinline__ unsigned long long *flag_ptr(const PeerArgs &pa, int r, int ch, int sender) {
    return reinterpret_cast<unsigned long long *>(pa.base[r] + pa.L.flags) + ch * kPeerMax + sender;
}

__device__ __forceinline__ void put_signal(const PeerArgs &pa, Scalars *sc, unsigned long long seq, int ch) {
    __shared__ bool am_last;
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) am_last = (atomicAdd(&sc->peer_ctr[ch], 1u) == gridDim.x - 1);
    __syncthreads();
    if (!am_last) return;
    if (threadIdx.x == 0) {
        sc->peer_ctr[ch] = 0;
        __threadfence_system();
        for (int r = 0; r < pa.P; ++r) st_release_sys(flag_ptr(pa, r, ch, pa.rank), seq);
    }
}

__global__ void k_peer_put_vec(PeerArgs pa, const double *__restrict__ src, int64_t count, size_t dst_off,
                               int64_t dst_base, int ch, Scalars *sc, int check_done) {
    if (check_done && sc->done) return;
    const unsigned long long seq = sc->peer_seq[ch] + 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = src[i];
        for (int r = 0; r < pa.P; ++r) reinterpret_cast<double *>(pa.base[r] + dst_off)[dst_base + i] = v;
    }
    put_signal(pa, sc, seq, ch);
}

__global__ void k_peer_put_loc(PeerArgs pa, int stage, Scalars *sc, int check_done) {
    if (check_done && sc->done) return;
    const unsigned long long seq = sc->peer_seq[0] + 1;
    const int k = threadIdx.x;
    if (k < 8) {
        const double v = sc->loc[k];
        for (int r = 0; r < pa.P; ++r)
            reinterpret_cast<double *>(pa.base[r] + pa.L.xall)[((size_t)stage * pa.P + pa.rank) * 8 + k] = v;
    }
    put_signal(pa, sc, seq, 0);
}

__global__ void k_peer_zput(PeerArgs pa, int zrows, int ldz, const double *__restrict__ zpart,
                            const int *__restrict__ zcol, Scalars *sc, int check_done) {
    if (check_done && sc->done) return;
    const unsigned long long seq = sc->peer_seq[0] + 1;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < zrows; q += gridDim.x * blockDim.x) {
        const double *z = zpart + (int64_t)q * ldz;
        double s = 0.0;
        for (int k = 0; k < ldz; ++k) s += z[k];           // slot order (k_zreduce's association)
        const int col = zcol[q];
        const int b = (int)(col / pa.chunk);
        reinterpret_cast<double *>(pa.base[b] + pa.L.zall)[pa.rank * pa.chunk + (col - (int64_t)b * pa.chunk)] = s;
    }
    put_signal(pa, sc, seq, 0);
}

__global__ void k_peer_wait(PeerArgs pa, Scalars *sc, int stage, double p0, double p1, int64_t p2, int check_done,
                            cudaGraphConditionalHandle h, int use_cond, int ch) {
    if (check_done && sc->done) {
        if (use_cond && threadIdx.x == 0) cudaGraphSetConditional(h, 0);
        return;
    }
    const unsigned long long seq = sc->peer_seq[ch] + 1;
    __shared__ int timed_out;
    if (threadIdx.x == 0) timed_out = 0;
    __syncthreads();
    const int r = threadIdx.x;
    if (r < pa.P) {
        const unsigned long long *f = flag_ptr(pa, pa.rank, ch, r);
        const unsigned long long t0 = gtimer_ns();
        unsigned int spins = 0;
        unsigned long long v;
        while ((v = ld_acquire_sys(f)) < seq) {
            if ((++spins & 1023u) == 0 && gtimer_ns() - t0 > pa.timeout_ns) {   // a peer is gone
                timed_out = 1;
                sc->peer_diag[0] = seq;          // diagnostics for the host's error message
                sc->peer_diag[1] = (unsigned long long)r;
                sc->peer_diag[2] = v;
                sc->peer_diag[3] = (unsigned long long)stage + 1000ull;
                break;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    sc->peer_seq[ch] = seq;
    if (timed_out) {
        sc->peer_timeout = 1;
        sc->done = 1;
        sc->breakdown = 1;
        if (use_cond) cudaGraphSetConditional(h, 0);
        return;
    }
    if (stage >= 0) {
        const double *xa = reinterpret_cast<const double *>(pa.base[pa.rank] + pa.L.xall) + (size_t)stage * pa.P * 8;
        xcombine_apply(sc, xa, pa.P, stage, p0, p1, p2);
    }
    if (use_cond) cudaGraphSetConditional(h, sc->done ? 0u : 1u);
}

__global__ void k_peer_zfold(PeerArgs pa, int nloc, double *__restrict__ ypart, int ldy, Scalars *sc,
                             int check_done) {
    if (check_done && sc->done) return;
    const double *zall = reinterpret_cast<const double *>(pa.base[pa.rank] + pa.L.zall);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nloc; i += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < pa.P; ++r) s += zall[(int64_t)r * pa.chunk + i];   // rank order (k_zfold's)
        ypart[(int64_t)i * ldy + ldy - 1] = s;
    }
}

}  // namespace

void launch_peer_put_vec(const PeerArgs &pa, const double *src, int64_t count, size_t dst_off, int64_t dst_base,
                         int ch, Scalars *sc, int check_done, cudaStream_t st) {
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(kMaxGrid, (count + 255) / 256));
    k_peer_put_vec<<<grid, 256, 0, st>>>(pa, src, count, dst_off, dst_base, ch, sc, check_done);
}

void launch_peer_put_loc(const PeerArgs &pa, int stage, Scalars *sc, int check_done, cudaStream_t st) {
    k_peer_put_loc<<<1, 32, 0, st>>>(pa, stage, sc, check_done);
}

void launch_peer_zput(const PeerArgs &pa, int zrows, int ldz, const double *zpart, const int *zcol, Scalars *sc,
                      int check_done, cudaStream_t st) {
    const int grid = std::max(1, std::min(kMaxGrid, (zrows + 255) / 256));
    k_peer_zput<<<grid, 256, 0, st>>>(pa, zrows, ldz, zpart, zcol, sc, check_done);
}

void launch_peer_wait(const PeerArgs &pa, Scalars *sc, int stage, double p0, double p1, int64_t p2, int check_done,
                      cudaGraphConditionalHandle h, int use_cond, cudaStream_t st, int ch) {
    k_peer_wait<<<1, 32, 0, st>>>(pa, sc, stage, p0, p1, p2, check_done, h, use_cond, ch);
}

void launch_peer_zfold(const PeerArgs &pa, int nloc, double *ypart, int ldy, Scalars *sc, int check_done,
                       cudaStream_t st) {
    k_peer_zfold<<<std::max(1, std::min(kMaxGrid, (nloc + 255) / 256)), 256, 0, st>>>(pa, nloc, ypart, ldy, sc,
                                                                                       check_done);
}


// Touch every kernel once (cudaFuncGetAttributes) so that CUDA's lazy module loading never
// has to load one while a peer-exchange wait kernel spins on the device (kernels.h).
template <class F>
static void touch_kernel(F f) {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(f));
}

void preload_peer() {
    touch_kernel(k_peer_put_vec); touch_kernel(k_peer_put_loc); touch_kernel(k_peer_zput);
    touch_kernel(k_peer_wait); touch_kernel(k_peer_zfold);
}

}  // namespace ipm
