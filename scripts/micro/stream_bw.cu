// Micro-benchmark (experiment, not part of libipm): HBM read rate of the access patterns a
// symmetric fp64 GEMV can use on B200.  n x n row-major fp64 matrix (n = 20000, 3.2 GB):
//   full   : every CTA streams a contiguous slice with 16-B loads (upper bound for LDG reads)
//   tri    : upper block triangle, 256 x 256 tiles, contiguous tile ranges per CTA; warp reads
//            2 KB row segments (16 B per lane x 4 per row), ROWS rows in flight per warp
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o stream_bw stream_bw.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void k_full(const double2 *__restrict__ a, int64_t n2, double *out) {
    double s = 0.0;
    const int64_t per = (n2 + gridDim.x - 1) / gridDim.x;
    const int64_t b = per * blockIdx.x, e = min(n2, b + per);
    for (int64_t i = b + threadIdx.x; i < e; i += 4 * blockDim.x) {
        double2 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = (i + k * blockDim.x < e) ? __ldcs(a + i + k * blockDim.x) : make_double2(0, 0);
#pragma unroll
        for (int k = 0; k < 4; ++k) s += v[k].x + v[k].y;
    }
    if (s == 1.2345) out[0] = s;
}

template <int ROWS, int TB = 256>
__global__ void k_tri(const double *__restrict__ H, int n, int nb, double *out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int64_t nt = (int64_t)nb * (nb + 1) / 2;
    const int64_t t0 = nt * blockIdx.x / gridDim.x, t1 = nt * (blockIdx.x + 1) / gridDim.x;
    int I = 0, J = 0;
    {
        int64_t c = 0;
        while (c + (nb - I) <= t0) { c += nb - I; ++I; }
        J = I + (int)(t0 - c);
    }
    double s = 0.0;
    for (int64_t t = t0; t < t1; ++t) {
        const int r0 = I * TB, c0 = J * TB;
        const int rows = min(TB, n - r0), cols = min(TB, n - c0);
        constexpr int KV = TB / 64;                 // 16-B loads per lane per row
        for (int r = warp * ROWS; r < rows; r += nw * ROWS) {
            double2 v[ROWS][KV];
#pragma unroll
            for (int q = 0; q < ROWS; ++q) {
                const double2 *row = reinterpret_cast<const double2 *>(H + (int64_t)(r0 + r + q) * n + c0);
#pragma unroll
                for (int k = 0; k < KV; ++k) {
                    const int col = 2 * (lane + 32 * k);
                    v[q][k] = (r + q < rows && col < cols) ? __ldcs(row + lane + 32 * k) : make_double2(0, 0);
                }
            }
#pragma unroll
            for (int q = 0; q < ROWS; ++q)
#pragma unroll
                for (int k = 0; k < KV; ++k) s += v[q][k].x * v[q][k].y;
        }
        if (++J == nb) { ++I; J = I; }
    }
    if (s == 1.2345) out[0] = s;
}

int main(int argc, char **argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 20000;
    double *H, *out;
    cudaMalloc(&H, (size_t)n * n * 8);
    cudaMalloc(&out, 8);
    cudaMemset(H, 0, (size_t)n * n * 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int nb = (n + 255) / 256, nb2 = (n + 511) / 512;
    double tri = 0, tri2 = 0;
    for (int i = 0; i < nb; ++i) for (int j = i; j < nb; ++j) tri += (double)std::min(256, n - i * 256) * std::min(256, n - j * 256);
    for (int i = 0; i < nb2; ++i) for (int j = i; j < nb2; ++j) tri2 += (double)std::min(512, n - i * 512) * std::min(512, n - j * 512);
    auto run = [&](const char *name, double bytes, auto launch) {
        for (int w = 0; w < 3; ++w) launch();
        cudaEventRecord(e0);
        for (int r = 0; r < 20; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"kernel\": \"%s\", \"us\": %.1f, \"GBps\": %.0f, \"err\": \"%s\"}\n", name, ms / 20 * 1e3,
               bytes / (ms / 20 * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    };
    for (int cps : {1, 2, 4, 8})
        for (int thr : {256, 512}) {
            char nm[64];
            snprintf(nm, 64, "full cps=%d thr=%d", cps, thr);
            run(nm, (double)n * n * 8, [&] { k_full<<<sms * cps, thr>>>((const double2 *)H, (int64_t)n * n / 2, out); });
        }
    for (int cps : {1, 2})
        for (int thr : {512, 1024}) {
            char nm[64];
            snprintf(nm, 64, "tri512 R2 cps=%d thr=%d", cps, thr);
            run(nm, tri2 * 8, [&] { k_tri<2, 512><<<sms * cps, thr>>>(H, n, nb2, out); });
            snprintf(nm, 64, "tri512 R4 cps=%d thr=%d", cps, thr);
            run(nm, tri2 * 8, [&] { k_tri<4, 512><<<sms * cps, thr>>>(H, n, nb2, out); });
        }
    for (int cps : {1, 2, 4})
        for (int thr : {512, 1024}) {
            char nm[64];
            snprintf(nm, 64, "tri R2 cps=%d thr=%d", cps, thr);
            run(nm, tri * 8, [&] { k_tri<2><<<sms * cps, thr>>>(H, n, nb, out); });
            snprintf(nm, 64, "tri R4 cps=%d thr=%d", cps, thr);
            run(nm, tri * 8, [&] { k_tri<4><<<sms * cps, thr>>>(H, n, nb, out); });
        }
    return 0;
}
