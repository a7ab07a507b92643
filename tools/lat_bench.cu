// Dependent-chain latencies on one warp (clock64), for the BLOCK step model:
// DFMA, DMUL, 64-bit SHFL.IDX, SHFL+DFMA, LDS, FSEL.  nvcc -arch=sm_100a -O3 lat_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4096;

__global__ void k_lat(double *out, long long *cyc, int src) {
    const int lane = threadIdx.x & 31;
    __shared__ double sm[64];
    sm[lane] = 1.0 + lane;
    sm[32 + lane] = 0.5;
    __syncwarp();
    double x = 1.0 + lane * 1e-3, a = 0.999999, b = 1e-7;
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) x = fma(x, a, b);
    t1 = clock64();
    if (lane == 0) cyc[0] = t1 - t0;
    // DMUL chain
    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) x = x * a;
    t1 = clock64();
    if (lane == 0) cyc[1] = t1 - t0;
    // 64-bit shuffle chain (source lane from a register)
    int s = (lane + src) & 31;
    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, s);
    t1 = clock64();
    if (lane == 0) cyc[2] = t1 - t0;
    // shuffle -> DFMA (the BLOCK step chain)
    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) x = fma(-a, __shfl_sync(0xffffffffu, x, s), b);
    t1 = clock64();
    if (lane == 0) cyc[3] = t1 - t0;
    // shuffle -> FSEL -> 3 DFMA -> DMUL (one step, 3 terms, select on each)
    const bool p0 = (lane & 1) != 0, p1 = (lane & 2) != 0, p2 = (lane & 4) != 0;
    const double e0 = 0.25, e1 = 0.125, e2 = 0.0625;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N / 4; ++i) {
        const double h0 = __shfl_sync(0xffffffffu, x, s);
        const double h1 = __shfl_sync(0xffffffffu, x, s + 1);
        const double h2 = __shfl_sync(0xffffffffu, x, s + 2);
        double acc = fma(-a, p0 ? e0 : h0, b);
        acc = fma(-a, p1 ? e1 : h1, acc);
        acc = fma(-a, p2 ? e2 : h2, acc);
        x = acc * 0.9;
    }
    t1 = clock64();
    if (lane == 0) cyc[4] = (t1 - t0) * 4;
    // LDS chain (address from loaded value)
    int idx = lane;
    t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) idx = (int)sm[idx & 63] & 31;
    t1 = clock64();
    if (lane == 0) cyc[5] = t1 - t0;
    out[threadIdx.x] = x + idx;
}

int main() {
    double *out;
    long long *cyc, h[8];
    cudaMalloc(&out, 1024 * sizeof(double));
    cudaMalloc(&cyc, 8 * sizeof(long long));
    for (int r = 0; r < 2; ++r) k_lat<<<1, 32>>>(out, cyc, 1);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const char *nm[] = {"DFMA", "DMUL", "SHFL.64", "SHFL->DFMA", "step(3 SHFL,FSEL,3 DFMA,DMUL)/4", "LDS->cvt"};
    for (int i = 0; i < 6; ++i) printf("%-34s %.2f cycles per op\n", nm[i], (double)h[i] / N);
    return 0;
}
