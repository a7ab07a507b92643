// Does an L2-hit load wait behind the SM's outstanding DRAM loads?  Warp 0 of
// each CTA streams cp.async (or LDG) gathers from a large buffer; warp 1 times
// dependent relaxed loads of an L2-resident word (clock64 per load).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__global__ void k_bench(const double *big, size_t nbig, const unsigned long long *hot, long long *out, int mode) {
    __shared__ double land[32 * 64];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (w == 0) {
        if (mode == 0) return;
        // stream random-ish gathers (DRAM misses): 64 cp.async per lane in flight, repeated
        unsigned long long idx = (blockIdx.x * 7919ull + lane * 104729ull) % nbig;
        for (int r = 0; r < 2000; ++r) {
            for (int k = 0; k < 8; ++k) {
                idx = (idx * 6364136223846793005ull + 1442695040888963407ull) % nbig;
                const unsigned dst = (unsigned)__cvta_generic_to_shared(&land[(k * 32 + lane)]);
                if (mode == 1)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(big + idx) : "memory");
                else
                    land[k * 32 + lane] += big[idx];
            }
            if (mode == 1) asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 6;" ::: "memory");
        }
        if (mode == 1) asm volatile("cp.async.wait_group 0;" ::: "memory");
    } else if (w == 1) {
        // dependent chain of L2-hit relaxed loads
        unsigned long long v = 0;
        long long t0 = clock64();
        for (int i = 0; i < 2000; ++i) v = ld_relaxed(hot + (v & 1));
        long long t1 = clock64();
        if (lane == 0) out[blockIdx.x] = (t1 - t0) / 2000 + (long long)(v == 12345);
    }
}

int main() {
    const size_t nbig = 1ull << 28;     // 2 GiB of doubles
    double *big;
    unsigned long long *hot;
    long long *out, h[148];
    cudaMalloc(&big, nbig * sizeof(double));
    cudaMemset(big, 0, nbig * sizeof(double));
    cudaMalloc(&hot, 64);
    cudaMemset(hot, 0, 64);
    cudaMalloc(&out, 148 * sizeof(long long));
    const char *nm[] = {"idle SM", "cp.async DRAM gathers on the SM", "LDG DRAM gathers on the SM"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) k_bench<<<148, 64>>>(big, nbig, hot, out, mode);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
        long long s = 0;
        for (int i = 0; i < 148; ++i) s += h[i];
        printf("%-36s L2-hit relaxed load latency: %lld cycles (mean over SMs)\n", nm[mode], s / 148);
    }
    return 0;
}
