// tools/microbench.cu -- latency/bandwidth probes that calibrate the SpTRSV
// design (hard part H1).  Not part of the product.
//   1. cross-SM flag handoff (ping-pong), relaxed value-as-flag vs release/acquire
//   2. fence.acq_rel.gpu cost
//   3. intra-CTA step cost: LDS -> DFMA chain -> STS -> __syncthreads
//   4. single-SM streaming bandwidth (LDG, various in-flight depths)
//   5. L2 / DRAM pointer-chase latency
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ int ldr(const int *p) { int v; asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ int lda(const int *p) { int v; asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void str(int *p, int v) { asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ void stl(int *p, int v) { asm volatile("st.release.gpu.global.b32 [%0], %1;" :: "l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ unsigned smid() { unsigned r; asm("mov.u32 %0, %%smid;" : "=r"(r)); return r; }

// ping-pong between block 0 and block `other` (different SMs): mode 0 relaxed, 1 release/acquire,
// 2 relaxed + explicit fence on both sides
__global__ void k_pingpong(int *flag, int iters, int mode, unsigned long long *out, unsigned *sms) {
    if (threadIdx.x != 0) return;
    int me = blockIdx.x;   // 0 or 1
    if (me == 0) sms[0] = smid(); else sms[1] = smid();
    unsigned long long t0 = gtime();
    for (int i = 0; i < iters; ++i) {
        int want = 2 * i + me;          // block 0 waits for even values, writes odd
        if (mode == 1) { while (lda(flag) != want) {} stl(flag, want + 1); }
        else if (mode == 0) { while (ldr(flag) != want) {} str(flag, want + 1); }
        else { while (ldr(flag) != want) {} asm volatile("fence.acq_rel.gpu;" ::: "memory"); asm volatile("fence.acq_rel.gpu;" ::: "memory"); str(flag, want + 1); }
    }
    unsigned long long t1 = gtime();
    if (me == 0) out[0] = t1 - t0;
}

// fence cost: each thread does `iters` fences, with or without a preceding store
__global__ void k_fence(int *buf, int iters, int with_store, unsigned long long *out) {
    unsigned long long t0 = gtime();
    for (int i = 0; i < iters; ++i) {
        if (with_store) buf[(blockIdx.x * blockDim.x + threadIdx.x) * 8 + (i & 7)] = i;
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    unsigned long long t1 = gtime();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

// intra-CTA level step: each thread reads 3 smem values written in the previous step, DFMA chain, writes.
__global__ void k_step(int steps, double *sink, unsigned long long *out) {
    extern __shared__ double xs[];
    const int T = blockDim.x;
    const int t = threadIdx.x;
    xs[t] = 1.0 + t;
    xs[T + t] = 0.5;
    __syncthreads();
    unsigned long long t0 = gtime();
    double acc = 0;
    for (int s = 0; s < steps; ++s) {
        const double *prev = xs + (s & 1) * T;
        double *cur = xs + ((s + 1) & 1) * T;
        double v = 0.25;
        v = fma(-0.1, prev[(t + 1) % T], v);
        v = fma(-0.1, prev[(t + 7) % T], v);
        v = fma(-0.1, prev[(t + 31) % T], v);
        cur[t] = v * 0.5;
        __syncthreads();
    }
    unsigned long long t1 = gtime();
    acc = xs[t];
    if (t == 0) { out[blockIdx.x] = t1 - t0; sink[blockIdx.x] = acc; }
}

// single-SM streaming read bandwidth: one CTA (1024 threads) reads `bytes` with 16B loads, `unroll` in flight
template <int U>
__global__ void k_stream(const int4 *src, long n16, unsigned long long *out, int *sink) {
    unsigned long long t0 = gtime();
    int acc = 0;
    long i = threadIdx.x;
    const long stride = blockDim.x;
    for (; i + (U - 1) * stride < n16; i += U * stride) {
        int4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].w;
    }
    __syncthreads();
    unsigned long long t1 = gtime();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    if (acc == 0x12345) sink[0] = acc;
}

// pointer chase latency
__global__ void k_chase(const int *next, int hops, unsigned long long *out, int *sink) {
    int p = 0;
    unsigned long long t0 = gtime();
    for (int i = 0; i < hops; ++i) p = __ldcg(next + p);
    unsigned long long t1 = gtime();
    out[0] = t1 - t0;
    sink[0] = p;
}

int main() {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    printf("{\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"results\": {\n", prop.name, prop.multiProcessorCount, prop.l2CacheSize);
    int *flag; unsigned long long *out; unsigned *sms; int *sink; double *dsink;
    CK(cudaMalloc(&flag, 64 << 20)); CK(cudaMalloc(&out, 4096)); CK(cudaMalloc(&sms, 64)); CK(cudaMalloc(&sink, 64)); CK(cudaMalloc(&dsink, 8 * 4096));
    unsigned long long h[148];
    unsigned hs[2];
    const int iters = 20000;
    const char *names[3] = {"relaxed", "release_acquire", "relaxed_plus_2fences"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int other : {1, 74, 147}) {
            // launch `other+1` blocks but only blocks 0 and `other` participate: use a grid of 2 with spread via large grid
            CK(cudaMemset(flag, 0, 4));
            k_pingpong<<<2, 32>>>(flag, iters, mode, out, sms);
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(hs, sms, 8, cudaMemcpyDeviceToHost));
            printf("  \"pingpong_%s_%d\": {\"one_way_ns\": %.1f, \"sm\": [%u, %u]},\n", names[mode], other, (double)h[0] / (2.0 * iters), hs[0], hs[1]);
            break;  // grid of 2: the placement is the scheduler's
        }
    }
    for (int ws = 0; ws < 2; ++ws) {
        for (int blocks : {1, 148, 592}) {
            k_fence<<<blocks, 256>>>(flag, 1000, ws, out);
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost));
            printf("  \"fence_%s_blocks%d\": {\"ns_per_fence\": %.1f},\n", ws ? "after_store" : "no_store", blocks, h[0] / 1000.0);
        }
    }
    for (int T : {128, 256, 512, 1024}) {
        k_step<<<1, T, 2 * T * 8>>>(10000, dsink, out);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost));
        printf("  \"cta_step_T%d\": {\"ns_per_step\": %.1f},\n", T, h[0] / 10000.0);
        k_step<<<148, T, 2 * T * 8>>>(10000, dsink, out);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost));
        printf("  \"cta_step_T%d_148ctas\": {\"ns_per_step\": %.1f},\n", T, h[0] / 10000.0);
    }
    long nbytes = 256L << 20;
    int4 *src; CK(cudaMalloc(&src, nbytes)); CK(cudaMemset(src, 1, nbytes));
    for (int rep = 0; rep < 2; ++rep) {
        long n16 = (64L << 20) / 16;    // 64 MiB from one SM
        k_stream<1><<<1, 1024>>>(src, n16, out, sink); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost));
        if (rep) printf("  \"sm_stream_u1\": {\"GBps\": %.1f},\n", (64.0 * (1 << 20)) / h[0]);
        k_stream<4><<<1, 1024>>>(src, n16, out, sink); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost));
        if (rep) printf("  \"sm_stream_u4\": {\"GBps\": %.1f},\n", (64.0 * (1 << 20)) / h[0]);
        k_stream<8><<<1, 1024>>>(src, n16, out, sink); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost));
        if (rep) printf("  \"sm_stream_u8\": {\"GBps\": %.1f},\n", (64.0 * (1 << 20)) / h[0]);
        k_stream<16><<<1, 1024>>>(src, n16, out, sink); CK(cudaDeviceSynchronize()); CK(cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost));
        if (rep) printf("  \"sm_stream_u16\": {\"GBps\": %.1f},\n", (64.0 * (1 << 20)) / h[0]);
    }
    // pointer chase: small (L2-resident) and large (DRAM) footprints, random cyclic permutation
    for (long foot : {1L << 20, 1L << 30}) {
        long n = foot / 4;
        std::vector<int> nxt(n);
        // stride permutation with a large odd step (touches distinct lines)
        long step = 4099 * 32 + 1;
        for (long i = 0; i < n; ++i) nxt[i] = (int)((i + step) % n);
        int *dn; CK(cudaMalloc(&dn, foot)); CK(cudaMemcpy(dn, nxt.data(), foot, cudaMemcpyHostToDevice));
        k_chase<<<1, 1>>>(dn, 2000, out, sink); CK(cudaDeviceSynchronize());
        k_chase<<<1, 1>>>(dn, 20000, out, sink); CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost));
        printf("  \"chase_%ldMiB\": {\"ns_per_hop\": %.1f},\n", foot >> 20, h[0] / 20000.0);
        cudaFree(dn);
    }
    printf("  \"end\": 0\n}}\n");
    return 0;
}
