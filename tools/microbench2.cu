// tools/microbench2.cu -- per-primitive costs for the single-warp step loop of
// SPTRSV_ALGO_BLOCK (cycles, one warp, clock64).  Not part of the product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1710_04985_b200/csrc/common.cuh"

using namespace sptrsv;

__global__ void k_prims(const double *g, double *gout, long long *out) {
    __shared__ __align__(16) unsigned char sm[32768];
    __shared__ uint64_t bar[4];
    double *xs = reinterpret_cast<double *>(sm);
    const int lane = threadIdx.x;
    for (int i = lane; i < 4096; i += 32) xs[i] = 1.0 + i;
    if (lane == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const int N = 1000;
    long long t0, t1;
    // 1. mbarrier try_wait on a completed phase
    if (lane == 0) { mbar_arrive_expect_tx(&bar[0], 0); }
    __syncwarp();
    t0 = clock64();
    unsigned acc = 0;
    for (int i = 0; i < N; ++i) acc += mbar_try_wait(&bar[0], 0);
    t1 = clock64();
    if (lane == 0) out[0] = (t1 - t0) / N;
    // 2. test_wait
    t0 = clock64();
    for (int i = 0; i < N; ++i) acc += mbar_test_wait(&bar[0], 0);
    t1 = clock64();
    if (lane == 0) out[1] = (t1 - t0) / N;
    // 3. dependent LDS chain
    int idx = lane;
    t0 = clock64();
    for (int i = 0; i < N; ++i) idx = (int)xs[idx & 4095] & 31;
    t1 = clock64();
    if (lane == 0) out[2] = (t1 - t0) / N;
    // 4. STS + __syncwarp + dependent LDS (one "level" of intra-warp handoff)
    double v = 1.0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) {
        xs[(i & 63) * 32 + lane] = v;
        __syncwarp();
        v = xs[(i & 63) * 32 + ((lane + 1) & 31)] * 0.5 + 1.0;
    }
    t1 = clock64();
    if (lane == 0) out[3] = (t1 - t0) / N;
    // 5. DFMA dependent chain (3 FMAs + 1 MUL per "row")
    double a = 1.0;
    t0 = clock64();
    for (int i = 0; i < N; ++i) { a = fma(-0.1, a, 1.0); a = fma(-0.1, a, 1.0); a = fma(-0.1, a, 1.0); a *= 0.9; }
    t1 = clock64();
    if (lane == 0) out[4] = (t1 - t0) / N;
    // 6. bulk copy issue + wait (global -> smem, 1.5 KB), latency
    t0 = clock64();
    for (int i = 0; i < 50; ++i) {
        const int slot = 1 + (i & 1);
        if (lane == 0) {
            mbar_arrive_expect_tx(&bar[slot], 1536);
            bulk_g2s(sm + 16384 + slot * 2048, g + (i * 192) % 100000, 1536, &bar[slot]);
        }
        mbar_wait(&bar[slot], (i >> 1) & 1);
    }
    t1 = clock64();
    if (lane == 0) out[5] = (t1 - t0) / 50;
    // 7. st.relaxed.gpu store issue cost
    t0 = clock64();
    for (int i = 0; i < N; ++i) st_relaxed_val(gout + (i & 255) * 32 + lane, a);
    t1 = clock64();
    if (lane == 0) out[6] = (t1 - t0) / N;
    // 8. L2-hit load latency (ld.relaxed.gpu, dependent)
    int j = lane;
    t0 = clock64();
    for (int i = 0; i < 200; ++i) j = ((int)ld_relaxed_val(g + j) + i) & 1023;
    t1 = clock64();
    if (lane == 0) out[7] = (t1 - t0) / 200;
    // 9. cp.async 8B + commit + wait_group 0 (latency)
    t0 = clock64();
    for (int i = 0; i < 200; ++i) {
        cp_async_8(xs + 2048 + lane, g + ((i * 37 + lane) & 1023));
        cp_async_commit();
        cp_async_wait<0>();
    }
    t1 = clock64();
    if (lane == 0) out[8] = (t1 - t0) / 200;
    // 10. volatile LDS poll (already-set value)
    t0 = clock64();
    double sum = 0;
    for (int i = 0; i < N; ++i) {
        double w;
        asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(w) : "r"(smem_u32(xs + ((i + lane) & 1023))));
        sum += w;
    }
    t1 = clock64();
    if (lane == 0) out[9] = (t1 - t0) / N;
    if (acc == 12345 || idx == 77 || v == 3.3 || sum == 1.5 || j == 99999) out[10] = 1;
}

int main() {
    double *g, *gout;
    long long *out;
    cudaMalloc(&g, 8 << 20);
    cudaMalloc(&gout, 8 << 20);
    cudaMalloc(&out, 256);
    cudaMemset(g, 0, 8 << 20);
    cudaMemset(out, 0, 256);
    k_prims<<<1, 32>>>(g, gout, out);
    k_prims<<<1, 32>>>(g, gout, out);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[16];
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    printf("{\"err\": \"%s\", \"cycles\": {\"mbar_try_wait_done\": %lld, \"mbar_test_wait\": %lld, "
           "\"lds_dependent\": %lld, \"sts_syncwarp_lds\": %lld, \"dfma3_dmul\": %lld, \"bulk_copy_1536B_rt\": %lld, "
           "\"st_relaxed_issue\": %lld, \"ld_relaxed_l2_dependent\": %lld, \"cp_async8_rt\": %lld, "
           "\"lds_volatile_indep\": %lld}}\n",
           cudaGetErrorString(e), h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8], h[9]);
    return 0;
}
