// common.cuh -- internal types and PTX helpers shared by the CUDA sources of
// libsptrsv.so (sm_100a only).  Nothing here is visible through the C ABI.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "sptrsv.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libsptrsv is built for sm_100a only"
#endif

namespace sptrsv {

constexpr int kWarp = 32;
// Rows with more than kTprMax referenced off-diagonal entries are solved
// warp-per-row (WPR); the others thread-per-row (TPR) in 32-row chunks.
constexpr int kTprMax = 16;

// Chunk descriptor of the level-ordered layout (16 bytes, one vector load).
//   pos    first solve position of the chunk (perm[pos..pos+nrows) are its rows)
//   meta   bits 0..5: nrows (1..32); bit 6: WPR flag; bits 8..31: width
//          (TPR: max entries of its rows, <= kTprMax; WPR: the row's entry count)
//   eptr   offset of the chunk's entries in ecol/eval.
//          TPR: entry k of lane r at eptr + k*32 + r (padding: col = -1, val = 0)
//          WPR: entries contiguous at eptr .. eptr+width
struct __align__(16) ChunkDesc {
    int32_t pos;
    uint32_t meta;
    int64_t eptr;
};

__host__ __device__ inline int chunk_nrows(uint32_t m) { return (int)(m & 63u); }
__host__ __device__ inline bool chunk_wpr(uint32_t m) { return (m & 64u) != 0; }
__host__ __device__ inline int chunk_width(uint32_t m) { return (int)(m >> 8); }
__host__ __device__ inline uint32_t chunk_meta(int nrows, bool wpr, int width) {
    return (uint32_t)nrows | (wpr ? 64u : 0u) | ((uint32_t)width << 8);
}

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ int ld_relaxed(const int *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(int *p, int v) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release(int *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// L2-coherent loads of values produced during the kernel by other SMs
// (bypass L1: .cg), and streaming loads of read-once data.
template <typename T> __device__ __forceinline__ T ld_cg(const T *p) { return __ldcg(p); }
template <typename T> __device__ __forceinline__ T ld_stream(const T *p) { return __ldcs(p); }

// Relaxed (morally strong) value loads/stores for value-as-flag polling.
// (volatile: never cached or merged by the compiler; no "memory" clobber, so
// independent loads around them can still be scheduled freely)
__device__ __forceinline__ double ld_relaxed_val(const double *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p));
    return __longlong_as_double((long long)v);
}
__device__ __forceinline__ float ld_relaxed_val(const float *p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return __uint_as_float(v);
}
__device__ __forceinline__ void st_relaxed_val(double *p, double x) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"((unsigned long long)__double_as_longlong(x)) : "memory");
}
__device__ __forceinline__ void st_relaxed_val(float *p, float x) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(__float_as_uint(x)) : "memory");
}

// Value-as-flag sentinel: a NaN payload that arithmetic never produces on
// NVIDIA GPUs (they return the canonical NaN); a computed value equal to it
// is replaced by the canonical NaN before it is published.
template <typename T> struct Sentinel;
template <> struct Sentinel<double> {
    static constexpr unsigned long long bits = 0xFFF7A5A5DEADBEEFull;   // signalling-NaN payload
    __device__ static bool is(double v) { return (unsigned long long)__double_as_longlong(v) == bits; }
    __device__ static double value() { return __longlong_as_double((long long)bits); }
    __device__ static double scrub(double v) { return is(v) ? __longlong_as_double(0x7FFFFFFFFFFFFFFFll) : v; }
};
template <> struct Sentinel<float> {
    static constexpr unsigned bits = 0xFFB5A5EFu;
    __device__ static bool is(float v) { return __float_as_uint(v) == bits; }
    __device__ static float value() { return __uint_as_float(bits); }
    __device__ static float scrub(float v) { return is(v) ? __uint_as_float(0x7FFFFFFFu) : v; }
};

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// fma helpers: s - a*x as one rounding
__device__ __forceinline__ double fnma(double a, double x, double s) { return __fma_rn(-a, x, s); }
__device__ __forceinline__ float fnma(float a, float x, float s) { return __fmaf_rn(-a, x, s); }

}  // namespace sptrsv

namespace sptrsv {
// ------------------------------------------------ mbarrier + TMA bulk copy
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ bool mbar_test_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void *p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
}  // namespace sptrsv

namespace sptrsv {
// ------------------------------------------------ cp.async (LDGSTS) helpers
__device__ __forceinline__ void cp_async_8(void *smem_dst, const void *gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_16(void *smem_dst, const void *gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_4(void *smem_dst, const void *gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
}  // namespace sptrsv
