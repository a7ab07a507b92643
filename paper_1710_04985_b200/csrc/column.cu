// column.cu -- column-wise solves over the CSC of the referenced strict
// triangle:
//
//   k_slfc  SLFC (Alg. SLFC, kernel P:631-653): self-scheduled.  The
//           unknown of column i waits until its dependency counter count(i)
//           (initialised to dp(i)) reaches 0, then x(i) := x(i)/d(i)
//           and every dependent row r of column i receives x(r) -= L(r,i) x(i)
//           and count(r) -= 1 -- the paper's critical section as
//           two L2 reductions: the x update (relaxed red.add), one release
//           fence per column, the counter decrements (relaxed red.add).  The
//           consumer's acquire poll of count(i) orders its read of x(i).
//           x starts as b ("x := f").  Columns are claimed by
//           ticket in jlev order, 32 per warp, lane = column; lanes wait and
//           push independently (no warp lockstep, P:680-684 / SURVEY Q12).
//   k_levc  LEVC (Alg. LEVC, kernel P:536-552): level-scheduled.  One
//           co-resident grid; per level thread = column: x(i) := x(i)/d(i), then
//           the red.add updates of its dependents; a grid-wide barrier between
//           levels (instead of one launch per level).
//
// Both accumulate with atomics in arrival order, so results vary in the last
// bits from run to run (the paper's own caveat for the critical-region form);
// parity is by the north-star tolerance.  Same division reading as the row
// kernels (Q7): multiply by 1/d.
#include <algorithm>
#include <cstdlib>

#include "internal.h"

namespace sptrsv {
namespace {

constexpr int kColThreads = 256;
constexpr int kLevcThreads = 1024;
constexpr int kLevcThreadsDefault = 128;   // cfg2 2.98 -> 1.70 ms, cfg3 17.8 -> 6.6 ms vs 1024 (grid barrier cost)

// ------------------------------------------------------------ CSC build
// entries of the per-position CSR (mr_*: row perm[p], dependency mr_col[k])
__global__ void k_csc_count(int n, const int32_t *__restrict__ mr_ptr, const int32_t *__restrict__ mr_col,
                            int32_t *cnt) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    for (int k = mr_ptr[p]; k < mr_ptr[p + 1]; ++k) atomicAdd(&cnt[mr_col[k]], 1);
}
template <typename T>
__global__ void k_csc_fill(int n, const int32_t *__restrict__ perm, const int32_t *__restrict__ mr_ptr,
                           const int32_t *__restrict__ mr_col, const T *__restrict__ mr_val,
                           const int32_t *__restrict__ cptr, int32_t *cur, int32_t *crow, T *cval) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int r = perm[p];
    for (int k = mr_ptr[p]; k < mr_ptr[p + 1]; ++k) {
        const int j = mr_col[k];
        const int q = cptr[j] + atomicAdd(&cur[j], 1);
        crow[q] = r;
        cval[q] = mr_val[k];
    }
}

__device__ __forceinline__ void red_add(double *p, double v) {
    asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void red_add(float *p, float v) {
    asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void red_dec(int32_t *p) {
    asm volatile("red.relaxed.gpu.global.add.s32 [%0], -1;" ::"l"(p) : "memory");
}
__device__ __forceinline__ int ld_acquire_i32(const int32_t *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ double ld_l2(const double *p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ float ld_l2(const float *p) {
    float v;
    asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    return v;
}

// one column: x(i) / d(i), then the updates of its dependents
template <typename T, bool UNIT>
__device__ __forceinline__ T column_update(int i, const T *__restrict__ invd_row, const int32_t *__restrict__ cptr,
                                           const int32_t *__restrict__ crow, const T *__restrict__ cval, T *x) {
    T xi = ld_l2(x + i);
    if (!UNIT) xi *= invd_row[i];
    x[i] = xi;
    const int k1 = cptr[i + 1];
    for (int k = cptr[i]; k < k1; ++k) red_add(x + crow[k], -cval[k] * xi);
    return xi;
}

// ------------------------------------------------------------ SLFC
template <typename T, bool UNIT>
__global__ void __launch_bounds__(kColThreads) k_slfc(int n, const int32_t *__restrict__ perm,
                                                      const T *__restrict__ invd_row,
                                                      const int32_t *__restrict__ cptr,
                                                      const int32_t *__restrict__ crow,
                                                      const T *__restrict__ cval, T *x, int32_t *count,
                                                      unsigned *ctr, unsigned nwarps_total) {
    const int lane = threadIdx.x & 31;
    const int nblk = (n + 31) / 32;
    for (;;) {
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(&ctr[0], 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if ((int)t >= nblk) break;
        const int p = (int)t * 32 + lane;
        if (p < n) {
            const int i = perm[p];
            // relaxed polls (an acquire load per poll also invalidates L1 and
            // floods L2), then one acquire load once the counter reads 0
            if (ld_relaxed(count + i) != 0) {
                do {
                    __nanosleep(32);
                } while (ld_relaxed(count + i) != 0);
            }
            (void)ld_acquire_i32(count + i);
            const int k0 = cptr[i], k1 = cptr[i + 1];
            column_update<T, UNIT>(i, invd_row, cptr, crow, cval, x);
            if (k1 > k0) {
                // the x updates above happen before any counter decrement below
                // (one fence per column; a red.release per decrement measured
                // 2.8x slower on cfg4, round 1)
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                for (int k = k0; k < k1; ++k) red_dec(count + crow[k]);
            }
        }
    }
    if (lane == 0) {            // the last warp out resets the ticket
        const unsigned e = atomicAdd(&ctr[1], 1u);
        if (e == nwarps_total - 1) {
            ctr[0] = 0;
            ctr[1] = 0;
        }
    }
}

// ------------------------------------------------------------ LEVC
__device__ __forceinline__ unsigned long long ld_acquire_u64c(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void grid_barrier_c(unsigned long long *bar, unsigned long long target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
        while (ld_acquire_u64c(bar) < target) {
        }
    }
    __syncthreads();
}

template <typename T, bool UNIT>
__global__ void __launch_bounds__(kLevcThreads, 1) k_levc(int nlev, const int32_t *__restrict__ ilev,
                                                         const int32_t *__restrict__ perm,
                                                         const T *__restrict__ invd_row,
                                                         const int32_t *__restrict__ cptr,
                                                         const int32_t *__restrict__ crow,
                                                         const T *__restrict__ cval, T *x,
                                                         unsigned long long *bar, unsigned long long bar_base) {
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int nt = gridDim.x * blockDim.x;
    for (int l = 0; l < nlev; ++l) {
        const int p1 = ilev[l + 1];
        for (int p = ilev[l] + tid; p < p1; p += nt) column_update<T, UNIT>(perm[p], invd_row, cptr, crow, cval, x);
        if (l + 1 < nlev) grid_barrier_c(bar, bar_base + (unsigned long long)(l + 1) * gridDim.x);
    }
}

template <typename T>
sptrsv_status_t build_csc(sptrsv_handle_t h, cudaStream_t s) {
    ArenaStream as_{h->arena, s};     // the handle's allocations in this call: stream-ordered on s
    const int n = h->n;
    DevArena tmp(s);
    struct Guard {
        DevArena &a;
        ~Guard() { a.release_all(); }
    } guard{tmp};
    sptrsv_status_t st;
    int32_t nnz = 0;                         // referenced strict entries = mr_ptr[n]
    SPTRSV_CUDA(cudaMemcpyAsync(&nnz, h->d_mr_ptr + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    int32_t *cnt = nullptr, *cur = nullptr;
    if ((st = tmp.alloc_n(&cnt, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&cur, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&h->d_c_ptr, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&h->d_c_row, (size_t)std::max<int32_t>(nnz, 1))) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc(&h->d_c_val, (size_t)std::max<int32_t>(nnz, 1) * sizeof(T))) != SPTRSV_SUCCESS)
        return st;
    if ((st = h->arena.alloc_n(&h->d_count, (size_t)n)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * ((size_t)n + 1), s));
    SPTRSV_CUDA(cudaMemsetAsync(cur, 0, sizeof(int32_t) * ((size_t)n + 1), s));
    const int g = (n + 255) / 256;
    k_csc_count<<<g, 256, 0, s>>>(n, h->d_mr_ptr, h->d_mr_col, cnt);
    if ((st = exclusive_scan_i32(cnt, h->d_c_ptr, (int64_t)n + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    k_csc_fill<T><<<g, 256, 0, s>>>(n, h->d_perm, h->d_mr_ptr, h->d_mr_col, (const T *)h->d_mr_val, h->d_c_ptr, cur,
                                    h->d_c_row, (T *)h->d_c_val);
    SPTRSV_CUDA(cudaGetLastError());
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    h->csc_built = true;
    h->info.device_bytes = h->arena.bytes + (int64_t)h->stage_bytes;
    return SPTRSV_SUCCESS;
}

template <typename T, bool UNIT>
sptrsv_status_t launch_column(sptrsv_handle_t h, const T *b, T *x, cudaStream_t s) {
    if (!h->mr_built) {
        sptrsv_status_t st = build_mr_any(h, s);
        if (st != SPTRSV_SUCCESS) return st;
    }
    if (!h->csc_built) {
        sptrsv_status_t st = build_csc<T>(h, s);
        if (st != SPTRSV_SUCCESS) return st;
    }
    const int n = h->n;
    if (b != x) SPTRSV_CUDA(cudaMemcpyAsync(x, b, sizeof(T) * (size_t)n, cudaMemcpyDeviceToDevice, s));   // x := f
    if (h->algo == SPTRSV_ALGO_SLFC) {
        SPTRSV_CUDA(cudaMemcpyAsync(h->d_count, h->d_dp, sizeof(int32_t) * (size_t)n, cudaMemcpyDeviceToDevice, s));
        if (h->slfc_grid == 0) {
            int per_sm = 0;
            SPTRSV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_slfc<T, UNIT>, kColThreads, 0));
            // at most 2 CTAs (16 warps) per SM: enough columns in flight, and
            // not so many spinning lanes that their polls slow the L2
            h->slfc_grid = std::max(1, std::min(per_sm, 1)) * h->num_sms;   // 1/SM: 2-6% faster than 2
        }
        const int grid = h->slfc_grid;
        k_slfc<T, UNIT><<<grid, kColThreads, 0, s>>>(n, h->d_perm, (const T *)h->d_invd_row, h->d_c_ptr, h->d_c_row,
                                                    (const T *)h->d_c_val, x, h->d_count, h->d_ctr,
                                                    (unsigned)(grid * (kColThreads / 32)));
        SPTRSV_CUDA(cudaGetLastError());
        return SPTRSV_SUCCESS;
    }
    const int grid = h->num_sms;
    const int nlev = h->info.nlev;
    void *args[] = {(void *)&nlev, (void *)&h->d_ilev, (void *)&h->d_perm, (void *)&h->d_invd_row,
                    (void *)&h->d_c_ptr, (void *)&h->d_c_row, (void *)&h->d_c_val, (void *)&x,
                    (void *)&h->d_bar, (void *)&h->bar_base};
    const int lt = kLevcThreadsDefault;
    SPTRSV_CUDA(cudaLaunchCooperativeKernel((const void *)k_levc<T, UNIT>, grid, lt, args, 0, s));
    h->bar_base += (unsigned long long)(nlev > 0 ? nlev - 1 : 0) * grid;
    return SPTRSV_SUCCESS;
}

}  // namespace

// new values (the per-position CSR already refreshed): refill the CSC (the
// order of a column's rows follows the atomic counters, rows and values are
// written together)
sptrsv_status_t csc_refresh_values(sptrsv_handle_t h, cudaStream_t s) {
    const int n = h->n;
    DevArena tmp(s);
    struct Guard {
        DevArena &a;
        ~Guard() { a.release_all(); }
    } guard{tmp};
    sptrsv_status_t st;
    int32_t *cur = nullptr;
    if ((st = tmp.alloc_n(&cur, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemsetAsync(cur, 0, sizeof(int32_t) * ((size_t)n + 1), s));
    const int g = (n + 255) / 256;
    if (h->dtype == SPTRSV_F64)
        k_csc_fill<double><<<g, 256, 0, s>>>(n, h->d_perm, h->d_mr_ptr, h->d_mr_col, (const double *)h->d_mr_val,
                                             h->d_c_ptr, cur, h->d_c_row, (double *)h->d_c_val);
    else
        k_csc_fill<float><<<g, 256, 0, s>>>(n, h->d_perm, h->d_mr_ptr, h->d_mr_col, (const float *)h->d_mr_val,
                                            h->d_c_ptr, cur, h->d_c_row, (float *)h->d_c_val);
    SPTRSV_CUDA(cudaGetLastError());
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    return SPTRSV_SUCCESS;
}

sptrsv_status_t column_solve(sptrsv_handle_t h, const void *b, void *x, cudaStream_t s) {
    if (h->n == 0) return SPTRSV_SUCCESS;
    if (h->dtype == SPTRSV_F64)
        return h->diag == SPTRSV_UNIT ? launch_column<double, true>(h, (const double *)b, (double *)x, s)
                                      : launch_column<double, false>(h, (const double *)b, (double *)x, s);
    return h->diag == SPTRSV_UNIT ? launch_column<float, true>(h, (const float *)b, (float *)x, s)
                                  : launch_column<float, false>(h, (const float *)b, (float *)x, s);
}

}  // namespace sptrsv
