// analyze.cu -- the setup phase on the GPU (§4.4, Table 1):
//   a1  CSR validation + triangle/diagonal selection
//   a2  dependency counts dp                               (DEP)
//   a3  level computation, sync-free (value-as-flag)       (LEV)
//   a4  level bucketing: stable radix sort -> ilev, jlev
//   a5  level-ordered copy of the triangle + row binning
// Everything runs in hand-written kernels; the host only sizes allocations.
#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <cstdio>
#include <cstring>

#include "internal.h"

namespace sptrsv {

// ------------------------------------------------------------------ scans
namespace {
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

// Per tile: exclusive scan of `in` into `out`, tile total into sums[tile].
template <typename T>
__global__ void __launch_bounds__(kScanThreads) k_scan_tile(const T *in, T *out, T *sums, int64_t n) {
    __shared__ T wsum[kScanThreads / 32];
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    T v[kScanItems];
    T tsum = 0;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        v[i] = (base + i < n) ? in[base + i] : T(0);
        tsum += v[i];
    }
    T incl = warp_incl_scan(tsum);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        T w = (lane < kScanThreads / 32) ? wsum[lane] : T(0);
        T wi = warp_incl_scan(w);
        if (lane < kScanThreads / 32) wsum[lane] = wi - w;
        if (lane == kScanThreads / 32 - 1 && sums) sums[blockIdx.x] = wi;
    }
    __syncthreads();
    T run = wsum[warp] + incl - tsum;
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        if (base + i < n) out[base + i] = run;
        run += v[i];
    }
}

template <typename T>
__global__ void k_scan_add(T *out, const T *offs, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * kScanTile + threadIdx.x;
    const T o = offs[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        int64_t j = i + (int64_t)k * kScanThreads;
        if (j < n) out[j] += o;
    }
}

template <typename T>
sptrsv_status_t exclusive_scan(const T *in, T *out, int64_t n, DevArena &tmp, cudaStream_t s) {
    if (n <= 0) return SPTRSV_SUCCESS;
    int64_t ntiles = (n + kScanTile - 1) / kScanTile;
    if (ntiles == 1) {
        k_scan_tile<T><<<1, kScanThreads, 0, s>>>(in, out, (T *)nullptr, n);
        SPTRSV_CUDA(cudaGetLastError());
        return SPTRSV_SUCCESS;
    }
    T *sums = nullptr, *offs = nullptr;
    sptrsv_status_t st;
    if ((st = tmp.alloc_n(&sums, ntiles)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&offs, ntiles)) != SPTRSV_SUCCESS) return st;
    k_scan_tile<T><<<(unsigned)ntiles, kScanThreads, 0, s>>>(in, out, sums, n);
    SPTRSV_CUDA(cudaGetLastError());
    if ((st = exclusive_scan<T>(sums, offs, ntiles, tmp, s)) != SPTRSV_SUCCESS) return st;
    k_scan_add<T><<<(unsigned)ntiles, kScanThreads, 0, s>>>(out, offs, n);
    SPTRSV_CUDA(cudaGetLastError());
    return SPTRSV_SUCCESS;
}

// ------------------------------------------------------------ radix sort
// Stable LSD radix sort of (uint32 key, int32 value) pairs, 8 bits per pass.
constexpr int kRsThreads = 256;
constexpr int kRsRounds = 8;
constexpr int kRsTile = kRsThreads * kRsRounds;

__global__ void __launch_bounds__(kRsThreads) k_rs_hist(const uint32_t *keys, int64_t n, int shift,
                                                        int32_t *hist, int ntiles) {
    __shared__ int32_t cnt[256];
    cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kRsTile;
    for (int r = 0; r < kRsRounds; ++r) {
        int64_t i = base + (int64_t)r * kRsThreads + threadIdx.x;
        if (i < n) atomicAdd(&cnt[(keys[i] >> shift) & 255u], 1);
    }
    __syncthreads();
    hist[(int64_t)threadIdx.x * ntiles + blockIdx.x] = cnt[threadIdx.x];
}

__global__ void __launch_bounds__(kRsThreads) k_rs_scatter(const uint32_t *kin, const int32_t *vin,
                                                           uint32_t *kout, int32_t *vout, int64_t n,
                                                           int shift, const int32_t *offs, int ntiles) {
    __shared__ int32_t sbase[256];
    __shared__ int32_t wcnt[kRsThreads / 32][257];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    sbase[threadIdx.x] = offs[(int64_t)threadIdx.x * ntiles + blockIdx.x];
    for (int w = 0; w < kRsThreads / 32; ++w) wcnt[w][threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kRsTile;
    for (int r = 0; r < kRsRounds; ++r) {
        int64_t i = base + (int64_t)r * kRsThreads + threadIdx.x;
        bool valid = i < n;
        uint32_t key = valid ? kin[i] : 0u;
        int d = valid ? (int)((key >> shift) & 255u) : 256;
        unsigned peers = __match_any_sync(0xffffffffu, d);
        int rank = __popc(peers & lanemask_lt());
        bool leader = (peers & lanemask_lt()) == 0;
        if (leader && valid) wcnt[warp][d] = __popc(peers);
        __syncthreads();
        if (valid) {
            int pos = sbase[d] + rank;
            for (int w = 0; w < warp; ++w) pos += wcnt[w][d];
            kout[pos] = key;
            vout[pos] = vin ? vin[i] : (int32_t)i;
        }
        __syncthreads();
        {
            int dd = threadIdx.x;
            int sum = 0;
            for (int w = 0; w < kRsThreads / 32; ++w) {
                sum += wcnt[w][dd];
                wcnt[w][dd] = 0;
            }
            sbase[dd] += sum;
        }
        __syncthreads();
    }
}
}  // namespace

sptrsv_status_t exclusive_scan_i32(const int32_t *in, int32_t *out, int64_t n, DevArena &tmp, cudaStream_t s) {
    return exclusive_scan<int32_t>(in, out, n, tmp, s);
}
sptrsv_status_t exclusive_scan_i64(const int64_t *in, int64_t *out, int64_t n, DevArena &tmp, cudaStream_t s) {
    return exclusive_scan<int64_t>(in, out, n, tmp, s);
}

// vals_in == nullptr means the identity 0..n-1.  Output buffers must not alias inputs.
sptrsv_status_t radix_sort_pairs(const uint32_t *keys_in, const int32_t *vals_in, uint32_t *keys_out,
                                 int32_t *vals_out, int64_t n, uint32_t max_key, DevArena &tmp,
                                 cudaStream_t s) {
    if (n <= 0) return SPTRSV_SUCCESS;
    int bits = 0;
    while (bits < 32 && (max_key >> bits) != 0) ++bits;
    int passes = std::max(1, (bits + 7) / 8);
    int ntiles = (int)((n + kRsTile - 1) / kRsTile);
    int32_t *hist = nullptr, *offs = nullptr;
    uint32_t *kbuf = nullptr;
    int32_t *vbuf = nullptr;
    sptrsv_status_t st;
    if ((st = tmp.alloc_n(&hist, (size_t)256 * ntiles)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&offs, (size_t)256 * ntiles)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&kbuf, (size_t)n)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&vbuf, (size_t)n)) != SPTRSV_SUCCESS) return st;
    // ping-pong so that the last pass lands in (keys_out, vals_out)
    const uint32_t *kin = keys_in;
    const int32_t *vin = vals_in;
    for (int p = 0; p < passes; ++p) {
        bool last_to_out = ((passes - 1 - p) % 2) == 0;
        uint32_t *ko = last_to_out ? keys_out : kbuf;
        int32_t *vo = last_to_out ? vals_out : vbuf;
        k_rs_hist<<<ntiles, kRsThreads, 0, s>>>(kin, n, 8 * p, hist, ntiles);
        SPTRSV_CUDA(cudaGetLastError());
        if ((st = exclusive_scan<int32_t>(hist, offs, (int64_t)256 * ntiles, tmp, s)) != SPTRSV_SUCCESS) return st;
        k_rs_scatter<<<ntiles, kRsThreads, 0, s>>>(kin, vin, ko, vo, n, 8 * p, offs, ntiles);
        SPTRSV_CUDA(cudaGetLastError());
        kin = ko;
        vin = vo;
    }
    return SPTRSV_SUCCESS;
}

// -------------------------------------------------------- a1/a2: validate
namespace {
struct AnalysisStatus {
    int32_t bad_row;          // atomicMin, INT32_MAX = none
    int32_t zero_pivot_row;   // atomicMin, INT32_MAX = none
    int32_t max_deps;         // atomicMax
    int32_t max_lev;          // atomicMax (levels kernel)
    unsigned long long ignored;
    unsigned long long used;
    int32_t max_width;        // atomicMax over levels of ilev[l+1] - ilev[l]
    int32_t nnz_input;        // rowptr[n]
};

// summary of the schedule: the widest level (read with the final status)
__global__ void k_summary(int nlev, const int32_t *ilev, AnalysisStatus *st) {
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l < nlev) atomicMax(&st->max_width, ilev[l + 1] - ilev[l]);
}
__global__ void k_nnz_input(const int32_t *rowptr, int n, AnalysisStatus *st) { st->nnz_input = rowptr[n]; }

__device__ __forceinline__ bool in_tri(int i, int j, int uplo) { return uplo == SPTRSV_LOWER ? (j < i) : (j > i); }

// Warp per row (grid-stride).  Rules: include/sptrsv.h, sptrsv_analyze.
template <typename T>
__global__ void __launch_bounds__(256) k_validate(int n, const int32_t *__restrict__ rowptr,
                                                  const int32_t *__restrict__ colidx,
                                                  const T *__restrict__ vals, int uplo, int diag,
                                                  int32_t *__restrict__ dp, T *__restrict__ invd,
                                                  AnalysisStatus *stat) {
    const int lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    const int nnz = rowptr[n];
    unsigned long long my_ign = 0, my_used = 0;
    int my_maxdeps = 0;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nwarps) {
        const int p = rowptr[i], q = rowptr[i + 1];
        bool bad = (p < 0) || (q < p) || (q > nnz) || (i == 0 && p != 0);
        int cnt = 0, ign = 0, dk = -1;
        if (!bad) {
            for (int k = p + lane; k < q; k += 32) {
                int c = colidx[k];
                if (c < 0 || c >= n) bad = true;
                if (k > p && c <= colidx[k - 1]) bad = true;
                if (c == i) dk = k;
                else if (in_tri(i, c, uplo)) ++cnt;
                else ++ign;
            }
        }
        bad = __any_sync(0xffffffffu, bad);
        if (bad) {
            if (lane == 0) atomicMin(&stat->bad_row, i);
            continue;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
            ign += __shfl_xor_sync(0xffffffffu, ign, o);
            dk = max(dk, __shfl_xor_sync(0xffffffffu, dk, o));
        }
        if (lane == 0) {
            dp[i] = cnt;
            if (diag == SPTRSV_UNIT) {
                ign += (dk >= 0);
                invd[i] = T(1);
            } else {
                T d = (dk >= 0) ? vals[dk] : T(0);
                if (d == T(0)) {
                    atomicMin(&stat->zero_pivot_row, i);
                    invd[i] = T(0);
                } else {
                    invd[i] = T(1) / d;
                }
            }
            my_ign += (unsigned long long)ign;
            my_used += (unsigned long long)cnt;
            my_maxdeps = max(my_maxdeps, cnt);
        }
    }
    if (lane == 0) {
        if (my_ign) atomicAdd(&stat->ignored, my_ign);
        if (my_used) atomicAdd(&stat->used, my_used);
        if (my_maxdeps) atomicMax(&stat->max_deps, my_maxdeps);
    }
}

// ------------------------------------------------------- a3: levels
// Sync-free level computation: lev[] starts at -1 and each value is its own
// ready flag.  Warps claim 32-row tickets in topological (natural) order --
// ascending for LOWER, descending for UPPER -- so every row a
// thread waits on was claimed earlier by a running warp: no deadlock for any
// grid size.  lev(i) = 0 without dependencies, else 1 + max lev(j).
__global__ void __launch_bounds__(256) k_levels(int n, const int32_t *__restrict__ rowptr,
                                                const int32_t *__restrict__ colidx, int uplo,
                                                int32_t *lev, unsigned *ticket, AnalysisStatus *stat) {
    const int lane = threadIdx.x & 31;
    const int nchunk = (n + 31) / 32;
    int my_max = -1;
    for (;;) {
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(ticket, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if ((int)t >= nchunk) break;
        const int r = (int)t * 32 + lane;
        if (r < n) {
            const int i = (uplo == SPTRSV_LOWER) ? r : n - 1 - r;
            const int p = rowptr[i], q = rowptr[i + 1];
            int l = 0;
            for (int k = p; k < q; k += 4) {
                int js[4], vs[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    int j = (k + u < q) ? colidx[k + u] : i;
                    js[u] = in_tri(i, j, uplo) ? j : -1;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) vs[u] = (js[u] >= 0) ? ld_relaxed(&lev[js[u]]) : 0;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    while (vs[u] < 0) {
                        __nanosleep(64);
                        vs[u] = ld_relaxed(&lev[js[u]]);
                    }
                    if (js[u] >= 0) l = max(l, vs[u] + 1);
                }
            }
            st_relaxed(&lev[i], l);
            my_max = max(my_max, l);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_max = max(my_max, __shfl_xor_sync(0xffffffffu, my_max, o));
    if (lane == 0 && my_max >= 0) atomicMax(&stat->max_lev, my_max);
}

// ------------------------------------------------------- a3 (default): Kahn by rounds
// The paper's analysis (Kahn's topological sort by rounds): the
// frontier of round l is exactly level l (0-based, reading Q4).  One
// cooperative kernel walks the rounds with a grid barrier between them
// instead of one launch per round; a frontier row's dependents
// (CSC of the referenced strict triangle) get their remaining-dependency
// counter decremented, and the one that reaches 0 is appended to the next
// frontier.  No spin-waiting on other rows: the sync-free k_levels above
// spends ~1 s on cfg4's 12,288 levels (its spinning warps load L2 and its
// chains serialise inside a warp).  Only lev[] is taken from here; ilev /
// jlev come from the stable radix sort, so the atomic append order (P:780,
// P:804) never shows.
__global__ void k_dep_count(int n, const int32_t *__restrict__ rowptr, const int32_t *__restrict__ colidx, int uplo,
                            int32_t *cnt) {
    const int lane = threadIdx.x & 31;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += (gridDim.x * blockDim.x) >> 5)
        for (int k = rowptr[i] + lane; k < rowptr[i + 1]; k += 32) {
            const int j = colidx[k];
            if (in_tri(i, j, uplo)) atomicAdd(&cnt[j], 1);
        }
}
__global__ void k_dep_fill(int n, const int32_t *__restrict__ rowptr, const int32_t *__restrict__ colidx, int uplo,
                           const int32_t *__restrict__ cptr, int32_t *cur, int32_t *crow) {
    const int lane = threadIdx.x & 31;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += (gridDim.x * blockDim.x) >> 5)
        for (int k = rowptr[i] + lane; k < rowptr[i + 1]; k += 32) {
            const int j = colidx[k];
            if (in_tri(i, j, uplo)) crow[cptr[j] + atomicAdd(&cur[j], 1)] = i;
        }
}
// One round of the paper's host-driven Kahn (FIND_LEVEL): the
// rows of frontier level l get lev = l and release their dependents into the
// next frontier; the host launches one round per level and reads the next
// frontier's size back (analysis-mode study, NEXT-2; the default analysis runs
// all rounds in one cooperative launch, k_kahn below).
__global__ void k_kahn_round(int nf, int l, const int32_t *__restrict__ cptr, const int32_t *__restrict__ crow,
                             int32_t *indeg, const int32_t *__restrict__ Fc, int32_t *Fn, int32_t *cnt_next,
                             int32_t *lev) {
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nwp = (gridDim.x * blockDim.x) >> 5;
    for (int idx = gw; idx < nf; idx += nwp) {
        const int i = Fc[idx];
        if (lane == 0) lev[i] = l;
        const int k1 = cptr[i + 1];
        for (int k = cptr[i] + lane; k < k1; k += 32) {
            const int r = crow[k];
            if (atomicSub(&indeg[r], 1) == 1) Fn[atomicAdd(cnt_next, 1)] = r;
        }
    }
}
__global__ void k_frontier0(int n, const int32_t *__restrict__ dp, int32_t *F, int32_t *cnt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && dp[i] == 0) F[atomicAdd(cnt, 1)] = i;
}
__device__ __forceinline__ unsigned long long ld_acquire_u64a(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void grid_barrier_a(unsigned long long *bar, unsigned long long target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
        while (ld_acquire_u64a(bar) < target) {
        }
    }
    __syncthreads();
}
constexpr int kKahnThreads = 128;
__global__ void __launch_bounds__(kKahnThreads) k_kahn(int n, const int32_t *__restrict__ cptr,
                                                       const int32_t *__restrict__ crow, int32_t *indeg,
                                                       int32_t *F0, int32_t *F1, int32_t *cnt, int32_t *lev,
                                                       unsigned long long *bar, AnalysisStatus *stat) {
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31, gw = tid >> 5, nwp = (gridDim.x * blockDim.x) >> 5;
    // three frontier counters: round l reads cnt[l%3], appends to cnt[(l+1)%3]
    // and clears cnt[(l+2)%3] (read in round l-1, appended to in round l+1):
    // one grid barrier per round
    int l = 0;
    for (;; ++l) {
        int32_t *Fc = (l & 1) ? F1 : F0;
        int32_t *Fn = (l & 1) ? F0 : F1;
        const int nf = __ldcg(&cnt[l % 3]);
        if (nf == 0) break;
        if (tid == 0) cnt[(l + 2) % 3] = 0;
        // warp per frontier row, lanes over its dependents (a dependent list
        // walked by one thread serialises its returning atomics: cfg4
        // analysis 297 -> 145 ms; a thread-per-row path for wide rounds was
        // slower and noisier on cfg4)
        for (int idx = gw; idx < nf; idx += nwp) {
            const int i = __ldcg(&Fc[idx]);
            if (lane == 0) lev[i] = l;
            const int k1 = cptr[i + 1];
            for (int k = cptr[i] + lane; k < k1; k += 32) {
                const int r = crow[k];
                if (atomicSub(&indeg[r], 1) == 1) Fn[atomicAdd(&cnt[(l + 1) % 3], 1)] = r;
            }
        }
        grid_barrier_a(bar, (unsigned long long)(l + 1) * gridDim.x);
    }
    if (tid == 0) stat->max_lev = l - 1;
}

// ------------------------------------------------------- a4: bucketing
// ilev from the level-sorted keys: level boundaries (no level is empty).
__global__ void k_ilev_from_sorted(const uint32_t *skeys, int n, int nlev, int32_t *ilev) {
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) {
        uint32_t k = skeys[p];
        if (p == 0 || skeys[p - 1] != k) ilev[k] = p;
    }
    if (p == 0) ilev[nlev] = n;
}

__global__ void k_level_keys(const int32_t *lev, int n, uint32_t *keys) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) keys[i] = (uint32_t)lev[i];
}

// ------------------------------------------------------- a5: layout
// Solve-order key: level, then WPR rows (bucket 0), then TPR rows by
// decreasing dependency count (buckets 1..kTprMax+1) -- homogeneous chunks.
constexpr int kBuckets = kTprMax + 2;
__device__ __forceinline__ uint32_t row_bucket(int deps) { return deps > kTprMax ? 0u : (uint32_t)(kTprMax + 1 - deps); }

__global__ void k_solve_keys(const int32_t *lev, const int32_t *dp, int n, uint32_t *keys) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) keys[i] = (uint32_t)lev[i] * kBuckets + row_bucket(dp[i]);
}

// per level: number of WPR rows (bucket 0) -- counted from sorted keys
__global__ void k_count_wpr(const uint32_t *skeys, int n, int32_t *wcnt) {
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n && (skeys[p] % kBuckets) == 0) atomicAdd(&wcnt[skeys[p] / kBuckets], 1);
}

__global__ void k_chunks_per_level(const int32_t *ilev, const int32_t *wcnt, int nlev, int32_t *nch) {
    int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l < nlev) {
        int width = ilev[l + 1] - ilev[l];
        int w = wcnt[l];
        nch[l] = w + (width - w + 31) / 32;
    }
    if (l == nlev) nch[l] = 0;
}

// one thread per level writes that level's chunk descriptors and entry counts
__global__ void k_chunk_desc(const int32_t *ilev, const int32_t *wcnt, const int32_t *lev_chunk, int nlev,
                             const int32_t *perm, const int32_t *dp, ChunkDesc *chunks, int64_t *ecount,
                             int32_t *chunk_lev) {
    int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= nlev) return;
    int c = lev_chunk[l];
    for (int cc = lev_chunk[l]; cc < lev_chunk[l + 1]; ++cc) chunk_lev[cc] = l;
    const int p0 = ilev[l], p1 = ilev[l + 1], w = wcnt[l];
    for (int p = p0; p < p0 + w; ++p, ++c) {
        int len = dp[perm[p]];
        chunks[c].pos = p;
        chunks[c].meta = chunk_meta(1, true, len);
        ecount[c] = len;
    }
    for (int p = p0 + w; p < p1; p += 32, ++c) {
        int nr = min(32, p1 - p);
        int width = dp[perm[p]];          // first row has the most dependencies
        chunks[c].pos = p;
        chunks[c].meta = chunk_meta(nr, false, width);
        ecount[c] = (int64_t)width * 32;
    }
}

__global__ void k_patch_eptr(ChunkDesc *chunks, const int64_t *eptr, int nchunks) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < nchunks) chunks[c].eptr = eptr[c];
}

template <typename T>
__global__ void __launch_bounds__(256) k_fill(int nchunks, const ChunkDesc *__restrict__ chunks,
                                              const int64_t *__restrict__ eptr, const int32_t *__restrict__ perm,
                                              const int32_t *__restrict__ rowptr, const int32_t *__restrict__ colidx,
                                              const T *__restrict__ vals, const T *__restrict__ invd_row,
                                              int uplo, int32_t *__restrict__ ecol, T *__restrict__ eval,
                                              T *__restrict__ invd_pos) {
    const int lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < nchunks; c += nwarps) {
        const ChunkDesc cd = chunks[c];
        const int nr = chunk_nrows(cd.meta), width = chunk_width(cd.meta);
        const int64_t e0 = eptr[c];
        if (!chunk_wpr(cd.meta)) {
            int k = 0;
            if (lane < nr) {
                const int i = perm[cd.pos + lane];
                invd_pos[cd.pos + lane] = invd_row[i];
                for (int kk = rowptr[i]; kk < rowptr[i + 1]; ++kk) {
                    int j = colidx[kk];
                    if (in_tri(i, j, uplo)) {
                        ecol[e0 + (int64_t)k * 32 + lane] = j;
                        eval[e0 + (int64_t)k * 32 + lane] = vals ? vals[kk] : T(0);
                        ++k;
                    }
                }
            }
            for (; k < width; ++k) {
                ecol[e0 + (int64_t)k * 32 + lane] = -1;
                eval[e0 + (int64_t)k * 32 + lane] = T(0);
            }
        } else {
            const int i = perm[cd.pos];
            if (lane == 0) invd_pos[cd.pos] = invd_row[i];
            int run = 0;
            for (int kk0 = rowptr[i]; kk0 < rowptr[i + 1]; kk0 += 32) {
                int kk = kk0 + lane;
                int j = (kk < rowptr[i + 1]) ? colidx[kk] : i;
                bool take = in_tri(i, j, uplo);
                unsigned bal = __ballot_sync(0xffffffffu, take);
                if (take) {
                    int o = run + __popc(bal & lanemask_lt());
                    ecol[e0 + o] = j;
                    eval[e0 + o] = vals ? vals[kk] : T(0);
                }
                run += __popc(bal);
            }
        }
    }
}
__global__ void k_chunk_eptr(int nchunks, const ChunkDesc *__restrict__ chunks, int64_t *__restrict__ eptr) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < nchunks) eptr[c] = chunks[c].eptr;
}
// count of positions where two int arrays differ
__global__ void k_count_diff(int64_t n, const int32_t *__restrict__ a, const int32_t *__restrict__ b, unsigned *cnt) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool d = i < n && a[i] != b[i];
    if (__any_sync(0xffffffffu, d) && d) atomicAdd(cnt, 1u);
}
}  // namespace

static int grid_for(int64_t items, int per_block, int cap) {
    int64_t g = (items + per_block - 1) / per_block;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, cap));
}

// Level computation of the analysis (debug / study setting, process-wide):
// 0 Kahn by rounds in one cooperative launch (default), 1 the sync-free
// value-as-flag kernel, 2 the paper's host loop with one launch per level.
int g_levels_mode = 0;

// ------------------------------------------------------------- driver
sptrsv_status_t analyze_impl(sptrsv_handle_t h, const int32_t *rowptr, const int32_t *colidx,
                             const void *vals, cudaStream_t s) {
    const int n = h->n;
    // SPTRSV_TIMING=1: host wall-clock per analysis phase (stream synchronised) to stderr
    const bool timing = getenv("SPTRSV_TIMING") && *getenv("SPTRSV_TIMING") == '1';
    auto tlast = std::chrono::steady_clock::now();
    auto phase = [&](const char *name) {
        if (!timing) return;
        cudaStreamSynchronize(s);
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[sptrsv analyze] %-10s %8.2f ms\n", name,
                std::chrono::duration<double, std::milli>(now - tlast).count());
        tlast = now;
    };
    DevArena tmp(s);
    struct Guard {
        DevArena &a;
        ~Guard() { a.release_all(); }
    } guard{tmp};
    sptrsv_status_t st;

    AnalysisStatus *d_stat = nullptr;
    if ((st = tmp.alloc_n(&d_stat, 1)) != SPTRSV_SUCCESS) return st;
    AnalysisStatus init{INT32_MAX, INT32_MAX, 0, -1, 0ull, 0ull, 0, 0};
    SPTRSV_CUDA(cudaMemcpyAsync(d_stat, &init, sizeof(init), cudaMemcpyHostToDevice, s));
    k_nnz_input<<<1, 1, 0, s>>>(rowptr, n, d_stat);

    if ((st = h->arena.alloc_n(&h->d_dp, n)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc(&h->d_invd_row, (size_t)n * h->esize)) != SPTRSV_SUCCESS) return st;
    const int vgrid = grid_for((int64_t)n * 32, 256, h->num_sms * 16);
    if (h->dtype == SPTRSV_F64)
        k_validate<double><<<vgrid, 256, 0, s>>>(n, rowptr, colidx, (const double *)vals, h->uplo, h->diag,
                                                 h->d_dp, (double *)h->d_invd_row, d_stat);
    else
        k_validate<float><<<vgrid, 256, 0, s>>>(n, rowptr, colidx, (const float *)vals, h->uplo, h->diag,
                                                h->d_dp, (float *)h->d_invd_row, d_stat);
    SPTRSV_CUDA(cudaGetLastError());
    AnalysisStatus hs;
    SPTRSV_CUDA(cudaMemcpyAsync(&hs, d_stat, sizeof(hs), cudaMemcpyDeviceToHost, s));
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    h->info.nnz_input = hs.nnz_input;
    h->info.ignored_entries = (int64_t)hs.ignored;
    h->info.nnz_used = (int64_t)hs.used;
    h->info.max_row_deps = hs.max_deps;
    if (hs.bad_row != INT32_MAX) {
        h->info.bad_row = hs.bad_row;
        h->info.ignored_entries = 0;
        h->info.nnz_used = 0;
        return SPTRSV_ERR_INVALID_MATRIX;
    }
    if (hs.zero_pivot_row != INT32_MAX) {
        h->info.zero_pivot_row = hs.zero_pivot_row;
        return SPTRSV_ERR_ZERO_PIVOT;
    }
    // UNIT without values: only a triangle without off-diagonal entries has
    // nothing to read (it used to solve with zero coefficients)
    if (!vals && hs.used > 0) return SPTRSV_ERR_INVALID_VALUE;

    phase("validate");
    // a3: levels
    if ((st = h->arena.alloc_n(&h->d_lev, n)) != SPTRSV_SUCCESS) return st;
    unsigned *d_ticket = nullptr;
    if ((st = tmp.alloc_n(&d_ticket, 1)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemsetAsync(d_ticket, 0, sizeof(unsigned), s));
    SPTRSV_CUDA(cudaMemsetAsync(h->d_lev, 0xFF, sizeof(int32_t) * (size_t)n, s));
    const int mode = g_levels_mode;                          // sptrsv_dbg_levels_mode (analysis study)
    if (mode == 1) {
        k_levels<<<grid_for(((int64_t)n + 31) / 32 * 32, 256, h->num_sms * 8), 256, 0, s>>>(
            n, rowptr, colidx, h->uplo, h->d_lev, d_ticket, d_stat);
    } else {
        // CSC of the referenced strict triangle (dependents), then Kahn by rounds
        int32_t *ccnt = nullptr, *cptr = nullptr, *ccur = nullptr, *crow = nullptr, *indeg = nullptr;
        int32_t *F0 = nullptr, *F1 = nullptr, *fcnt = nullptr;
        unsigned long long *kbar = nullptr;
        const int64_t nstrict = (int64_t)hs.used;           // referenced strict entries
        if ((st = tmp.alloc_n(&ccnt, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
        if ((st = tmp.alloc_n(&cptr, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
        if ((st = tmp.alloc_n(&ccur, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
        if ((st = tmp.alloc_n(&crow, (size_t)std::max<int64_t>(nstrict, 1))) != SPTRSV_SUCCESS) return st;
        if ((st = tmp.alloc_n(&indeg, (size_t)n)) != SPTRSV_SUCCESS) return st;
        if ((st = tmp.alloc_n(&F0, (size_t)n)) != SPTRSV_SUCCESS) return st;
        if ((st = tmp.alloc_n(&F1, (size_t)n)) != SPTRSV_SUCCESS) return st;
        if ((st = tmp.alloc_n(&fcnt, 3)) != SPTRSV_SUCCESS) return st;
        if ((st = tmp.alloc_n(&kbar, 1)) != SPTRSV_SUCCESS) return st;
        SPTRSV_CUDA(cudaMemsetAsync(ccnt, 0, sizeof(int32_t) * ((size_t)n + 1), s));
        SPTRSV_CUDA(cudaMemsetAsync(ccur, 0, sizeof(int32_t) * ((size_t)n + 1), s));
        SPTRSV_CUDA(cudaMemsetAsync(fcnt, 0, sizeof(int32_t) * 3, s));
        SPTRSV_CUDA(cudaMemsetAsync(kbar, 0, sizeof(unsigned long long), s));
        const int wg = grid_for((int64_t)n * 32, 256, h->num_sms * 16);
        k_dep_count<<<wg, 256, 0, s>>>(n, rowptr, colidx, h->uplo, ccnt);
        if ((st = exclusive_scan_i32(ccnt, cptr, (int64_t)n + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
        k_dep_fill<<<wg, 256, 0, s>>>(n, rowptr, colidx, h->uplo, cptr, ccur, crow);
        SPTRSV_CUDA(cudaMemcpyAsync(indeg, h->d_dp, sizeof(int32_t) * (size_t)n, cudaMemcpyDeviceToDevice, s));
        k_frontier0<<<(n + 255) / 256, 256, 0, s>>>(n, h->d_dp, F0, fcnt);
        SPTRSV_CUDA(cudaGetLastError());
        if (mode == 2) {
            // the paper's host loop: one launch per level, the frontier size read back each time
            int nf = 0, l = 0;
            SPTRSV_CUDA(cudaMemcpyAsync(&nf, fcnt, sizeof(int), cudaMemcpyDeviceToHost, s));
            SPTRSV_CUDA(cudaStreamSynchronize(s));
            while (nf > 0) {
                int32_t *Fc = (l & 1) ? F1 : F0, *Fn = (l & 1) ? F0 : F1;
                int32_t *cn = fcnt + ((l + 1) & 1);
                SPTRSV_CUDA(cudaMemsetAsync(cn, 0, sizeof(int32_t), s));
                k_kahn_round<<<grid_for((int64_t)nf * 32, 256, h->num_sms * 8), 256, 0, s>>>(nf, l, cptr, crow, indeg,
                                                                                           Fc, Fn, cn, h->d_lev);
                SPTRSV_CUDA(cudaGetLastError());
                SPTRSV_CUDA(cudaMemcpyAsync(&nf, cn, sizeof(int), cudaMemcpyDeviceToHost, s));
                SPTRSV_CUDA(cudaStreamSynchronize(s));
                ++l;
            }
            AnalysisStatus hl;
            SPTRSV_CUDA(cudaMemcpyAsync(&hl, d_stat, sizeof(hl), cudaMemcpyDeviceToHost, s));
            SPTRSV_CUDA(cudaStreamSynchronize(s));
            hl.max_lev = l - 1;
            SPTRSV_CUDA(cudaMemcpyAsync(d_stat, &hl, sizeof(hl), cudaMemcpyHostToDevice, s));
        } else {
            int per_sm = 0;
            SPTRSV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_kahn, kKahnThreads, 0));
            const int kg = std::max(1, std::min(per_sm, 1)) * h->num_sms;
            void *args[] = {(void *)&n, (void *)&cptr, (void *)&crow, (void *)&indeg, (void *)&F0, (void *)&F1,
                            (void *)&fcnt, (void *)&h->d_lev, (void *)&kbar, (void *)&d_stat};
            SPTRSV_CUDA(cudaLaunchCooperativeKernel((const void *)k_kahn, kg, kKahnThreads, args, 0, s));
        }
    }
    SPTRSV_CUDA(cudaGetLastError());
    SPTRSV_CUDA(cudaMemcpyAsync(&hs, d_stat, sizeof(hs), cudaMemcpyDeviceToHost, s));
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    const int nlev = hs.max_lev + 1;
    h->info.nlev = nlev;
    if ((uint64_t)nlev * kBuckets >= (1ull << 32)) return SPTRSV_ERR_NOT_SUPPORTED;

    phase("levels");
    // a4: jlev = rows stably sorted by level; ilev = level boundaries
    uint32_t *keys = nullptr, *skeys = nullptr;
    if ((st = tmp.alloc_n(&keys, n)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&skeys, n)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&h->d_jlev, n)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&h->d_ilev, (size_t)nlev + 1)) != SPTRSV_SUCCESS) return st;
    const int eg = (n + 255) / 256;
    k_level_keys<<<eg, 256, 0, s>>>(h->d_lev, n, keys);
    if ((st = radix_sort_pairs(keys, nullptr, skeys, h->d_jlev, n, (uint32_t)(nlev - 1), tmp, s)) != SPTRSV_SUCCESS)
        return st;
    k_ilev_from_sorted<<<eg, 256, 0, s>>>(skeys, n, nlev, h->d_ilev);
    SPTRSV_CUDA(cudaGetLastError());

    phase("bucket");
    // a5: solve order (level, WPR first, TPR by decreasing deps) and chunks
    if ((st = h->arena.alloc_n(&h->d_perm, n)) != SPTRSV_SUCCESS) return st;
    k_solve_keys<<<eg, 256, 0, s>>>(h->d_lev, h->d_dp, n, keys);
    if ((st = radix_sort_pairs(keys, nullptr, skeys, h->d_perm, n, (uint32_t)nlev * kBuckets - 1, tmp, s)) !=
        SPTRSV_SUCCESS)
        return st;
    int32_t *wcnt = nullptr, *nch = nullptr;
    if ((st = tmp.alloc_n(&wcnt, (size_t)nlev + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&nch, (size_t)nlev + 1)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemsetAsync(wcnt, 0, sizeof(int32_t) * ((size_t)nlev + 1), s));
    k_count_wpr<<<eg, 256, 0, s>>>(skeys, n, wcnt);
    if ((st = h->arena.alloc_n(&h->d_lev_chunk, (size_t)nlev + 1)) != SPTRSV_SUCCESS) return st;
    k_chunks_per_level<<<(nlev + 1 + 255) / 256, 256, 0, s>>>(h->d_ilev, wcnt, nlev, nch);
    if ((st = exclusive_scan_i32(nch, h->d_lev_chunk, (int64_t)nlev + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    int32_t nchunks = 0;
    SPTRSV_CUDA(cudaMemcpyAsync(&nchunks, h->d_lev_chunk + nlev, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    h->nchunks = nchunks;
    int64_t *ecount = nullptr, *eptr = nullptr;
    if ((st = h->arena.alloc_n(&h->d_chunks, (size_t)nchunks + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&ecount, (size_t)nchunks + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&eptr, (size_t)nchunks + 1)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemsetAsync(ecount, 0, sizeof(int64_t) * ((size_t)nchunks + 1), s));
    if ((st = h->arena.alloc_n(&h->d_chunk_lev, (size_t)nchunks + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&h->d_done, (size_t)nlev + 1)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemsetAsync(h->d_done, 0, sizeof(unsigned) * ((size_t)nlev + 1), s));
    h->self_epoch = 0;
    k_chunk_desc<<<(nlev + 127) / 128, 128, 0, s>>>(h->d_ilev, wcnt, h->d_lev_chunk, nlev, h->d_perm, h->d_dp,
                                                     h->d_chunks, ecount, h->d_chunk_lev);
    SPTRSV_CUDA(cudaGetLastError());
    if ((st = exclusive_scan_i64(ecount, eptr, (int64_t)nchunks + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    int64_t nent = 0;
    SPTRSV_CUDA(cudaMemcpyAsync(&nent, eptr + nchunks, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    h->nent = nent;
    if ((st = h->arena.alloc_n(&h->d_ecol, (size_t)std::max<int64_t>(nent, 1))) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc(&h->d_eval, (size_t)std::max<int64_t>(nent, 1) * h->esize)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc(&h->d_invd, (size_t)n * h->esize)) != SPTRSV_SUCCESS) return st;
    if (nchunks > 0) k_patch_eptr<<<(nchunks + 255) / 256, 256, 0, s>>>(h->d_chunks, eptr, nchunks);
    const int fgrid = grid_for((int64_t)nchunks * 32, 256, h->num_sms * 16);
    if (h->dtype == SPTRSV_F64)
        k_fill<double><<<fgrid, 256, 0, s>>>(nchunks, h->d_chunks, eptr, h->d_perm, rowptr, colidx,
                                             (const double *)vals, (const double *)h->d_invd_row, h->uplo,
                                             h->d_ecol, (double *)h->d_eval, (double *)h->d_invd);
    else
        k_fill<float><<<fgrid, 256, 0, s>>>(nchunks, h->d_chunks, eptr, h->d_perm, rowptr, colidx,
                                            (const float *)vals, (const float *)h->d_invd_row, h->uplo,
                                            h->d_ecol, (float *)h->d_eval, (float *)h->d_invd);
    SPTRSV_CUDA(cudaGetLastError());

    phase("layout");
    // synchronisation state
    if ((st = h->arena.alloc_n(&h->d_flags, n)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemsetAsync(h->d_flags, 0, sizeof(int32_t) * (size_t)n, s));
    if ((st = h->arena.alloc_n(&h->d_ctr, 4)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemsetAsync(h->d_ctr, 0, sizeof(unsigned) * 4, s));
    // per-CTA arrival slots of the level-scheduled grid barrier (<= 64 CTAs per SM)
    if ((st = h->arena.alloc_n(&h->d_bar, (size_t)h->num_sms * 64)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemsetAsync(h->d_bar, 0, sizeof(unsigned long long) * (size_t)h->num_sms * 64, s));
    h->epoch = 0;
    h->bar_base = 0;

    phase("sync");
    // summary: widest level and rowptr[n], one read with the status
    k_summary<<<(nlev + 255) / 256, 256, 0, s>>>(nlev, h->d_ilev, d_stat);
    SPTRSV_CUDA(cudaGetLastError());
    SPTRSV_CUDA(cudaMemcpyAsync(&hs, d_stat, sizeof(hs), cudaMemcpyDeviceToHost, s));
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    h->info.max_level_width = hs.max_width;
    phase("summary");
    return SPTRSV_SUCCESS;
}

// sptrsv_update_values (NEXT-2; numerical refactorization keeps the
// pattern, so the analysis is reused): validate the new values with the same
// rules as sptrsv_analyze, check that the referenced pattern is the analyzed
// one (dependency counts and the level-ordered column ids equal), then
// replace the values of every layout the handle holds.  On any error the
// handle keeps its old values.
sptrsv_status_t update_values_impl(sptrsv_handle_t h, const int32_t *rowptr, const int32_t *colidx,
                                   const void *vals, cudaStream_t s) {
    const int n = h->n;
    DevArena tmp(s);
    struct Guard {
        DevArena &a;
        ~Guard() { a.release_all(); }
    } guard{tmp};
    sptrsv_status_t st;
    AnalysisStatus *d_stat = nullptr;
    int32_t *dp = nullptr, *ecol = nullptr;
    void *invd_row = nullptr, *eval = nullptr, *invd = nullptr;
    int64_t *eptr = nullptr;
    unsigned *cnt = nullptr;
    const size_t es = h->esize;
    if ((st = tmp.alloc_n(&d_stat, 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&dp, (size_t)n)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc(&invd_row, (size_t)n * es)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&ecol, (size_t)std::max<int64_t>(h->nent, 1))) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc(&eval, (size_t)std::max<int64_t>(h->nent, 1) * es)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc(&invd, (size_t)n * es)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&eptr, (size_t)h->nchunks + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&cnt, 2)) != SPTRSV_SUCCESS) return st;
    AnalysisStatus init{INT32_MAX, INT32_MAX, 0, -1, 0ull, 0ull, 0, 0};
    SPTRSV_CUDA(cudaMemcpyAsync(d_stat, &init, sizeof(init), cudaMemcpyHostToDevice, s));
    SPTRSV_CUDA(cudaMemsetAsync(cnt, 0, 2 * sizeof(unsigned), s));
    const int vgrid = grid_for((int64_t)n * 32, 256, h->num_sms * 16);
    const int fgrid = grid_for((int64_t)h->nchunks * 32, 256, h->num_sms * 16);
    const bool f64 = h->dtype == SPTRSV_F64;
    if (f64)
        k_validate<double><<<vgrid, 256, 0, s>>>(n, rowptr, colidx, (const double *)vals, h->uplo, h->diag, dp,
                                                 (double *)invd_row, d_stat);
    else
        k_validate<float><<<vgrid, 256, 0, s>>>(n, rowptr, colidx, (const float *)vals, h->uplo, h->diag, dp,
                                                (float *)invd_row, d_stat);
    k_count_diff<<<(n + 255) / 256, 256, 0, s>>>(n, dp, h->d_dp, cnt);
    if (h->nchunks > 0) {
        k_chunk_eptr<<<(h->nchunks + 255) / 256, 256, 0, s>>>(h->nchunks, h->d_chunks, eptr);
        if (f64)
            k_fill<double><<<fgrid, 256, 0, s>>>(h->nchunks, h->d_chunks, eptr, h->d_perm, rowptr, colidx,
                                                 (const double *)vals, (const double *)invd_row, h->uplo, ecol,
                                                 (double *)eval, (double *)invd);
        else
            k_fill<float><<<fgrid, 256, 0, s>>>(h->nchunks, h->d_chunks, eptr, h->d_perm, rowptr, colidx,
                                                (const float *)vals, (const float *)invd_row, h->uplo, ecol,
                                                (float *)eval, (float *)invd);
        k_count_diff<<<(int)((h->nent + 255) / 256), 256, 0, s>>>(h->nent, ecol, h->d_ecol, cnt + 1);
    }
    SPTRSV_CUDA(cudaGetLastError());
    AnalysisStatus hs;
    unsigned hc[2] = {0, 0};
    SPTRSV_CUDA(cudaMemcpyAsync(&hs, d_stat, sizeof(hs), cudaMemcpyDeviceToHost, s));
    SPTRSV_CUDA(cudaMemcpyAsync(hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, s));
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    if (hs.bad_row != INT32_MAX) return SPTRSV_ERR_INVALID_MATRIX;
    if (hs.zero_pivot_row != INT32_MAX) return SPTRSV_ERR_ZERO_PIVOT;
    if (hc[0] != 0 || hc[1] != 0 || (int64_t)hs.used != h->info.nnz_used) return SPTRSV_ERR_INVALID_VALUE;   // not the analyzed pattern
    // commit: level-ordered layout
    SPTRSV_CUDA(cudaMemcpyAsync(h->d_invd_row, invd_row, (size_t)n * es, cudaMemcpyDeviceToDevice, s));
    SPTRSV_CUDA(cudaMemcpyAsync(h->d_invd, invd, (size_t)n * es, cudaMemcpyDeviceToDevice, s));
    if (h->nent > 0) SPTRSV_CUDA(cudaMemcpyAsync(h->d_eval, eval, (size_t)h->nent * es, cudaMemcpyDeviceToDevice, s));
    // derived layouts
    if ((st = refresh_derived_values(h, s)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    return SPTRSV_SUCCESS;
}

}  // namespace sptrsv
