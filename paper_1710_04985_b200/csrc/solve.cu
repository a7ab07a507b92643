// solve.cu -- the solve phase over the level-ordered layout built by analyze.cu.
//
//   k_self   a6: self-scheduled solve (Alg. 3 SLFR; kernel P:577-619),
//            re-expressed with PULL-style per-row ready flags.  The flag of row
//            j is its value x(j) itself: x is prefilled with a NaN-payload
//            sentinel (k_prefill) and a row spins on relaxed loads of its
//            dependencies until none is the sentinel, then stores x(i) with a
//            relaxed store.  64-bit aligned accesses are single-copy atomic,
//            so no fence is needed (the paper's __threadfence, P:603, P:616-619,
//            becomes unnecessary) -- one L2 round trip per handoff.
//            Warps claim 32-row chunks by an atomic ticket in jlev order (the
//            paper's warp-unknown mapping), so a wait only ever
//            targets rows claimed earlier by running warps: deadlock-free for
//            any grid size (the paper's static wid mapping is not).
//   k_level  a7: level-scheduled solve (Alg. 1 LEVR): one persistent
//            co-resident grid, a grid-wide barrier between levels instead of
//            one launch per level.
//   k_mrhs   a8: multiple right-hand sides: one flag per row, lanes over RHS.
//
// Row arithmetic (all kernels, all dtypes): s = b(i); s = fma(-a(k), x(ja(k)), s)
// in storage order; x(i) = s * inv_d(i) (UNIT: s).  WPR rows in k_self /
// k_level reduce lane partial sums with a fixed shuffle tree.
#include <algorithm>
#include <vector>

#include <cstdlib>

#include "internal.h"

namespace sptrsv {
namespace {

constexpr int kThreads = 256;
// back-off between SELF poll rounds (ns)
#ifndef SPTRSV_SELF_POLL_NS
#define SPTRSV_SELF_POLL_NS 20
#endif
constexpr unsigned kSelfPollNs = SPTRSV_SELF_POLL_NS;

// Debug hook (sptrsv_dbg_self_trace, not part of include/sptrsv.h): when set,
// k_self writes %globaltimer at the publication of every row.
__device__ unsigned long long *g_tpub = nullptr;
__device__ __forceinline__ void trace_pub(unsigned long long *p, int row) {
    if (p != nullptr) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p[row] = t;
    }
}

template <typename T, bool UNIT>
__device__ __forceinline__ T finish(T s, T di) { return UNIT ? s : s * di; }

// Wait until every dependency of this lane is published (relaxed polling of
// all flags at once, then one acquire fence for the whole set).
template <int N>
__device__ __forceinline__ void wait_flags(const int *flags, const int (&cols)[N], int width, int epoch) {
    unsigned pend = 0;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        if (k < width && cols[k] >= 0 && ld_relaxed(&flags[cols[k]]) != epoch) pend |= 1u << k;
    }
    int spins = 0;
    while (pend) {
        if (++spins > 8) __nanosleep(32);
#pragma unroll
        for (int k = 0; k < N; ++k) {
            if ((pend >> k) & 1u) {
                if (ld_relaxed(&flags[cols[k]]) == epoch) pend &= ~(1u << k);
            }
        }
    }
}

// Value-as-flag wait: re-load every pending value (relaxed, L2) after a short
// sleep until none is the sentinel.  (A two-wave variant with reloads half a
// round trip apart measured slower on cfg4: 38 vs 32 ms, the spinning warps
// load the SMs and L2 more than the shorter overshoot saves.)
template <typename T, int N>
__device__ __forceinline__ bool pending_any(const int (&c)[N], const T (&v)[N]) {
    bool pend = false;
#pragma unroll
    for (int u = 0; u < N; ++u) pend |= c[u] >= 0 && Sentinel<T>::is(v[u]);
    return pend;
}
template <typename T, int N>
__device__ __forceinline__ void reload_pending(const int (&c)[N], T (&v)[N], const T *x) {
#pragma unroll
    for (int u = 0; u < N; ++u)
        if (c[u] >= 0 && Sentinel<T>::is(v[u])) v[u] = ld_relaxed_val(x + c[u]);
}
// ---------------------------------------------------------------- TPR row
// One chunk of up to 32 rows, thread per row.  Entry k of lane r at
// eptr + k*32 + r.  WAIT: dependencies are polled as VALUES (value-as-flag,
// x prefilled with Sentinel<T>): every pending value is re-loaded with a
// relaxed (L2-coherent) load until it is no longer the sentinel -- one L2
// round trip per handoff and no fences (B200 measurement: a fence after
// stores costs ~580 ns, the relaxed handoff ~220 ns; profiles/).
template <typename T, bool UNIT, bool WAIT>
__device__ __forceinline__ void tpr_chunk(const ChunkDesc &cd, int lane, const int32_t *__restrict__ perm,
                                          const T *__restrict__ invd, const int32_t *__restrict__ ecol,
                                          const T *__restrict__ eval, const T *b, T *x,
                                          unsigned long long *tp = nullptr) {
    const int nr = chunk_nrows(cd.meta), width = chunk_width(cd.meta);
    const bool act = lane < nr;
    int row = 0;
    T di = T(0), s = T(0);
    if (act) {
        row = perm[cd.pos + lane];
        di = invd[cd.pos + lane];
        s = ld_cg(b + row);
    }
    int cols[kTprMax];
    T vals[kTprMax];
    T xv[kTprMax];
    const int32_t *ec = ecol + cd.eptr + lane;
    const T *ev = eval + cd.eptr + lane;
#pragma unroll
    for (int k = 0; k < kTprMax; ++k) {
        cols[k] = -1;
        vals[k] = T(0);
        if (k < width) {
            cols[k] = ld_stream(ec + k * 32);
            vals[k] = ld_stream(ev + k * 32);
        }
    }
    if (WAIT) {
#pragma unroll
        for (int k = 0; k < kTprMax; ++k) xv[k] = (cols[k] >= 0) ? ld_relaxed_val(x + cols[k]) : T(0);
        // Warp-converged loop; each lane publishes as soon as its own row is
        // ready (not when the chunk's slowest lane is).  Every pending value is
        // re-polled each round (polling only the last one measured slower with
        // one CTA per SM: cfg4 26.8 vs 31.2 ms, cfg3 2.46 vs 2.91 ms).
        bool done = !act;
        for (;;) {
            if (!done && !pending_any<T, kTprMax>(cols, xv)) {
#pragma unroll
                for (int k = 0; k < kTprMax; ++k) {
                    if (cols[k] >= 0) s = fnma(vals[k], xv[k], s);
                }
                st_relaxed_val(x + row, Sentinel<T>::scrub(finish<T, UNIT>(s, di)));
                trace_pub(tp, row);
                done = true;
            }
            if (__all_sync(0xffffffffu, done)) return;
            __nanosleep(kSelfPollNs);
            reload_pending<T, kTprMax>(cols, xv, x);
        }
    } else {
#pragma unroll
        for (int k = 0; k < kTprMax; ++k) xv[k] = (cols[k] >= 0) ? ld_cg(x + cols[k]) : T(0);
    }
#pragma unroll
    for (int k = 0; k < kTprMax; ++k) {
        if (cols[k] >= 0) s = fnma(vals[k], xv[k], s);
    }
    if (act) {
        const T r = finish<T, UNIT>(s, di);
        if (WAIT) st_relaxed_val(x + row, Sentinel<T>::scrub(r));
        else x[row] = r;
    }
}

// ---------------------------------------------------------------- WPR row
template <typename T, bool UNIT, bool WAIT, int U = 8>
__device__ __forceinline__ void wpr_row(const ChunkDesc &cd, int lane, const int32_t *__restrict__ perm,
                                        const T *__restrict__ invd, const int32_t *__restrict__ ecol,
                                        const T *__restrict__ eval, const T *b, T *x,
                                        unsigned long long *tp = nullptr) {
    // Batches of 32 x U entries: every lane has U dependency loads in
    // flight at once (one L2 round trip per batch instead of per 32 entries),
    // and the next batch's indices/values are loaded before this batch is
    // polled.  Per lane the entries are still accumulated k = lane, lane+32,
    // ... in increasing order (bitwise equal to the one-at-a-time loop).
    const int width = chunk_width(cd.meta);
    const int row = perm[cd.pos];
    const int32_t *ec = ecol + cd.eptr;
    const T *ev = eval + cd.eptr;
    // b(i) and 1/d(i) before the dependencies: not a DRAM round trip after the reduction
    const T bi = lane == 0 ? ld_cg(b + row) : T(0);
    const T di = lane == 0 ? invd[cd.pos] : T(0);
    T acc = T(0);
    int cn[U];
    T an[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int k = u * 32 + lane;
        cn[u] = k < width ? ld_stream(ec + k) : -1;
        an[u] = k < width ? ld_stream(ev + k) : T(0);
    }
    for (int base = 0; base < width; base += 32 * U) {
        int c[U];
        T a[U], v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            c[u] = cn[u];
            a[u] = an[u];
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            v[u] = c[u] >= 0 ? (WAIT ? ld_relaxed_val(x + c[u]) : ld_cg(x + c[u])) : T(0);
        if (base + 32 * U < width) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int k = base + 32 * U + u * 32 + lane;
                cn[u] = k < width ? ld_stream(ec + k) : -1;
                an[u] = k < width ? ld_stream(ev + k) : T(0);
            }
        }
        if (WAIT) {
            while (pending_any<T, U>(c, v)) {       // (lazy polling measured slower here)
                __nanosleep(kSelfPollNs);
                reload_pending<T, U>(c, v, x);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (c[u] >= 0) acc = __fma_rn(a[u], v[u], acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
        const T r = finish<T, UNIT>(bi - acc, di);
        if (WAIT) {
            st_relaxed_val(x + row, Sentinel<T>::scrub(r));
            trace_pub(tp, row);
        }
        else x[row] = r;
    }
}

// ---------------------------------------------------------------- SELF
// x must hold Sentinel<T> in every row on entry (k_prefill).
template <typename T, bool UNIT, int U>
__global__ void __launch_bounds__(kThreads) k_self(const ChunkDesc *__restrict__ chunks, int nchunks,
                                                   const int32_t *__restrict__ perm, const T *__restrict__ invd,
                                                   const int32_t *__restrict__ ecol, const T *__restrict__ eval,
                                                   const T *b, T *x, unsigned *ctr, unsigned nwarps_total) {
    const int lane = threadIdx.x & 31;
    unsigned long long *tp = g_tpub;         // debug trace (read once)
    for (;;) {
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(&ctr[0], 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if ((int)t >= nchunks) break;
        const ChunkDesc cd = chunks[t];
        if (!chunk_wpr(cd.meta))
            tpr_chunk<T, UNIT, true>(cd, lane, perm, invd, ecol, eval, b, x, tp);
        else
            wpr_row<T, UNIT, true, U>(cd, lane, perm, invd, ecol, eval, b, x, tp);
    }
    // the last warp out resets the ticket for the next solve on this stream
    if (lane == 0) {
        unsigned e = atomicAdd(&ctr[1], 1u);
        if (e == nwarps_total - 1) {
            ctr[0] = 0;
            ctr[1] = 0;
        }
    }
}

template <typename T>
__global__ void k_prefill(T *x, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (; i < n; i += stride) x[i] = Sentinel<T>::value();
}

// ---------------------------------------------------------------- LEVEL
// Grid barrier over the co-resident grid (one CTA per SM): arrival is a
// release reduction on one monotone counter (no reset between solves), the
// wait is one thread polling it with relaxed loads, then an acquire fence.
__device__ __forceinline__ void grid_barrier(unsigned long long *bar, unsigned long long target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
        // acquire polls: no separate fence after the wait (a fence.acq_rel
        // costs ~150-580 ns on B200, profiles/microbench_r1.json)
        while (ld_acquire_u64(bar) < target) {
        }
    }
    __syncthreads();
}

constexpr int kLevelThreads = 1024;
// k_level (single RHS): 128 threads per CTA.  The grid barrier's two
// __syncthreads grow with the CTA, and a level of cfg2 keeps only ~170 warps
// busy: 1024 -> 128 threads took cfg2 2.20 -> 1.55 ms, cfg3 12.1 -> 5.9 ms,
// cfg4 61.5 -> 55.8 ms (SPTRSV_LEVEL_THREADS overrides).
constexpr int kLevelThreads1 = 128;

template <typename T, bool UNIT>
__global__ void __launch_bounds__(kLevelThreads1, 1) k_level(const ChunkDesc *__restrict__ chunks,
                                                    const int32_t *__restrict__ lev_chunk, int nlev,
                                                    const int32_t *__restrict__ perm, const T *__restrict__ invd,
                                                    const int32_t *__restrict__ ecol, const T *__restrict__ eval,
                                                    const T *b, T *x, unsigned long long *bar,
                                                    unsigned long long bar_base) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int l = 0; l < nlev; ++l) {
        const int c0 = lev_chunk[l], c1 = lev_chunk[l + 1];
        for (int c = c0 + gw; c < c1; c += nw) {
            const ChunkDesc cd = chunks[c];
            if (!chunk_wpr(cd.meta))
                tpr_chunk<T, UNIT, false>(cd, lane, perm, invd, ecol, eval, b, x);
            else
                wpr_row<T, UNIT, false>(cd, lane, perm, invd, ecol, eval, b, x);
        }
        if (l + 1 < nlev) grid_barrier(bar, bar_base + (unsigned long long)(l + 1) * gridDim.x);
    }
}

// ---------------------------------------------------------------- MRHS
// Multiple right-hand sides (a8).  Warp per ROW, lanes over the RHS columns
// (CPL columns per lane), rows claimed by ticket in the solve order (levels
// ascending), G rows per claim so that the b rows and entries of the next
// rows are in flight while the first one waits on its dependencies.  One
// ready flag per row (epoch-tagged): polled with acquire loads by the lanes
// holding the dependencies, published with a release store after the row's
// x values.  Per (row, column) the arithmetic is the TPR sequence, so each
// column equals the nrhs == 1 TPR result bitwise and does not depend on nrhs
// (SURVEY §8e partition invariant).  Entries come from a per-position CSR
// (mr_*), built on the first multi-RHS solve.
// Multi-RHS with per-(row, column) value-as-flag (k_mrhs_vf, nrhs <= 16):
// x is prefilled with the sentinel; a warp claims 32/W rows by ticket in
// solve order (W = nrhs rounded up to a power of two), lane = (row slot,
// column).  A lane polls only ITS column of its row's dependencies (relaxed
// loads, all in flight at once) and publishes x(row, column) with a relaxed
// store: no flags, no fences -- the SELF protocol per column.  Per column the
// arithmetic is the TPR sequence (bitwise equal to the other multi-RHS
// kernels and to nrhs == 1).  The level-scheduled kernel costs ~4.5 us per
// level whatever nrhs is (tools/mrhs_sweep.py), so for the few columns of a
// multi-GPU rank (cfg5: 64/G) this is the faster path.
template <typename T, bool UNIT, int W>
__global__ void __launch_bounds__(kThreads) k_mrhs_vf(int n, const int32_t *__restrict__ perm,
                                                      const T *__restrict__ invd,
                                                      const int32_t *__restrict__ mr_ptr,
                                                      const int32_t *__restrict__ mr_col,
                                                      const T *__restrict__ mr_val, const T *b, T *x, int nrhs,
                                                      int64_t ld, unsigned *ctr, unsigned nwarps_total) {
    constexpr int RPW = 32 / W;               // rows per warp
    constexpr int DB = 8;                     // dependency loads in flight per lane
    const int lane = threadIdx.x & 31;
    const int g = lane / W, c = lane % W;
    for (;;) {
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(&ctr[0], (unsigned)RPW);
        t = __shfl_sync(0xffffffffu, t, 0);
        if ((int)t >= n) break;
        const int p = (int)t + g;
        if (p < n && c < nrhs) {
            const int row = perm[p];
            const T di = invd[p];
            const int e0 = mr_ptr[p], e1 = mr_ptr[p + 1];
            T acc = ld_cg(b + (int64_t)row * ld + c);
            for (int k0 = e0; k0 < e1; k0 += DB) {
                int cj[DB];
                T a[DB], v[DB];
#pragma unroll
                for (int u = 0; u < DB; ++u) {
                    cj[u] = k0 + u < e1 ? mr_col[k0 + u] : -1;
                    a[u] = k0 + u < e1 ? mr_val[k0 + u] : T(0);
                }
#pragma unroll
                for (int u = 0; u < DB; ++u) v[u] = cj[u] >= 0 ? ld_relaxed_val(x + (int64_t)cj[u] * ld + c) : T(0);
                for (;;) {
                    bool pend = false;
#pragma unroll
                    for (int u = 0; u < DB; ++u) pend |= cj[u] >= 0 && Sentinel<T>::is(v[u]);
                    if (!pend) break;
                    __nanosleep(20);
#pragma unroll
                    for (int u = 0; u < DB; ++u)
                        if (cj[u] >= 0 && Sentinel<T>::is(v[u])) v[u] = ld_relaxed_val(x + (int64_t)cj[u] * ld + c);
                }
#pragma unroll
                for (int u = 0; u < DB; ++u)
                    if (cj[u] >= 0) acc = fnma(a[u], v[u], acc);
            }
            st_relaxed_val(x + (int64_t)row * ld + c, Sentinel<T>::scrub(finish<T, UNIT>(acc, di)));
        }
        __syncwarp();
    }
    if (lane == 0) {
        const unsigned e = atomicAdd(&ctr[1], 1u);
        if (e == nwarps_total - 1) {
            ctr[0] = 0;
            ctr[1] = 0;
        }
    }
}

sptrsv_status_t ensure_scratch(sptrsv_handle_t h, size_t bytes, cudaStream_t s);
// nrhs <= 16 columns (kVfMax): one launch; the caller handles the in-place copy
template <typename T, bool UNIT>
sptrsv_status_t launch_mrhs_vf(sptrsv_handle_t h, const T *b, T *x, int ncols, int64_t ld, cudaStream_t s) {
    auto kern = ncols <= 2 ? k_mrhs_vf<T, UNIT, 2> : ncols <= 4 ? k_mrhs_vf<T, UNIT, 4>
              : ncols <= 8 ? k_mrhs_vf<T, UNIT, 8> : k_mrhs_vf<T, UNIT, 16>;
    // 4 CTAs per SM (occupancy permitting), computed once per handle
    if (h->vf_grid == 0) {
        int per_sm = 0;
        SPTRSV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mrhs_vf<T, UNIT, 16>, kThreads, 0));
        h->vf_grid = std::max(1, std::min(per_sm, 4)) * h->num_sms;
    }
    const int grid = h->vf_grid;
    kern<<<grid, kThreads, 0, s>>>(h->n, h->d_perm, (const T *)h->d_invd, h->d_mr_ptr, h->d_mr_col,
                                   (const T *)h->d_mr_val, b, x, ncols, ld, h->d_ctr, (unsigned)(grid * (kThreads / 32)));
    SPTRSV_CUDA(cudaGetLastError());
    return SPTRSV_SUCCESS;
}

// Level-scheduled multiple right-hand sides (Alg. 1 LEVR over nrhs columns):
// warp per row of the current level (grid-stride over the level's positions,
// lanes over columns), then a grid barrier.  No flags: the barrier orders
// the levels.  The b rows of the next level are prefetched into L2 before
// the barrier.
template <typename T, int CPL>
struct MrRow {
    int row, e0, deg, col;
    T di, val;
    T bv[CPL];
};

template <typename T, int CPL>
__device__ __forceinline__ void mr_load(MrRow<T, CPL> &R, int p, int lane, const int32_t *__restrict__ perm,
                                        const T *__restrict__ invd, const int32_t *__restrict__ mr_ptr,
                                        const int32_t *__restrict__ mr_col, const T *__restrict__ mr_val, const T *b,
                                        int nrhs, int64_t ld) {
    R.row = perm[p];
    R.di = invd[p];
    R.e0 = mr_ptr[p];
    R.deg = mr_ptr[p + 1] - R.e0;
    R.col = lane < R.deg ? mr_col[R.e0 + lane] : 0;
    R.val = lane < R.deg ? mr_val[R.e0 + lane] : T(0);
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
        const int c = lane + 32 * j;
        if (c < nrhs) R.bv[j] = ld_cg(b + (int64_t)R.row * ld + c);
    }
}

template <typename T, bool UNIT, int CPL>
__device__ __forceinline__ void mr_solve(const MrRow<T, CPL> &R, int lane, const int32_t *__restrict__ mr_col,
                                         const T *__restrict__ mr_val, T *x, int nrhs, int64_t ld) {
    // the x rows of the first kBatch dependencies are loaded together (one
    // memory latency instead of one per dependency); the FMAs then run in
    // storage order, as before
    constexpr int kBatch = 4;
    T acc[CPL];
#pragma unroll
    for (int j = 0; j < CPL; ++j) acc[j] = R.bv[j];
    T xv[kBatch][CPL];
#pragma unroll
    for (int k = 0; k < kBatch; ++k) {
        const int ck = __shfl_sync(0xffffffffu, R.col, k);
#pragma unroll
        for (int j = 0; j < CPL; ++j) {
            const int c = lane + 32 * j;
            xv[k][j] = (k < R.deg && c < nrhs) ? ld_cg(x + (int64_t)ck * ld + c) : T(0);
        }
    }
#pragma unroll
    for (int k = 0; k < kBatch; ++k) {
        const T vk = __shfl_sync(0xffffffffu, R.val, k);
        if (k < R.deg) {
#pragma unroll
            for (int j = 0; j < CPL; ++j) acc[j] = fnma(vk, xv[k][j], acc[j]);
        }
    }
    for (int k = kBatch; k < R.deg; ++k) {
        const int ck = k < 32 ? __shfl_sync(0xffffffffu, R.col, k) : mr_col[R.e0 + k];
        const T vk = k < 32 ? __shfl_sync(0xffffffffu, R.val, k) : mr_val[R.e0 + k];
#pragma unroll
        for (int j = 0; j < CPL; ++j) {
            const int c = lane + 32 * j;
            if (c < nrhs) acc[j] = fnma(vk, ld_cg(x + (int64_t)ck * ld + c), acc[j]);
        }
    }
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
        const int c = lane + 32 * j;
        if (c < nrhs) x[(int64_t)R.row * ld + c] = finish<T, UNIT>(acc[j], R.di);
    }
}

// Level-scheduled multiple right-hand sides (Alg. 1 LEVR over nrhs columns):
// warp per row of the current level (grid-stride over the level's positions,
// lanes over columns), then a grid barrier.  No flags: the barrier orders the
// levels.  Each warp loads the metadata and b of its FIRST row of the next
// level before the barrier, so after it only the x loads of the dependencies
// remain on the critical path.
template <typename T, bool UNIT, int CPL>
__global__ void __launch_bounds__(kLevelThreads, 1) k_level_mrhs(const int32_t *__restrict__ ilev, int nlev,
                                                         const int32_t *__restrict__ perm, const T *__restrict__ invd,
                                                         const int32_t *__restrict__ mr_ptr,
                                                         const int32_t *__restrict__ mr_col,
                                                         const T *__restrict__ mr_val, const T *b, T *x, int nrhs,
                                                         int64_t ld, unsigned long long *bar, unsigned long long bar_base) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    MrRow<T, CPL> pre;
    int have = 0;
    if (nlev > 0 && ilev[0] + gw < ilev[1]) {
        mr_load(pre, ilev[0] + gw, lane, perm, invd, mr_ptr, mr_col, mr_val, b, nrhs, ld);
        have = 1;
    }
    for (int l = 0; l < nlev; ++l) {
        const int p0 = ilev[l], p1 = ilev[l + 1];
        // further rows of this level (wide levels): the next row's metadata and
        // b are loaded before the current row is solved
        for (int p = p0 + gw; have; p += nw) {
            MrRow<T, CPL> nxt;
            const bool more = p + nw < p1;
            if (more) mr_load(nxt, p + nw, lane, perm, invd, mr_ptr, mr_col, mr_val, b, nrhs, ld);
            mr_solve<T, UNIT, CPL>(pre, lane, mr_col, mr_val, x, nrhs, ld);
            if (!more) break;
            pre = nxt;
        }
        if (l + 1 < nlev) {
            have = 0;
            const int q = ilev[l + 1] + gw;
            if (q < ilev[l + 2]) {
                mr_load(pre, q, lane, perm, invd, mr_ptr, mr_col, mr_val, b, nrhs, ld);
                have = 1;
            }
            grid_barrier(bar, bar_base + (unsigned long long)(l + 1) * gridDim.x);
        }
    }
}

// ---------------------------------------------------------------- SMALL
// Small systems (SPTRSV_ALGO_SMALL; AUTO when the level-ordered layout fits in
// shared memory): ONE CTA of 32 x (widest level's chunks) threads solves the
// whole triangle level by level (LEVR) with the layout -- chunk
// descriptors, level ranges, permutation, 1/d, entries -- and x staged in
// shared memory: a level costs a CTA barrier and shared-memory latencies, not a
// grid barrier or an L2 round trip.  The per-row arithmetic is the TPR / WPR
// sequence of the other row kernels (bitwise equal to SELF and LEVEL).
struct SmallLayout {
    uint32_t off_chunks, off_levc, off_perm, off_invd, off_ecol, off_eval, off_x, bytes;
};
__host__ __device__ inline uint32_t align16(uint32_t v) { return (v + 15u) & ~15u; }
__host__ __device__ inline SmallLayout small_layout(int n, int nlev, int nchunks, int64_t nent, int es) {
    SmallLayout L;
    uint32_t o = 0;
    L.off_chunks = o; o = align16(o + (uint32_t)nchunks * 16u);
    L.off_levc = o;   o = align16(o + (uint32_t)(nlev + 1) * 4u);
    L.off_perm = o;   o = align16(o + (uint32_t)n * 4u);
    L.off_invd = o;   o = align16(o + (uint32_t)n * (uint32_t)es);
    L.off_ecol = o;   o = align16(o + (uint32_t)nent * 4u);
    L.off_eval = o;   o = align16(o + (uint32_t)nent * (uint32_t)es);
    L.off_x = o;      o = align16(o + (uint32_t)n * (uint32_t)es);
    L.bytes = o + 16u;                         // + the mbarrier
    return L;
}

__device__ __forceinline__ void cp_async_val_s(double *dst, const double *src) { cp_async_8(dst, src); }
__device__ __forceinline__ void cp_async_val_s(float *dst, const float *src) { cp_async_4(dst, src); }

template <typename T, bool UNIT>
__global__ void k_small(int n, int nlev, int nchunks, int64_t nent, const ChunkDesc *__restrict__ chunks,
                        const int32_t *__restrict__ lev_chunk, const int32_t *__restrict__ perm,
                        const T *__restrict__ invd, const int32_t *__restrict__ ecol, const T *__restrict__ eval,
                        const T *b, T *x) {
    extern __shared__ __align__(128) unsigned char sm[];
    const SmallLayout L = small_layout(n, nlev, nchunks, nent, (int)sizeof(T));
    const ChunkDesc *sc = reinterpret_cast<const ChunkDesc *>(sm + L.off_chunks);
    const int32_t *slc = reinterpret_cast<const int32_t *>(sm + L.off_levc);
    const int32_t *sp = reinterpret_cast<const int32_t *>(sm + L.off_perm);
    const T *sd = reinterpret_cast<const T *>(sm + L.off_invd);
    const int32_t *se = reinterpret_cast<const int32_t *>(sm + L.off_ecol);
    const T *sv = reinterpret_cast<const T *>(sm + L.off_eval);
    T *xs = reinterpret_cast<T *>(sm + L.off_x);
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + L.bytes - 16u);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // the layout by TMA bulk copies (16-byte rounded: the handle's arrays are
    // 256-byte aligned allocations), b by coalesced loads into x's slots
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t sz[6] = {align16((uint32_t)nchunks * 16u), align16((uint32_t)(nlev + 1) * 4u),
                                align16((uint32_t)n * 4u), align16((uint32_t)n * (uint32_t)sizeof(T)),
                                align16((uint32_t)nent * 4u), align16((uint32_t)nent * (uint32_t)sizeof(T))};
        const void *src[6] = {chunks, lev_chunk, perm, invd, ecol, eval};
        const uint32_t dst[6] = {L.off_chunks, L.off_levc, L.off_perm, L.off_invd, L.off_ecol, L.off_eval};
        uint32_t tot = 0;
        for (int i = 0; i < 6; ++i) tot += sz[i];
        mbar_arrive_expect_tx(bar, tot);
        for (int i = 0; i < 6; ++i)
            if (sz[i]) bulk_g2s(sm + dst[i], src[i], sz[i], bar);
    }
    // b: one cp.async per element, all in flight at once (a load/store loop of
    // a 32-thread CTA serialised ~n/32 DRAM round trips)
    for (int i = threadIdx.x; i < n; i += blockDim.x) cp_async_val_s(xs + i, b + i);
    cp_async_commit();
    cp_async_wait<0>();
    mbar_wait(bar, 0);
    __syncthreads();
    for (int l = 0; l < nlev; ++l) {
        for (int c = slc[l] + w; c < slc[l + 1]; c += nw) {
            const ChunkDesc cd = sc[c];
            const int width = chunk_width(cd.meta);
            if (!chunk_wpr(cd.meta)) {
                if (lane < chunk_nrows(cd.meta)) {
                    const int row = sp[cd.pos + lane];
                    T s = xs[row];
                    for (int k = 0; k < width; ++k) {
                        const int j = se[cd.eptr + (int64_t)k * 32 + lane];
                        if (j < 0) break;
                        s = fnma(sv[cd.eptr + (int64_t)k * 32 + lane], xs[j], s);
                    }
                    xs[row] = finish<T, UNIT>(s, sd[cd.pos + lane]);
                }
            } else {
                const int row = sp[cd.pos];
                T acc = T(0);
                for (int k = lane; k < width; k += 32) acc = __fma_rn(sv[cd.eptr + k], xs[se[cd.eptr + k]], acc);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (lane == 0) xs[row] = finish<T, UNIT>(xs[row] - acc, sd[cd.pos]);
            }
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = xs[i];
}

// per-position CSR of the referenced strict triangle (multi-RHS layout)
__global__ void k_mr_deg(int n, const int32_t *perm, const int32_t *dp, int32_t *deg) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) deg[p] = dp[perm[p]];
    if (p == n) deg[p] = 0;
}

template <typename T>
__global__ void k_mr_fill(int nchunks, const ChunkDesc *__restrict__ chunks, const int32_t *__restrict__ ecol,
                          const T *__restrict__ eval, const int32_t *__restrict__ mr_ptr, int32_t *__restrict__ mr_col,
                          T *__restrict__ mr_val) {
    const int lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < nchunks; c += nwarps) {
        const ChunkDesc cd = chunks[c];
        const int width = chunk_width(cd.meta);
        if (!chunk_wpr(cd.meta)) {
            if (lane < chunk_nrows(cd.meta)) {
                const int base = mr_ptr[cd.pos + lane];
                for (int k = 0; k < width; ++k) {
                    const int j = ecol[cd.eptr + (int64_t)k * 32 + lane];
                    if (j < 0) break;
                    mr_col[base + k] = j;
                    mr_val[base + k] = eval[cd.eptr + (int64_t)k * 32 + lane];
                }
            }
        } else {
            const int base = mr_ptr[cd.pos];
            for (int k = lane; k < width; k += 32) {
                mr_col[base + k] = ecol[cd.eptr + k];
                mr_val[base + k] = eval[cd.eptr + k];
            }
        }
    }
}

// Scratch buffer of the handle (copy of b for in-place value-as-flag solves).
// Grown on demand; the old buffer is released after `s` drains (stream-ordered).
sptrsv_status_t ensure_scratch(sptrsv_handle_t h, size_t bytes, cudaStream_t s) {
    if (h->scratch_bytes >= bytes) return SPTRSV_SUCCESS;
    if (h->d_scratch) {
        SPTRSV_CUDA(cudaFreeAsync(h->d_scratch, s));
        h->d_scratch = nullptr;
        h->scratch_bytes = 0;
    }
    SPTRSV_CUDA(cudaMallocAsync(&h->d_scratch, bytes, s));
    h->scratch_bytes = bytes;
    return SPTRSV_SUCCESS;
}

template <typename T>
sptrsv_status_t build_mr(sptrsv_handle_t h, cudaStream_t s) {
    ArenaStream as_{h->arena, s};     // the handle's allocations in this call: stream-ordered on s
    const int n = h->n;
    DevArena tmp(s);
    struct Guard {
        DevArena &a;
        ~Guard() { a.release_all(); }
    } guard{tmp};
    sptrsv_status_t st;
    int32_t *deg = nullptr;
    if ((st = tmp.alloc_n(&deg, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&h->d_mr_ptr, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    const int64_t nnz = std::max<int64_t>(h->info.nnz_used, 1);
    if ((st = h->arena.alloc_n(&h->d_mr_col, (size_t)nnz)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc(&h->d_mr_val, (size_t)nnz * sizeof(T))) != SPTRSV_SUCCESS) return st;
    k_mr_deg<<<(n + 1 + 255) / 256, 256, 0, s>>>(n, h->d_perm, h->d_dp, deg);
    if ((st = exclusive_scan_i32(deg, h->d_mr_ptr, (int64_t)n + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    const int grid = std::max(1, std::min((h->nchunks * 32 + 255) / 256, h->num_sms * 16));
    k_mr_fill<T><<<grid, 256, 0, s>>>(h->nchunks, h->d_chunks, h->d_ecol, (const T *)h->d_eval, h->d_mr_ptr,
                                      h->d_mr_col, (T *)h->d_mr_val);
    SPTRSV_CUDA(cudaGetLastError());
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    h->mr_built = true;
    h->info.device_bytes = h->arena.bytes;
    return SPTRSV_SUCCESS;
}

template <typename T, bool UNIT, int CPL>
sptrsv_status_t launch_level_mrhs(sptrsv_handle_t h, const T *b, T *x, int ncols, int64_t ld, cudaStream_t s) {
    const int grid = h->num_sms;
    const int nlev = h->info.nlev;
    void *args[] = {(void *)&h->d_ilev, (void *)&nlev, (void *)&h->d_perm, (void *)&h->d_invd, (void *)&h->d_mr_ptr,
                    (void *)&h->d_mr_col, (void *)&h->d_mr_val, (void *)&b, (void *)&x, (void *)&ncols, (void *)&ld,
                    (void *)&h->d_bar, (void *)&h->bar_base};
    SPTRSV_CUDA(cudaLaunchCooperativeKernel((const void *)k_level_mrhs<T, UNIT, CPL>, grid, kLevelThreads, args, 0, s));
    h->bar_base += (unsigned long long)(nlev > 0 ? nlev - 1 : 0) * grid;
    return SPTRSV_SUCCESS;
}

template <typename K>
int resident_grid(K kernel, int num_sms) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, 0);
    return std::max(1, per_sm) * num_sms;
}

constexpr int kVfMax = 16;       // widest column block of the value-as-flag multi-RHS kernel
constexpr int kLevelMax = 128;   // widest column block of the level-scheduled multi-RHS kernel

template <typename T, bool UNIT>
sptrsv_status_t launch(sptrsv_handle_t h, const T *b, T *x, int nrhs, cudaStream_t s) {
    if (h->nchunks == 0) return SPTRSV_SUCCESS;
    if (nrhs == 1 && h->algo == SPTRSV_ALGO_SMALL) {
        const SmallLayout L = small_layout(h->n, h->info.nlev, h->nchunks, h->nent, (int)sizeof(T));
        k_small<T, UNIT><<<1, h->small_threads, L.bytes, s>>>(h->n, h->info.nlev, h->nchunks, h->nent, h->d_chunks,
                                                              h->d_lev_chunk, h->d_perm, (const T *)h->d_invd,
                                                              h->d_ecol, (const T *)h->d_eval, b, x);
        SPTRSV_CUDA(cudaGetLastError());
        return SPTRSV_SUCCESS;
    }
    if (nrhs == 1 && h->algo == SPTRSV_ALGO_LEVEL) {
        const int grid = h->num_sms;
        const int nlev = h->info.nlev;
        void *args[] = {(void *)&h->d_chunks, (void *)&h->d_lev_chunk, (void *)&nlev, (void *)&h->d_perm,
                        (void *)&h->d_invd, (void *)&h->d_ecol, (void *)&h->d_eval, (void *)&b,
                        (void *)&x, (void *)&h->d_bar, (void *)&h->bar_base};
        SPTRSV_CUDA(cudaLaunchCooperativeKernel((const void *)k_level<T, UNIT>, grid, kLevelThreads1, args, 0, s));
        h->bar_base += (unsigned long long)(nlev > 0 ? nlev - 1 : 0) * grid;
        return SPTRSV_SUCCESS;
    }
    const bool level_req = h->algo == SPTRSV_ALGO_LEVEL || h->algo == SPTRSV_ALGO_LEVC;
    // multi-RHS with > 16 columns on factors with <= 4 dependencies per row:
    // the tile kernel (mrt.cu), which streams the matrix once per 64 columns
    // and keeps each CTA's previous level in shared memory (cfg5, 64 RHS:
    // 1.69 vs 1.79 ms for the level-scheduled kernel; 32 RHS 1.44-1.49 vs
    // 1.77 ms; at <= 16 columns the value-as-flag kernel is faster: 1.04 vs
    // 1.44 ms at 16, 0.59 vs 1.39 ms at 8 -- profiles/mrhs_r2.md).  Falls
    // through if its plan cannot be built.
    if (nrhs > kVfMax && !level_req && h->mrhs_path != 1 && mrt_eligible(h, b, x, nrhs)) {
        sptrsv_status_t st = mrt_solve(h, b, x, nrhs, s);
        if (st == SPTRSV_SUCCESS || h->mrt.built) return st;
    }
    // value-as-flag paths (SELF nrhs = 1, multi-RHS up to 16 columns): x is
    // the flag array, so an in-place solve keeps b aside first
    const bool vf = nrhs == 1 || (nrhs <= kVfMax && !level_req);
    if (vf && (const void *)b == (const void *)x) {
        const size_t bytes = (size_t)h->n * (size_t)nrhs * sizeof(T);
        sptrsv_status_t st = ensure_scratch(h, bytes, s);
        if (st != SPTRSV_SUCCESS) return st;
        SPTRSV_CUDA(cudaMemcpyAsync(h->d_scratch, b, bytes, cudaMemcpyDeviceToDevice, s));
        b = (const T *)h->d_scratch;
    }
    if (nrhs == 1) {
        if (h->self_grid == 0) {
            // one CTA (8 warps) per SM: 74-148 CTAs solve cfg2/3/4 equally fast,
            // 2 CTAs/SM are 10-35% slower -- spinning warps' polls load L2
            // (cfg3 3.92 -> 2.87 ms, cfg2 0.63 -> 0.54 ms, cfg4 34.0 -> 31.1 ms)
            h->self_grid = std::min(resident_grid(k_self<T, UNIT, 8>, h->num_sms), h->num_sms);
            // rows with many dependencies (mean >= 8) poll more values per lane:
            // half the SMs' worth of warps is enough and loads L2 less
            // (cfg3, 13 deps/row: 2.47 -> 2.14 ms; cfg4 26.8 -> 26.6 ms; cfg2,
            // 3 deps/row, prefers 148 CTAs: 0.54 vs 0.62 ms)
            const int64_t strict = h->info.nnz_used;          // referenced strict entries
            if (h->n > 0 && strict >= 8 * (int64_t)h->n) h->self_grid = std::max(1, h->self_grid / 2);
        }
        const int grid = h->self_grid;
        k_prefill<T><<<h->num_sms * 4, 512, 0, s>>>(x, (int64_t)h->n);
        k_self<T, UNIT, 8><<<grid, kThreads, 0, s>>>(h->d_chunks, h->nchunks, h->d_perm, (const T *)h->d_invd,
                                                     h->d_ecol, (const T *)h->d_eval, b, x, h->d_ctr,
                                                     (unsigned)(grid * (kThreads / 32)));
        SPTRSV_CUDA(cudaGetLastError());
        return SPTRSV_SUCCESS;
    }
    if (!h->mr_built) {          // first multi-RHS solve on the handle: builds the per-position CSR (syncs)
        sptrsv_status_t st = build_mr<T>(h, s);
        if (st != SPTRSV_SUCCESS) return st;
    }
    // value-as-flag multi-RHS for nrhs <= 16 (cfg5 ranks of 4 / 8 GPUs: 16 RHS
    // 1.02 vs 1.73 ms, 8 RHS 0.59 vs 1.72 ms for the level-scheduled kernel;
    // 32 RHS: 2.02 vs 1.74 ms), unless LEVEL / LEVC was asked for
    if (vf) {
        k_prefill<T><<<h->num_sms * 4, 512, 0, s>>>(x, (int64_t)h->n * nrhs);
        return launch_mrhs_vf<T, UNIT>(h, b, x, nrhs, nrhs, s);
    }
    // level-scheduled, in independent column blocks of <= 128 (each column's
    // arithmetic is the same whatever block it is in)
    for (int c0 = 0; c0 < nrhs; c0 += kLevelMax) {
        const int nc = std::min(kLevelMax, nrhs - c0);
        sptrsv_status_t st;
        if (nc <= 32) st = launch_level_mrhs<T, UNIT, 1>(h, b + c0, x + c0, nc, nrhs, s);
        else if (nc <= 64) st = launch_level_mrhs<T, UNIT, 2>(h, b + c0, x + c0, nc, nrhs, s);
        else st = launch_level_mrhs<T, UNIT, 4>(h, b + c0, x + c0, nc, nrhs, s);
        if (st != SPTRSV_SUCCESS) return st;
    }
    return SPTRSV_SUCCESS;
}

}  // namespace

sptrsv_status_t refresh_derived_values(sptrsv_handle_t h, cudaStream_t s) {
    sptrsv_status_t st;
    if (h->mr_built) {                        // per-position CSR: same positions, new values
        const int grid = std::max(1, std::min((h->nchunks * 32 + 255) / 256, h->num_sms * 16));
        if (h->dtype == SPTRSV_F64)
            k_mr_fill<double><<<grid, 256, 0, s>>>(h->nchunks, h->d_chunks, h->d_ecol, (const double *)h->d_eval,
                                                   h->d_mr_ptr, h->d_mr_col, (double *)h->d_mr_val);
        else
            k_mr_fill<float><<<grid, 256, 0, s>>>(h->nchunks, h->d_chunks, h->d_ecol, (const float *)h->d_eval,
                                                  h->d_mr_ptr, h->d_mr_col, (float *)h->d_mr_val);
        SPTRSV_CUDA(cudaGetLastError());
        if (h->csc_built && (st = csc_refresh_values(h, s)) != SPTRSV_SUCCESS) return st;
    }
    if (h->block.built || h->mrt.built) {
        DevArena tmp(s);
        struct Guard {
            DevArena &a;
            ~Guard() { a.release_all(); }
        } guard{tmp};
        int32_t *tri_ptr = nullptr, *tri_col = nullptr;
        void *tri_val = nullptr;
        if ((st = build_tri_csr(h, tmp, s, &tri_ptr, &tri_col, &tri_val)) != SPTRSV_SUCCESS) return st;
        if (h->block.built && (st = block_refresh_values(h, tri_ptr, tri_val, s)) != SPTRSV_SUCCESS) return st;
        if (h->mrt.built && (st = mrt_refresh_values(h, tri_ptr, tri_val, s)) != SPTRSV_SUCCESS) return st;
        SPTRSV_CUDA(cudaStreamSynchronize(s));      // before the temporaries are released
    }
    return SPTRSV_SUCCESS;
}

// SMALL plan: the layout fits in one CTA's shared memory; threads = 32 x the
// most chunks of one level (<= 32 warps).  NOT_SUPPORTED if it does not fit,
// or (AUTO) if some level needs more than one pass of 32 warps.
sptrsv_status_t small_plan(sptrsv_handle_t h, bool explicit_request) {
    if (h->small_threads > 0) return SPTRSV_SUCCESS;
    if (h->n == 0 || h->nchunks == 0) return SPTRSV_ERR_NOT_SUPPORTED;
    int max_smem = 0;
    SPTRSV_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
    const SmallLayout L = small_layout(h->n, h->info.nlev, h->nchunks, h->nent, (int)h->esize);
    if ((int64_t)L.bytes > max_smem - 1024 || h->nent > (1 << 26)) return SPTRSV_ERR_NOT_SUPPORTED;
    std::vector<int32_t> lc((size_t)h->info.nlev + 1);
    SPTRSV_CUDA(cudaMemcpy(lc.data(), h->d_lev_chunk, sizeof(int32_t) * lc.size(), cudaMemcpyDeviceToHost));
    int mc = 1;
    for (int l = 0; l < h->info.nlev; ++l) mc = std::max(mc, lc[l + 1] - lc[l]);
    if (!explicit_request && mc > 32) return SPTRSV_ERR_NOT_SUPPORTED;   // AUTO: every level in one pass of <= 32 warps
    const int threads = 32 * std::min(mc, 32);
    void *k = h->dtype == SPTRSV_F64 ? (h->diag == SPTRSV_UNIT ? (void *)k_small<double, true> : (void *)k_small<double, false>)
                                     : (h->diag == SPTRSV_UNIT ? (void *)k_small<float, true> : (void *)k_small<float, false>);
    SPTRSV_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.bytes));
    h->small_threads = threads;
    return SPTRSV_SUCCESS;
}

sptrsv_status_t build_mr_any(sptrsv_handle_t h, cudaStream_t s) {
    return h->dtype == SPTRSV_F64 ? build_mr<double>(h, s) : build_mr<float>(h, s);
}

sptrsv_status_t solve_impl(sptrsv_handle_t h, const void *b, void *x, int32_t nrhs, cudaStream_t s) {
    if (nrhs == 1 && (h->algo == SPTRSV_ALGO_SLFC || h->algo == SPTRSV_ALGO_LEVC)) return column_solve(h, b, x, s);
    if (nrhs == 1 && h->algo == SPTRSV_ALGO_BLOCK) return block_solve(h, b, x, s);
    if (h->dtype == SPTRSV_F64) {
        return h->diag == SPTRSV_UNIT ? launch<double, true>(h, (const double *)b, (double *)x, nrhs, s)
                                      : launch<double, false>(h, (const double *)b, (double *)x, nrhs, s);
    }
    return h->diag == SPTRSV_UNIT ? launch<float, true>(h, (const float *)b, (float *)x, nrhs, s)
                                  : launch<float, false>(h, (const float *)b, (float *)x, nrhs, s);
}

}  // namespace sptrsv

extern "C" int sptrsv_dbg_self_trace(void *dev_buf) {
    unsigned long long *p = (unsigned long long *)dev_buf;
    return cudaMemcpyToSymbol(sptrsv::g_tpub, &p, sizeof(p)) == cudaSuccess ? 0 : 5;
}
