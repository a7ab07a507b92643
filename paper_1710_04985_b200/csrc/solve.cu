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

#include "internal.h"

namespace sptrsv {
namespace {

constexpr int kThreads = 256;

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
                                          const T *__restrict__ eval, const T *b, T *x) {
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
        bool pend = false;
#pragma unroll
        for (int k = 0; k < kTprMax; ++k) pend |= (cols[k] >= 0) && Sentinel<T>::is(xv[k]);
        while (pend) {
            pend = false;
            __nanosleep(20);
#pragma unroll
            for (int k = 0; k < kTprMax; ++k) {
                if (cols[k] >= 0 && Sentinel<T>::is(xv[k])) {
                    xv[k] = ld_relaxed_val(x + cols[k]);
                    pend |= Sentinel<T>::is(xv[k]);
                }
            }
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
template <typename T, bool UNIT, bool WAIT>
__device__ __forceinline__ void wpr_row(const ChunkDesc &cd, int lane, const int32_t *__restrict__ perm,
                                        const T *__restrict__ invd, const int32_t *__restrict__ ecol,
                                        const T *__restrict__ eval, const T *b, T *x) {
    const int width = chunk_width(cd.meta);
    const int row = perm[cd.pos];
    const int32_t *ec = ecol + cd.eptr;
    const T *ev = eval + cd.eptr;
    T acc = T(0);
    for (int k = lane; k < width; k += 32) {
        const int c = ec[k];
        T v;
        if (WAIT) {
            v = ld_relaxed_val(x + c);
            while (Sentinel<T>::is(v)) v = ld_relaxed_val(x + c);
        } else {
            v = ld_cg(x + c);
        }
        acc = __fma_rn(ld_stream(ev + k), v, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
        const T r = finish<T, UNIT>(ld_cg(b + row) - acc, invd[cd.pos]);
        if (WAIT) st_relaxed_val(x + row, Sentinel<T>::scrub(r));
        else x[row] = r;
    }
}

// ---------------------------------------------------------------- SELF
// x must hold Sentinel<T> in every row on entry (k_prefill).
template <typename T, bool UNIT>
__global__ void __launch_bounds__(kThreads) k_self(const ChunkDesc *__restrict__ chunks, int nchunks,
                                                   const int32_t *__restrict__ perm, const T *__restrict__ invd,
                                                   const int32_t *__restrict__ ecol, const T *__restrict__ eval,
                                                   const T *b, T *x, unsigned *ctr, unsigned nwarps_total) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(&ctr[0], 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if ((int)t >= nchunks) break;
        const ChunkDesc cd = chunks[t];
        if (!chunk_wpr(cd.meta))
            tpr_chunk<T, UNIT, true>(cd, lane, perm, invd, ecol, eval, b, x);
        else
            wpr_row<T, UNIT, true>(cd, lane, perm, invd, ecol, eval, b, x);
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
__device__ __forceinline__ void grid_barrier(unsigned long long *bar, unsigned long long target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        fence_acq_rel_gpu();
        atomicAdd(bar, 1ull);
        while (ld_relaxed_u64(bar) < target) {
        }
        fence_acq_rel_gpu();
    }
    __syncthreads();
}

template <typename T, bool UNIT>
__global__ void __launch_bounds__(kThreads) k_level(const ChunkDesc *__restrict__ chunks,
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
// Warp per chunk; lane r polls the flags of chunk row r, then the warp walks
// the rows with lanes over RHS columns.  Per (row, column) the arithmetic is
// the TPR sequence, so each column equals the nrhs == 1 TPR result bitwise
// and does not depend on nrhs (SURVEY §8e partition invariant).
template <typename T, bool UNIT>
__global__ void __launch_bounds__(kThreads) k_mrhs(const ChunkDesc *__restrict__ chunks, int nchunks,
                                                   const int32_t *__restrict__ perm, const T *__restrict__ invd,
                                                   const int32_t *__restrict__ ecol, const T *__restrict__ eval,
                                                   const T *b, T *x, int nrhs, int *flags, int epoch,
                                                   unsigned *ctr, unsigned nwarps_total) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(&ctr[0], 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        if ((int)t >= nchunks) break;
        const ChunkDesc cd = chunks[t];
        const int width = chunk_width(cd.meta);
        if (!chunk_wpr(cd.meta)) {
            const int nr = chunk_nrows(cd.meta);
            const bool act = lane < nr;
            int myrow = act ? perm[cd.pos + lane] : 0;
            T mydi = act ? invd[cd.pos + lane] : T(0);
            int cols[kTprMax];
            T vals[kTprMax];
#pragma unroll
            for (int k = 0; k < kTprMax; ++k) {
                cols[k] = -1;
                vals[k] = T(0);
                if (k < width) {
                    cols[k] = ld_stream(ecol + cd.eptr + k * 32 + lane);
                    vals[k] = ld_stream(eval + cd.eptr + k * 32 + lane);
                }
            }
            wait_flags<kTprMax>(flags, cols, width, epoch);
            fence_acq_rel_gpu();
            __syncwarp();
            for (int r = 0; r < nr; ++r) {
                const int row = __shfl_sync(0xffffffffu, myrow, r);
                const T di = __shfl_sync(0xffffffffu, mydi, r);
                int rc[kTprMax];
                T rv[kTprMax];
#pragma unroll
                for (int k = 0; k < kTprMax; ++k) {
                    rc[k] = __shfl_sync(0xffffffffu, cols[k], r);
                    rv[k] = __shfl_sync(0xffffffffu, vals[k], r);
                }
                for (int c = lane; c < nrhs; c += 32) {
                    T s = ld_cg(b + (int64_t)row * nrhs + c);
#pragma unroll
                    for (int k = 0; k < kTprMax; ++k) {
                        if (k < width && rc[k] >= 0) s = fnma(rv[k], ld_cg(x + (int64_t)rc[k] * nrhs + c), s);
                    }
                    x[(int64_t)row * nrhs + c] = finish<T, UNIT>(s, di);
                }
            }
            __syncwarp();
            if (act) st_release(&flags[myrow], epoch);
        } else {
            const int row = perm[cd.pos];
            const int32_t *ec = ecol + cd.eptr;
            const T *ev = eval + cd.eptr;
            for (int k = lane; k < width; k += 32) {
                const int c = ec[k];
                int spins = 0;
                while (ld_relaxed(&flags[c]) != epoch) {
                    if (++spins > 8) __nanosleep(32);
                }
            }
            fence_acq_rel_gpu();
            __syncwarp();
            const T di = invd[cd.pos];
            for (int c = lane; c < nrhs; c += 32) {
                T s = ld_cg(b + (int64_t)row * nrhs + c);
                for (int k = 0; k < width; ++k) s = fnma(ev[k], ld_cg(x + (int64_t)ec[k] * nrhs + c), s);
                x[(int64_t)row * nrhs + c] = finish<T, UNIT>(s, di);
            }
            __syncwarp();
            if (lane == 0) st_release(&flags[row], epoch);
        }
    }
    if (lane == 0) {
        unsigned e = atomicAdd(&ctr[1], 1u);
        if (e == nwarps_total - 1) {
            ctr[0] = 0;
            ctr[1] = 0;
        }
    }
}

sptrsv_status_t ensure_scratch(sptrsv_handle_t h, size_t bytes) {
    if (h->scratch_bytes >= bytes) return SPTRSV_SUCCESS;
    if (h->d_scratch) {
        SPTRSV_CUDA(cudaDeviceSynchronize());
        cudaFree(h->d_scratch);
        h->d_scratch = nullptr;
        h->scratch_bytes = 0;
    }
    SPTRSV_CUDA(cudaMalloc(&h->d_scratch, bytes));
    h->scratch_bytes = bytes;
    return SPTRSV_SUCCESS;
}

template <typename K>
int resident_grid(K kernel, int num_sms) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, 0);
    return std::max(1, per_sm) * num_sms;
}

template <typename T, bool UNIT>
sptrsv_status_t launch(sptrsv_handle_t h, const T *b, T *x, int nrhs, cudaStream_t s) {
    if (h->nchunks == 0) return SPTRSV_SUCCESS;
    if (nrhs == 1 && h->algo == SPTRSV_ALGO_LEVEL) {
        if (h->level_grid == 0) {
            int per_sm = 0;
            SPTRSV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_level<T, UNIT>, kThreads, 0));
            h->level_grid = std::max(1, per_sm) * h->num_sms;
        }
        const int grid = h->level_grid;
        const int nlev = h->info.nlev;
        void *args[] = {(void *)&h->d_chunks, (void *)&h->d_lev_chunk, (void *)&nlev, (void *)&h->d_perm,
                        (void *)&h->d_invd, (void *)&h->d_ecol, (void *)&h->d_eval, (void *)&b,
                        (void *)&x, (void *)&h->d_bar, (void *)&h->bar_base};
        SPTRSV_CUDA(cudaLaunchCooperativeKernel((const void *)k_level<T, UNIT>, grid, kThreads, args, 0, s));
        h->bar_base += (unsigned long long)(nlev > 0 ? nlev - 1 : 0) * grid;
        return SPTRSV_SUCCESS;
    }
    if (++h->epoch == INT32_MAX) {   // flag wrap: restart the epoch sequence
        SPTRSV_CUDA(cudaMemsetAsync(h->d_flags, 0, sizeof(int32_t) * (size_t)h->n, s));
        h->epoch = 1;
    }
    if (nrhs == 1) {
        if (h->self_grid == 0) h->self_grid = resident_grid(k_self<T, UNIT>, h->num_sms);
        const int grid = h->self_grid;
        if ((const void *)b == (const void *)x) {   // in place: keep b aside, x becomes the flag array
            sptrsv_status_t st = ensure_scratch(h, (size_t)h->n * sizeof(T));
            if (st != SPTRSV_SUCCESS) return st;
            SPTRSV_CUDA(cudaMemcpyAsync(h->d_scratch, b, (size_t)h->n * sizeof(T), cudaMemcpyDeviceToDevice, s));
            b = (const T *)h->d_scratch;
        }
        k_prefill<T><<<h->num_sms * 4, 512, 0, s>>>(x, (int64_t)h->n);
        k_self<T, UNIT><<<grid, kThreads, 0, s>>>(h->d_chunks, h->nchunks, h->d_perm, (const T *)h->d_invd,
                                                  h->d_ecol, (const T *)h->d_eval, b, x, h->d_ctr,
                                                  (unsigned)(grid * (kThreads / 32)));
    } else {
        if (h->mrhs_grid == 0) h->mrhs_grid = resident_grid(k_mrhs<T, UNIT>, h->num_sms);
        const int grid = h->mrhs_grid;
        k_mrhs<T, UNIT><<<grid, kThreads, 0, s>>>(h->d_chunks, h->nchunks, h->d_perm, (const T *)h->d_invd,
                                                  h->d_ecol, (const T *)h->d_eval, b, x, nrhs, h->d_flags,
                                                  h->epoch, h->d_ctr, (unsigned)(grid * (kThreads / 32)));
    }
    SPTRSV_CUDA(cudaGetLastError());
    return SPTRSV_SUCCESS;
}

}  // namespace

sptrsv_status_t solve_impl(sptrsv_handle_t h, const void *b, void *x, int32_t nrhs, cudaStream_t s) {
    if (nrhs == 1 && h->algo == SPTRSV_ALGO_BLOCK) return block_solve(h, b, x, s);
    if (h->dtype == SPTRSV_F64) {
        return h->diag == SPTRSV_UNIT ? launch<double, true>(h, (const double *)b, (double *)x, nrhs, s)
                                      : launch<double, false>(h, (const double *)b, (double *)x, nrhs, s);
    }
    return h->diag == SPTRSV_UNIT ? launch<float, true>(h, (const float *)b, (float *)x, nrhs, s)
                                  : launch<float, false>(h, (const float *)b, (float *)x, nrhs, s);
}

}  // namespace sptrsv
