// tile.cu -- SPTRSV_ALGO_TILE: CTA tiles, level-synchronous inside a CTA,
// point-to-point level counters between CTAs.
//
// The rows are partitioned over co-resident CTAs with the BLOCK partition
// (block.cu: detected 3-D/2-D grids cut into (x, y) tiles of z-columns), and
// inside a CTA they are solved level by level (LEVR) with
// ONE __syncthreads per level: the CTA's own x lives in shared memory (every
// row of the CTA has a slot), so a dependency inside the CTA is one LDS after
// the barrier.  Between CTAs there is no grid barrier: CTA c publishes
// done[c] = "all my rows of level < l are solved" (release) and a consumer
// waits (acquire, cached) only for the CTAs that produce its dependencies
// (every dependency has a lower level).
//
// Everything a level needs is fetched ahead, so the per-level critical path is
// barrier -> LDS -> FMA chain -> STS:
//   * the level's records (row, dependency codes, 1/d, values; 48 B per row
//     for fp64) by TMA bulk copies into a ring of kRL levels (mbarriers);
//   * b[row] and the x of every dependency owned by ANOTHER CTA by cp.async
//     into per-thread rings, kTD levels ahead -- the producers are waited for
//     up to the level kTD ahead, so the CTA dependency graph must be acyclic
//     (checked at build time; true for the 7-point / 5-point grid tiles).
// Codes: >= 0 local x slot (position - first position of the CTA; the slot
// after the last holds 0 for padding), < 0: -(1 + j), x[j] of another CTA.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "internal.h"

namespace sptrsv {
namespace {

constexpr int kTW = 3;        // dependencies per row (7-point / 5-point lower or upper)
constexpr int kRL = 8;        // record ring (levels)
constexpr int kTD = 4;        // lookahead of b / foreign x (levels)
static_assert(kTD < kRL, "record ring shorter than the fetch lookahead");

// b: read-only during the solve (L1 allowed)
__device__ __forceinline__ void cpa_val(double *dst, const double *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_val(float *dst, const float *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// x of another CTA, written during this solve: through L2 only (.cg needs 16
// bytes: the aligned 16-byte group holding the value)
__device__ __forceinline__ void cpa_16_cg(void *dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

__global__ void k_pos_of_row(int n, const int32_t *tm_perm, int32_t *pos) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) pos[tm_perm[p]] = p;
}

// per position: int4 {row, code0, code1, code2}; T[4] {1/d, v0, v1, v2}
template <typename T>
__global__ void k_trec_fill(int n, int nlev, int wpc, const int32_t *__restrict__ tm_perm,
                            const int32_t *__restrict__ tm_ptr, const int32_t *__restrict__ tm_col,
                            const T *__restrict__ tm_val, const T *__restrict__ tm_invd,
                            const int32_t *__restrict__ unit, const int32_t *__restrict__ off,
                            const int32_t *__restrict__ pos_of_row, int4 *__restrict__ ri, T *__restrict__ rv,
                            unsigned *bad) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int row = tm_perm[p];
    const int c = unit[row] / wpc;
    const int p0 = off[(size_t)c * nlev], p1 = off[(size_t)(c + 1) * nlev];
    int code[kTW];
    T v[kTW];
    const int a = tm_ptr[p], e = tm_ptr[p + 1];
    if (e - a > kTW) atomicAdd(bad, 1u);
    for (int k = 0; k < kTW; ++k) {
        if (a + k < e) {
            const int j = tm_col[a + k];
            code[k] = (unit[j] / wpc == c) ? pos_of_row[j] - p0 : -1 - j;
            v[k] = tm_val[a + k];
        } else {
            code[k] = p1 - p0;       // the zero slot
            v[k] = T(0);
        }
    }
    ri[p] = make_int4(row, code[0], code[1], code[2]);
    rv[4 * (size_t)p] = tm_invd[p];
    for (int k = 0; k < kTW; ++k) rv[4 * (size_t)p + 1 + k] = v[k];
}

struct TileArgs {
    const int4 *clist;        // per CTA non-empty levels: {level, first position, rows, 0}
    const int32_t *cptr;      // [K+1] into clist
    const int32_t *cpos;      // [K+1] first position of every CTA
    const int32_t *dptr, *dl; // producer CTAs
    unsigned long long *done;
    unsigned long long base;
    const int4 *ri;
    const void *rv;
    const void *b;
    void *x;
    int nlev, maxr;
};

template <typename T, bool UNIT>
__global__ void __launch_bounds__(1024, 1) k_tile(const TileArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ uint64_t bars[kRL];
    constexpr int ES = (int)sizeof(T);
    const int c = blockIdx.x, t = threadIdx.x, nt = blockDim.x, MR = a.maxr;
    const int P0 = a.cpos[c], nloc = a.cpos[c + 1] - P0;
    const int4 *cl = a.clist + a.cptr[c];
    const int nk = a.cptr[c + 1] - a.cptr[c];
    // shared memory: record ring [kRL][MR] int4 | [kRL][MR][4] T | b ring [kTD][nt] T |
    //                foreign-x ring [kTD][kTW][nt] 16-byte groups | x slots [nloc + 1] T
    int4 *rring = reinterpret_cast<int4 *>(smem_raw);
    T *vring = reinterpret_cast<T *>(rring + kRL * MR);
    T *bring = vring + (size_t)kRL * MR * 4;
    constexpr int G = 16 / ES;                  // values per 16-byte group
    T *fring = bring + kTD * nt;
    T *xs = fring + (size_t)kTD * kTW * nt * G;
    const T *b = static_cast<const T *>(a.b);
    T *x = static_cast<T *>(a.x);
    const T *grv = static_cast<const T *>(a.rv);

    for (int i = t; i <= nloc; i += nt) xs[i] = T(0);
    if (t == 0) {
        for (int i = 0; i < kRL; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
        st_release_u64(&a.done[c], a.base + (unsigned long long)(nk > 0 ? cl[0].x : a.nlev));
    }
    __syncthreads();
    if (nk == 0) return;
    const int d0 = a.dptr[c], nd = a.dptr[c + 1] - d0;
    unsigned long long seen = 0;              // cached producer counter (threads t < nd)
    const unsigned long long *pf = t < nd ? &a.done[a.dl[d0 + t]] : nullptr;

    auto issue_rec = [&](int k) {            // thread 0: records of level index k -> slot k % kRL
        const int4 L = cl[k];
        const int slot = k % kRL;
        const uint32_t bi = (uint32_t)L.z * 16u, bv = (uint32_t)L.z * 4u * ES;
        mbar_arrive_expect_tx(&bars[slot], bi + bv);
        bulk_g2s(rring + slot * MR, a.ri + L.y, bi, &bars[slot]);
        bulk_g2s(vring + (size_t)slot * MR * 4, grv + 4 * (size_t)L.y, bv, &bars[slot]);
    };
    auto rec_wait = [&](int k) { mbar_wait(&bars[k % kRL], (uint32_t)((k / kRL) & 1)); };
    auto issue_fetch = [&](int k) {          // b / foreign x of level index k (records landed)
        const int4 L = cl[k];
        const int fs = k % kTD;
        if (t < L.z) {
            const int4 r = rring[(k % kRL) * MR + t];
            cpa_val(&bring[fs * nt + t], b + r.x);
            const int cd[kTW] = {r.y, r.z, r.w};
#pragma unroll
            for (int q = 0; q < kTW; ++q)
                if (cd[q] < 0) cpa_16_cg(&fring[((fs * kTW + q) * nt + t) * G], x + ((-1 - cd[q]) & ~(G - 1)));
        }
    };
    auto wait_producers = [&](int lv) {      // producers done with every level < lv (acquire, cached)
        const unsigned long long target = a.base + (unsigned long long)lv;
        if (t < nd && seen < target) {
            unsigned long long v = ld_acquire_u64(pf);
            while (v < target) v = ld_acquire_u64(pf);
            seen = v;
        }
    };

    if (t == 0)
        for (int k = 0; k < min(nk, kRL); ++k) issue_rec(k);
    for (int k = 0; k < kTD; ++k) {
        if (k < nk) {
            wait_producers(cl[k].x);
            rec_wait(k);
            __syncthreads();
            issue_fetch(k);
        }
        cp_async_commit();
    }
#pragma unroll 1
    for (int k = 0; k < nk; ++k) {
        const int kf = k + kTD;
        if (kf < nk) {
            wait_producers(cl[kf].x);
            rec_wait(kf);
        }
        rec_wait(k);
        cp_async_wait<kTD - 1>();
        __syncthreads();                        // x of levels < cl[k].x visible; producers checked
        const int4 L = cl[k];
        if (t == 0) {
            st_release_u64(&a.done[c], a.base + (unsigned long long)L.x);
            if (k >= 1 && k - 1 + kRL < nk) issue_rec(k - 1 + kRL);    // every thread is past level k-1
        }
        const int rs = k % kRL, fs = k % kTD;
        if (t < L.z) {
            const int4 r = rring[rs * MR + t];
            const T *vp = vring + ((size_t)rs * MR + t) * 4;
            T acc = bring[fs * nt + t];
            const int cd[kTW] = {r.y, r.z, r.w};
#pragma unroll
            for (int q = 0; q < kTW; ++q) {
                const T xv = cd[q] >= 0 ? xs[cd[q]] : fring[((fs * kTW + q) * nt + t) * G + ((-1 - cd[q]) & (G - 1))];
                acc = fnma(vp[1 + q], xv, acc);
            }
            const T res = UNIT ? acc : acc * vp[0];
            xs[L.y + t - P0] = res;
            __stcg(x + r.x, res);
        }
        if (kf < nk) issue_fetch(kf);           // into slot fs, after this level's reads of it
        cp_async_commit();
    }
    cp_async_wait<0>();
    __syncthreads();
    if (t == 0) st_release_u64(&a.done[c], a.base + (unsigned long long)a.nlev);
}

}  // namespace

// Built on top of the BLOCK partition and the CTA-tile multi-RHS plan
// (block.cu: tile_mrhs_build): per position the fixed-width records, per CTA
// its non-empty levels, and the acyclicity check of the producer graph.
sptrsv_status_t tile_build(sptrsv_handle_t h, cudaStream_t s) {
    BlockPlan &B = h->block;
    if (!B.tm_built) return SPTRSV_ERR_NOT_SUPPORTED;
    if (h->info.max_row_deps > kTW) return SPTRSV_ERR_NOT_SUPPORTED;
    const int n = h->n, nlev = h->info.nlev, K = B.tm_K;
    const size_t es = h->esize;
    DevArena tmp;
    struct Guard {
        DevArena &a;
        ~Guard() { a.release_all(); }
    } guard{tmp};
    sptrsv_status_t st;
    // producer graph acyclic (the kTD-level lookahead waits ahead of the CTA's own level)
    std::vector<int32_t> dptr(K + 1), dl;
    SPTRSV_CUDA(cudaMemcpyAsync(dptr.data(), B.d_tm_dptr, sizeof(int32_t) * (K + 1), cudaMemcpyDeviceToHost, s));
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    dl.resize(std::max(dptr[K], 1));
    SPTRSV_CUDA(cudaMemcpyAsync(dl.data(), B.d_tm_dl, sizeof(int32_t) * dl.size(), cudaMemcpyDeviceToHost, s));
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    {
        std::vector<int> indeg(K, 0), order;
        std::vector<std::vector<int>> out(K);
        for (int c = 0; c < K; ++c)
            for (int q = dptr[c]; q < dptr[c + 1]; ++q) {
                out[dl[q]].push_back(c);
                ++indeg[c];
            }
        for (int c = 0; c < K; ++c)
            if (indeg[c] == 0) order.push_back(c);
        for (size_t i = 0; i < order.size(); ++i)
            for (int d : out[order[i]])
                if (--indeg[d] == 0) order.push_back(d);
        if ((int)order.size() != K) return SPTRSV_ERR_NOT_SUPPORTED;
    }
    // per-CTA level lists
    std::vector<int32_t> off((size_t)K * nlev + 1);
    SPTRSV_CUDA(cudaMemcpyAsync(off.data(), B.d_tm_off, sizeof(int32_t) * off.size(), cudaMemcpyDeviceToHost, s));
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    std::vector<int4> clist;
    std::vector<int32_t> cptr(K + 1, 0), cpos(K + 1, 0);
    int maxr = 1, maxloc = 0;
    for (int c = 0; c < K; ++c) {
        cpos[c] = off[(size_t)c * nlev];
        for (int l = 0; l < nlev; ++l) {
            const int q0 = off[(size_t)c * nlev + l], q1 = off[(size_t)c * nlev + l + 1];
            if (q1 > q0) {
                clist.push_back(make_int4(l, q0, q1 - q0, 0));
                maxr = std::max(maxr, q1 - q0);
            }
        }
        cptr[c + 1] = (int32_t)clist.size();
    }
    cpos[K] = n;
    for (int c = 0; c < K; ++c) maxloc = std::max(maxloc, cpos[c + 1] - cpos[c]);
    if (clist.empty()) clist.push_back(make_int4(0, 0, 0, 0));
    const int nt = std::min(1024, (maxr + 31) / 32 * 32);
    if (maxr > nt) return SPTRSV_ERR_NOT_SUPPORTED;
    const size_t smem = (size_t)kRL * maxr * 16 + (size_t)kRL * maxr * 4 * es + (size_t)kTD * nt * es +
                        (size_t)kTD * kTW * nt * 16 + ((size_t)maxloc + 1) * es;
    int max_smem = 0;
    SPTRSV_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
    if (smem + 1024 > (size_t)max_smem) return SPTRSV_ERR_NOT_SUPPORTED;

    TilePlan &P = h->tile;
    if ((st = h->arena.alloc_n(&P.d_clist, clist.size())) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&P.d_cptr, (size_t)K + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&P.d_cpos, (size_t)K + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&P.d_ri, (size_t)std::max(n, 1))) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc(&P.d_rv, (size_t)std::max(n, 1) * 4 * es)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&P.d_done, (size_t)K)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemcpyAsync(P.d_clist, clist.data(), sizeof(int4) * clist.size(), cudaMemcpyHostToDevice, s));
    SPTRSV_CUDA(cudaMemcpyAsync(P.d_cptr, cptr.data(), sizeof(int32_t) * (K + 1), cudaMemcpyHostToDevice, s));
    SPTRSV_CUDA(cudaMemcpyAsync(P.d_cpos, cpos.data(), sizeof(int32_t) * (K + 1), cudaMemcpyHostToDevice, s));
    SPTRSV_CUDA(cudaMemsetAsync(P.d_done, 0, sizeof(unsigned long long) * K, s));
    int32_t *pos = nullptr;
    unsigned *bad = nullptr;
    if ((st = tmp.alloc_n(&pos, (size_t)std::max(n, 1))) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&bad, 1)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned), s));
    const int eg = (n + 255) / 256;
    k_pos_of_row<<<eg, 256, 0, s>>>(n, B.d_tm_perm, pos);
    if (h->dtype == SPTRSV_F64)
        k_trec_fill<double><<<eg, 256, 0, s>>>(n, nlev, B.wpc, B.d_tm_perm, B.d_tm_ptr, B.d_tm_col,
                                               (const double *)B.d_tm_val, (const double *)B.d_tm_invd, B.d_unit,
                                               B.d_tm_off, pos, P.d_ri, (double *)P.d_rv, bad);
    else
        k_trec_fill<float><<<eg, 256, 0, s>>>(n, nlev, B.wpc, B.d_tm_perm, B.d_tm_ptr, B.d_tm_col,
                                              (const float *)B.d_tm_val, (const float *)B.d_tm_invd, B.d_unit,
                                              B.d_tm_off, pos, P.d_ri, (float *)P.d_rv, bad);
    SPTRSV_CUDA(cudaGetLastError());
    unsigned hb = 0;
    SPTRSV_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    if (hb) return SPTRSV_ERR_NOT_SUPPORTED;
    void *kn = h->dtype == SPTRSV_F64
                   ? (h->diag == SPTRSV_UNIT ? (void *)k_tile<double, true> : (void *)k_tile<double, false>)
                   : (h->diag == SPTRSV_UNIT ? (void *)k_tile<float, true> : (void *)k_tile<float, false>);
    SPTRSV_CUDA(cudaFuncSetAttribute(kn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    SPTRSV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kn, nt, smem));
    if (per_sm * h->num_sms < K) return SPTRSV_ERR_NOT_SUPPORTED;
    P.kernel = kn;
    P.smem = smem;
    P.threads = nt;
    P.maxr = maxr;
    P.K = K;
    P.base = 0;
    P.built = true;
    h->info.device_bytes = h->arena.bytes;
    return SPTRSV_SUCCESS;
}

sptrsv_status_t tile_solve(sptrsv_handle_t h, const void *b, void *x, cudaStream_t s) {
    TilePlan &P = h->tile;
    BlockPlan &B = h->block;
    if (!P.built) return SPTRSV_ERR_NOT_SUPPORTED;
    // (in place is safe: a row's b is fetched, and has landed, kTD levels before
    // the same CTA writes that row's x)
    TileArgs a;
    a.clist = P.d_clist;
    a.cptr = P.d_cptr;
    a.cpos = P.d_cpos;
    a.dptr = B.d_tm_dptr;
    a.dl = B.d_tm_dl;
    a.done = P.d_done;
    a.base = P.base;
    a.ri = P.d_ri;
    a.rv = P.d_rv;
    a.b = b;
    a.x = x;
    a.nlev = h->info.nlev;
    a.maxr = P.maxr;
    void *args[] = {(void *)&a};
    SPTRSV_CUDA(cudaLaunchCooperativeKernel(P.kernel, P.K, P.threads, args, P.smem, s));
    P.base += (unsigned long long)h->info.nlev + 1;
    return SPTRSV_SUCCESS;
}

}  // namespace sptrsv
