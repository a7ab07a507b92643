// api.cu -- the C ABI of include/sptrsv.h: argument checks, handle lifecycle,
// host staging.  All arithmetic runs in analyze.cu / solve.cu / block.cu.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <new>

#include "internal.h"

namespace sptrsv {

static thread_local char g_last_cuda[256] = "";

sptrsv_status_t cuda_fail(cudaError_t e, const char *where) {
    snprintf(g_last_cuda, sizeof(g_last_cuda), "%s: %s", where, cudaGetErrorString(e));
    if (e == cudaErrorMemoryAllocation) return SPTRSV_ERR_ALLOC;
    return SPTRSV_ERR_CUDA;
}

sptrsv_status_t DevArena::alloc(void **p, size_t nbytes) {
    *p = nullptr;
    if (nbytes == 0) nbytes = 16;
    nbytes = (nbytes + 255) & ~(size_t)255;          // 256-byte aligned sub-allocations
    cudaError_t e = cudaMallocAsync(p, nbytes, stream);
    if (e != cudaSuccess) {
        *p = nullptr;
        cudaGetLastError();
        return cuda_fail(e, "cudaMallocAsync");
    }
    ptrs.push_back(*p);
    bytes += (int64_t)nbytes;
    return SPTRSV_SUCCESS;
}

void DevArena::release_all() {
    for (void *p : ptrs) cudaFreeAsync(p, stream);
    ptrs.clear();
    bytes = 0;
}

// The default memory pool of the device keeps up to 16 GiB of freed memory
// for reuse (stream-ordered allocations of later handles and temporaries
// then cost no driver round trip; beyond that it returns memory at the next
// synchronisation).
void keep_pool_memory(int dev) {
    static bool done[64] = {};
    if (dev < 0 || dev >= 64 || done[dev]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = 16ull << 30;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    done[dev] = true;
}

}  // namespace sptrsv

using namespace sptrsv;

static bool valid_enum(int v) { return v == 0 || v == 1; }

extern "C" sptrsv_status_t sptrsv_analyze(int32_t n, const int32_t *rowptr, const int32_t *colidx,
                                          const void *vals, sptrsv_uplo_t uplo, sptrsv_diag_t diag,
                                          sptrsv_dtype_t dtype, sptrsv_stream_t stream,
                                          sptrsv_handle_t *out) {
    if (!out) return SPTRSV_ERR_INVALID_VALUE;
    *out = nullptr;
    if (n < 0 || !valid_enum(uplo) || !valid_enum(diag) || !valid_enum(dtype)) return SPTRSV_ERR_INVALID_VALUE;
    if (n > 0 && (!rowptr || !colidx || (!vals && diag == SPTRSV_NON_UNIT))) return SPTRSV_ERR_INVALID_VALUE;

    auto t0 = std::chrono::steady_clock::now();
    int dev = 0;
    SPTRSV_CUDA(cudaGetDevice(&dev));
    cudaDeviceProp prop;
    SPTRSV_CUDA(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10) return SPTRSV_ERR_NOT_SUPPORTED;

    sptrsv_handle_t h = new (std::nothrow) sptrsv_handle_s();
    if (!h) return SPTRSV_ERR_ALLOC;
    h->n = n;
    h->uplo = uplo;
    h->diag = diag;
    h->dtype = dtype;
    h->device = dev;
    h->num_sms = prop.multiProcessorCount;
    h->esize = dtype == SPTRSV_F64 ? 8 : 4;
    h->info.n = n;
    h->info.uplo = uplo;
    h->info.diag = diag;
    h->info.dtype = dtype;
    h->info.algo = SPTRSV_ALGO_SELF;
    h->info.zero_pivot_row = -1;
    h->info.bad_row = -1;

    sptrsv_status_t st = SPTRSV_SUCCESS;
    keep_pool_memory(dev);
    h->arena.stream = (cudaStream_t)stream;
    if (n > 0) st = analyze_impl(h, rowptr, colidx, vals, (cudaStream_t)stream);
    if (h->arena.stream != nullptr) SPTRSV_CUDA(cudaStreamSynchronize(h->arena.stream));
    h->arena.stream = nullptr;               // later builds / frees: the legacy default stream
    h->status = st;
    h->info.status = st;
    h->info.device_bytes = h->arena.bytes;
    h->info.analysis_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (st == SPTRSV_SUCCESS || st == SPTRSV_ERR_INVALID_MATRIX || st == SPTRSV_ERR_ZERO_PIVOT) {
        *out = h;
        return st;
    }
    h->arena.release_all();
    delete h;
    return st;
}

extern "C" sptrsv_status_t sptrsv_solve(sptrsv_handle_t h, const void *b, void *x, int32_t nrhs,
                                        sptrsv_stream_t stream) {
    if (!h || nrhs < 1) return SPTRSV_ERR_INVALID_VALUE;
    if (h->status != SPTRSV_SUCCESS) return h->status;
    if (h->n == 0) return SPTRSV_SUCCESS;
    if (!b || !x) return SPTRSV_ERR_INVALID_VALUE;
    SPTRSV_CUDA(cudaSetDevice(h->device));
    return solve_impl(h, b, x, nrhs, (cudaStream_t)stream);
}

extern "C" sptrsv_status_t sptrsv_solve_host(sptrsv_handle_t h, const void *b_host, void *x_host,
                                             int32_t nrhs, sptrsv_stream_t stream) {
    if (!h || nrhs < 1) return SPTRSV_ERR_INVALID_VALUE;
    if (h->status != SPTRSV_SUCCESS) return h->status;
    if (h->n == 0) return SPTRSV_SUCCESS;
    if (!b_host || !x_host) return SPTRSV_ERR_INVALID_VALUE;
    SPTRSV_CUDA(cudaSetDevice(h->device));
    cudaStream_t s = (cudaStream_t)stream;
    const size_t bytes = (size_t)h->n * (size_t)nrhs * h->esize;
    if (h->stage_bytes < 2 * bytes) {
        if (h->d_stage) {
            SPTRSV_CUDA(cudaStreamSynchronize(s));
            cudaFree(h->d_stage);
            h->info.device_bytes -= (int64_t)h->stage_bytes;
            h->d_stage = nullptr;
            h->stage_bytes = 0;
        }
        SPTRSV_CUDA(cudaMalloc(&h->d_stage, 2 * bytes));
        h->stage_bytes = 2 * bytes;
        h->info.device_bytes += (int64_t)h->stage_bytes;
    }
    char *db = (char *)h->d_stage;
    char *dx = db + bytes;
    SPTRSV_CUDA(cudaMemcpyAsync(db, b_host, bytes, cudaMemcpyHostToDevice, s));
    sptrsv_status_t st = solve_impl(h, db, dx, nrhs, s);
    if (st != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemcpyAsync(x_host, dx, bytes, cudaMemcpyDeviceToHost, s));
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    return SPTRSV_SUCCESS;
}

extern "C" sptrsv_status_t sptrsv_update_values(sptrsv_handle_t h, const int32_t *rowptr, const int32_t *colidx,
                                                 const void *vals, sptrsv_stream_t stream) {
    if (!h) return SPTRSV_ERR_INVALID_VALUE;
    if (h->status != SPTRSV_SUCCESS) return h->status;
    if (h->n == 0) return SPTRSV_SUCCESS;
    if (!rowptr || !colidx || (!vals && h->diag == SPTRSV_NON_UNIT)) return SPTRSV_ERR_INVALID_VALUE;
    SPTRSV_CUDA(cudaSetDevice(h->device));
    return update_values_impl(h, rowptr, colidx, vals, (cudaStream_t)stream);
}

extern "C" sptrsv_status_t sptrsv_destroy(sptrsv_handle_t h) {
    if (!h) return SPTRSV_SUCCESS;
    cudaSetDevice(h->device);
    h->arena.release_all();
    if (h->d_stage) cudaFree(h->d_stage);
    if (h->d_scratch) cudaFree(h->d_scratch);
    delete h;
    return SPTRSV_SUCCESS;
}

extern "C" sptrsv_status_t sptrsv_set_algo(sptrsv_handle_t h, sptrsv_algo_t algo) {
    if (!h) return SPTRSV_ERR_INVALID_VALUE;
    if (algo != SPTRSV_ALGO_SELF && algo != SPTRSV_ALGO_LEVEL && algo != SPTRSV_ALGO_BLOCK &&
        algo != SPTRSV_ALGO_AUTO && algo != SPTRSV_ALGO_SLFC && algo != SPTRSV_ALGO_LEVC && algo != SPTRSV_ALGO_SMALL)
        return SPTRSV_ERR_INVALID_VALUE;
    if (h->status != SPTRSV_SUCCESS) return h->status;
    if (h->n > 0) SPTRSV_CUDA(cudaSetDevice(h->device));
    if (algo == SPTRSV_ALGO_SMALL) {         // the whole level-ordered layout in one CTA's shared memory
        const sptrsv_status_t st = h->n > 0 ? small_plan(h, true) : SPTRSV_ERR_NOT_SUPPORTED;
        if (st != SPTRSV_SUCCESS) return st;
        h->algo = SPTRSV_ALGO_SMALL;
        h->info.algo = SPTRSV_ALGO_SMALL;
        return SPTRSV_SUCCESS;
    }
    // AUTO only uses BLOCK for rows with <= 3 dependencies: skip its build otherwise
    const bool want_block = algo == SPTRSV_ALGO_BLOCK || (algo == SPTRSV_ALGO_AUTO && h->info.max_row_deps <= 3);
    if (want_block && !h->block.built && h->n > 0) {
        SPTRSV_CUDA(cudaSetDevice(h->device));
        sptrsv_status_t st = block_build(h, nullptr);
        if (st != SPTRSV_SUCCESS && algo != SPTRSV_ALGO_AUTO) return st;
        h->info.nblocks = h->block.built ? h->block.nblocks : 0;
        h->info.device_bytes = h->arena.bytes + (int64_t)h->stage_bytes;
    }
    // BLOCK on a natural-order partition (no grid detected) with more than 3
    // dependencies per row on average: most terms would take the overflow
    // path (cfg4 measured 75x slower than SELF in round 1) -- refused
    if (algo == SPTRSV_ALGO_BLOCK && h->n > 0 && h->block.grid_nx == 0 && h->info.nnz_used > 3 * (int64_t)h->n)
        return SPTRSV_ERR_NOT_SUPPORTED;
    // AUTO: BLOCK on detected grids with <= 3 dependencies per row (5- / 7-point
    // factors); otherwise SMALL when the triangle fits one CTA's shared memory
    // (every level in one pass of <= 32 warps); otherwise SELF (27-point ILU
    // cfg3, general matrices)
    if (algo == SPTRSV_ALGO_AUTO) {
        if (h->block.built && h->block.grid_nx > 0 && h->info.max_row_deps <= 3) algo = SPTRSV_ALGO_BLOCK;
        else if (h->n > 0 && small_plan(h, false) == SPTRSV_SUCCESS) algo = SPTRSV_ALGO_SMALL;
        else algo = SPTRSV_ALGO_SELF;
        cudaGetLastError();
    }
    h->algo = algo;
    h->info.algo = algo;
    return SPTRSV_SUCCESS;
}

extern "C" sptrsv_status_t sptrsv_get_info(sptrsv_handle_t h, sptrsv_info_t *info) {
    if (!h || !info) return SPTRSV_ERR_INVALID_VALUE;
    *info = h->info;
    return SPTRSV_SUCCESS;
}

extern "C" sptrsv_status_t sptrsv_get_levels(sptrsv_handle_t h, int32_t *lev, int32_t *ilev, int32_t *jlev) {
    if (!h) return SPTRSV_ERR_INVALID_VALUE;
    if (h->status != SPTRSV_SUCCESS) return h->status;
    if (h->n == 0) {
        if (ilev) ilev[0] = 0;
        return SPTRSV_SUCCESS;
    }
    SPTRSV_CUDA(cudaSetDevice(h->device));
    if (lev) SPTRSV_CUDA(cudaMemcpy(lev, h->d_lev, sizeof(int32_t) * (size_t)h->n, cudaMemcpyDeviceToHost));
    if (ilev)
        SPTRSV_CUDA(cudaMemcpy(ilev, h->d_ilev, sizeof(int32_t) * ((size_t)h->info.nlev + 1), cudaMemcpyDeviceToHost));
    if (jlev) SPTRSV_CUDA(cudaMemcpy(jlev, h->d_jlev, sizeof(int32_t) * (size_t)h->n, cudaMemcpyDeviceToHost));
    return SPTRSV_SUCCESS;
}

extern "C" sptrsv_status_t sptrsv_get_dep_counts(sptrsv_handle_t h, int32_t *dp) {
    if (!h || !dp) return SPTRSV_ERR_INVALID_VALUE;
    if (h->status != SPTRSV_SUCCESS) return h->status;
    if (h->n == 0) return SPTRSV_SUCCESS;
    SPTRSV_CUDA(cudaSetDevice(h->device));
    SPTRSV_CUDA(cudaMemcpy(dp, h->d_dp, sizeof(int32_t) * (size_t)h->n, cudaMemcpyDeviceToHost));
    return SPTRSV_SUCCESS;
}

extern "C" sptrsv_status_t sptrsv_get_solve_status(sptrsv_handle_t h) {
    if (!h) return SPTRSV_ERR_INVALID_VALUE;
    if (h->status != SPTRSV_SUCCESS) return h->status;
    if (h->n == 0) return SPTRSV_SUCCESS;
    SPTRSV_CUDA(cudaSetDevice(h->device));
    SPTRSV_CUDA(cudaDeviceSynchronize());
    if (h->last_solve == 1) return block_solve_status(h);
    if (h->last_solve == 2) return mrt_solve_status(h);
    return SPTRSV_SUCCESS;
}

extern "C" const char *sptrsv_status_string(sptrsv_status_t s) {
    switch (s) {
        case SPTRSV_SUCCESS: return "SPTRSV_SUCCESS";
        case SPTRSV_ERR_INVALID_VALUE: return "SPTRSV_ERR_INVALID_VALUE";
        case SPTRSV_ERR_INVALID_MATRIX: return "SPTRSV_ERR_INVALID_MATRIX";
        case SPTRSV_ERR_ZERO_PIVOT: return "SPTRSV_ERR_ZERO_PIVOT";
        case SPTRSV_ERR_ALLOC: return "SPTRSV_ERR_ALLOC";
        case SPTRSV_ERR_CUDA: return "SPTRSV_ERR_CUDA";
        case SPTRSV_ERR_NOT_SUPPORTED: return "SPTRSV_ERR_NOT_SUPPORTED";
        case SPTRSV_ERR_TIMEOUT: return "SPTRSV_ERR_TIMEOUT";
    }
    return "SPTRSV_UNKNOWN_STATUS";
}

extern "C" const char *sptrsv_last_cuda_error(void) { return sptrsv::g_last_cuda; }

// ---------------------------------------------------------------- debug hooks
// Not part of include/sptrsv.h: test and profiling instrumentation.

// Level computation of later analyses (process-wide, for the analysis-cost
// study and tests): 0 Kahn by rounds in one cooperative kernel (default),
// 1 the sync-free kernel, 2 one launch per level from a host loop.
extern "C" int sptrsv_dbg_levels_mode(int mode) {
    if (mode < 0 || mode > 2) return SPTRSV_ERR_INVALID_VALUE;
    sptrsv::g_levels_mode = mode;
    return SPTRSV_SUCCESS;
}

// Multi-RHS kernel selection for A/B measurements: 0 automatic, 1 never the
// tile kernel (value-as-flag / level-scheduled kernels only).
extern "C" int sptrsv_dbg_mrhs_path(sptrsv_handle_t h, int mode) {
    if (!h) return SPTRSV_ERR_INVALID_VALUE;
    h->mrhs_path = mode;
    return SPTRSV_SUCCESS;
}

// Per-CTA group trace of multi-RHS tile solves: dev_buf holds K x cap x 2
// uint64 %globaltimer stamps per group (mrt.cu MrtArgs::trace);
// NULL disables.  Returns the CTA count K in *k_out (plan built by a solve).
extern "C" int sptrsv_dbg_mrt_trace(sptrsv_handle_t h, void *dev_buf, int cap, int *k_out) {
    if (!h) return SPTRSV_ERR_INVALID_VALUE;
    h->mrt.trace = dev_buf;
    h->mrt.trace_cap = dev_buf ? cap : 0;
    if (k_out) *k_out = h->mrt.K;
    return SPTRSV_SUCCESS;
}

// BLOCK spin-watchdog timeout of the handle in ns (default 4e9).  Tests set a
// tiny value to force SPTRSV_ERR_TIMEOUT.
extern "C" int sptrsv_dbg_set_timeout_ns(sptrsv_handle_t h, unsigned long long ns) {
    if (!h) return SPTRSV_ERR_INVALID_VALUE;
    h->timeout_ns = ns;
    return SPTRSV_SUCCESS;
}

// Per-warp %globaltimer trace of BLOCK solves: dev_buf holds nunits x cap
// uint64 (entry t: start of step t, t < cap - 1, at TMA-block starts; entry
// cap - 1: end).  NULL disables.
extern "C" int sptrsv_dbg_block_trace(sptrsv_handle_t h, void *dev_buf, int cap) {
    if (!h) return SPTRSV_ERR_INVALID_VALUE;
    h->block.trace = dev_buf;
    h->block.trace_cap = dev_buf ? cap : 0;
    return SPTRSV_SUCCESS;
}

// Inbound-item delivery trace of BLOCK solves: dev_buf holds nitems uint64
// (%globaltimer when the fetcher stored the item), NULL disables.  Items are
// reported by sptrsv_dbg_block_items.
extern "C" int sptrsv_dbg_block_ftrace(sptrsv_handle_t h, void *dev_buf) {
    if (!h) return SPTRSV_ERR_INVALID_VALUE;
    h->block.ftrace = dev_buf;
    return SPTRSV_SUCCESS;
}

// Mailbox publication trace of BLOCK solves (active only while the step
// trace is on): dev_buf holds G uint64 (%globaltimer when mailbox g was
// written), NULL disables.
extern "C" int sptrsv_dbg_block_ptrace(sptrsv_handle_t h, void *dev_buf) {
    if (!h) return SPTRSV_ERR_INVALID_VALUE;
    h->block.ptrace = dev_buf;
    return SPTRSV_SUCCESS;
}

// Copies the inbound items {mailbox, slot} (nitems int2, by (warp, level)), the
// per-warp item ranges (K*wpc+1 int) and the items' (warp * nlev + level) keys to host buffers.
extern "C" int sptrsv_dbg_block_items(sptrsv_handle_t h, void *items, void *fptr, void *keys) {
    if (!h || !h->block.built) return SPTRSV_ERR_INVALID_VALUE;
    const sptrsv::BlockPlan &B = h->block;
    if (keys && B.nitems > 0 && cudaMemcpy(keys, B.d_fkey, sizeof(uint32_t) * B.nitems, cudaMemcpyDeviceToHost) != cudaSuccess)
        return SPTRSV_ERR_CUDA;
    if (items && B.nitems > 0 && cudaMemcpy(items, B.d_fitems, sizeof(int2) * B.nitems, cudaMemcpyDeviceToHost) != cudaSuccess)
        return SPTRSV_ERR_CUDA;
    if (fptr && cudaMemcpy(fptr, B.d_fptr, sizeof(int32_t) * (B.nunits + 1), cudaMemcpyDeviceToHost) != cudaSuccess)
        return SPTRSV_ERR_CUDA;
    return SPTRSV_SUCCESS;
}

// BLOCK plan summary for tools: {K, wpc, nsteps, G, nslots, smem, rec_bytes,
// tile_w, tile_h, cluster size, cluster x extent, inbound items, gl}
extern "C" int sptrsv_dbg_block_plan(sptrsv_handle_t h, long long *out13) {
    if (!h || !out13) return SPTRSV_ERR_INVALID_VALUE;
    const sptrsv::BlockPlan &B = h->block;
    const long long v[13] = {B.nblocks, B.wpc, B.nsteps, B.G, B.nslots, (long long)B.smem, B.rec_bytes, B.tile_w,
                             B.tile_h, B.cs, B.csx, B.nitems, B.gl ? 1 : 0};
    for (int i = 0; i < 13; ++i) out13[i] = v[i];
    return B.built ? SPTRSV_SUCCESS : SPTRSV_ERR_NOT_SUPPORTED;
}
