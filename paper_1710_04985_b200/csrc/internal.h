// internal.h -- the handle and host-side helpers of libsptrsv (not part of the ABI).
#pragma once

#include <cstdint>
#include <string>
#include <vector>
#include <cuda_runtime.h>

#include "sptrsv.h"
#include "common.cuh"

namespace sptrsv {

// Records the last CUDA error message (thread-local) and maps it to a status.
sptrsv_status_t cuda_fail(cudaError_t e, const char *where);
#define SPTRSV_CUDA(call)                                                   \
    do {                                                                    \
        cudaError_t _e = (call);                                            \
        if (_e != cudaSuccess) return ::sptrsv::cuda_fail(_e, #call);       \
    } while (0)

// Device allocation bookkeeping of one handle (or of one call's temporaries).
// Stream-ordered allocations from the device's default memory pool
// (cudaMallocAsync / cudaFreeAsync on `stream`): no device-wide
// synchronisation on free, and pool reuse across handles (the pool keeps its
// memory: release threshold set at the first analysis).
struct DevArena {
    std::vector<void *> ptrs;
    int64_t bytes = 0;
    cudaStream_t stream = nullptr;
    DevArena() = default;
    explicit DevArena(cudaStream_t s) : stream(s) {}
    sptrsv_status_t alloc(void **p, size_t nbytes);
    template <typename T> sptrsv_status_t alloc_n(T **p, size_t n) {
        return alloc(reinterpret_cast<void **>(p), n * sizeof(T));
    }
    void release_all();
};
// Scoped stream of a handle arena's allocations (restored on exit).
struct ArenaStream {
    DevArena &a;
    cudaStream_t old;
    ArenaStream(DevArena &arena, cudaStream_t s) : a(arena), old(arena.stream) { a.stream = s; }
    ~ArenaStream() { a.stream = old; }
};

// Block-schedule (SPTRSV_ALGO_BLOCK) device data; see block.cu.
struct BlockPlan {
    bool built = false;
    int32_t nblocks = 0;      // K co-resident CTAs
    int32_t wpc = 0;          // warp tiles per CTA
    int32_t nunits = 0;       // K x wpc tiles (one warp each)
    int32_t nsteps = 0;       // (warp, level) steps of <= 32 rows
    int32_t npad = 0;         // steps after padding every warp to a multiple of the loop unroll
    int32_t G = 0;            // global mailboxes (values read by another CTA)
    int32_t nslots = 0;       // shared slots per CTA (values read by another warp of the CTA)
    int32_t novf = 0, threads = 0, rec_bytes = 0;   // rec_bytes: both streams, per step
    int32_t grid_nx = 0, grid_ny = 0, tile_w = 0, tile_h = 0;   // detected grid / warp tile (0 = natural)
    int64_t nent = 0;         // record bytes
    size_t smem = 0;
    void *kernel = nullptr;
    int32_t *d_unit_step0 = nullptr;  // [U+1] first step of every warp
    int32_t *d_unit_lev0 = nullptr;   // [U] level of every warp's first row (prologue stagger)
    void *d_ctl = nullptr;            // step records: control stream (see block.cu)
    void *d_coef = nullptr;           // step records: coefficient stream
    int32_t *d_cta_g0 = nullptr;      // [K+1] mailbox range of every CTA
    int2 *d_fitems = nullptr;         // inbound items {mailbox, shared slot} by (CTA, level) (fetcher warps)
    int32_t *d_fptr = nullptr;        // [K*wpc+1] inbound item range of every compute warp
    uint32_t *d_fkey = nullptr;       // [nitems] (CTA, level) key of every item (tools)
    int32_t nitems = 0;
    bool gl = false;                  // fallback: consumers poll mailboxes themselves (slots did not fit)
    int32_t cs = 1, csx = 1;          // CTAs per cluster (DSMEM hand-offs inside a cluster), x extent
    int32_t *d_ovf_code = nullptr;    // overflow lists (rows with > 3 dependencies)
    void *d_ovf_val = nullptr;
    void *d_gmb = nullptr;            // [2][G] mailboxes (value-as-flag), roles swap per solve
    unsigned *d_ctr = nullptr;        // [0] solve epoch, [1] finished CTAs, [2] timed-out epoch + 1
    int32_t *d_unit = nullptr;        // [n] warp tile of every row (CTA = unit / wpc)
    void *trace = nullptr;            // debug (sptrsv_dbg_block_trace): per-warp step timestamps
    void *ftrace = nullptr;           // debug: inbound item delivery timestamps
    void *ptrace = nullptr;           // debug: mailbox publication timestamps (with trace on)
    int32_t trace_cap = 0;
};

// Multi-RHS tile plan (mrt.cu)
struct MrtPlan {
    bool built = false, failed = false;
    int32_t K = 0, ngroups = 0, nwaits = 0;
    int32_t *d_gc0 = nullptr;         // [K+1] first group of every CTA
    int32_t *d_gstart = nullptr;      // [ngroups+1] first solve position of every group
    int32_t *d_wptr = nullptr;        // [ngroups+1] wait list of every group
    int2 *d_waits = nullptr;          // {producer CTA, groups needed}
    int32_t *d_hptr = nullptr;        // [ngroups+1] halo list of every group
    int32_t *d_hrow = nullptr;        // halo rows (TMA-copied before their group)
    int32_t nhalo = 0;
    unsigned char *d_rec = nullptr;   // per-position records
    unsigned long long *d_prog = nullptr;   // [K] (epoch << 32) | groups done
    unsigned *d_status = nullptr;     // [0] epoch of the last launch whose wait timed out
    unsigned epoch = 0, solve_first = 0;
    void *trace = nullptr;            // debug (sptrsv_dbg_mrt_trace)
    int32_t trace_cap = 0;
};

}  // namespace sptrsv

struct sptrsv_handle_s {
    int32_t n = 0;
    int32_t uplo = 0, diag = 0, dtype = 0, algo = SPTRSV_ALGO_SELF;
    sptrsv_status_t status = SPTRSV_SUCCESS;
    sptrsv_info_t info{};
    int device = 0;
    int num_sms = 0;
    size_t esize = 8;                        // sizeof value type

    sptrsv::DevArena arena;
    // analysis results
    int32_t *d_dp = nullptr;                 // [n] dependency counts
    int32_t *d_lev = nullptr;                // [n]
    int32_t *d_ilev = nullptr;               // [nlev+1]
    int32_t *d_jlev = nullptr;               // [n]
    void *d_invd_row = nullptr;              // [n] 1/d(i) by row (dtype)
    // level-ordered layout (SELF / LEVEL / MRHS)
    int32_t nchunks = 0;
    sptrsv::ChunkDesc *d_chunks = nullptr;   // [nchunks]
    int32_t *d_lev_chunk = nullptr;          // [nlev+1]
    int32_t *d_chunk_lev = nullptr;          // [nchunks] level of each chunk
    unsigned *d_done = nullptr;              // [nlev] per-level completed-chunk counters (SELF hint)
    unsigned self_epoch = 0;                 // SELF solves so far (done[l] == self_epoch * chunks(l))
    int32_t *d_perm = nullptr;               // [n] solve position -> row
    void *d_invd = nullptr;                  // [n] 1/d by solve position
    int32_t *d_ecol = nullptr;
    void *d_eval = nullptr;
    int64_t nent = 0;
    // multi-RHS per-position CSR (built on the first nrhs > 1 solve)
    bool mr_built = false;
    int32_t *d_mr_ptr = nullptr;
    int32_t *d_mr_col = nullptr;
    void *d_mr_val = nullptr;
    // CSC of the referenced strict triangle (SLFC / LEVC, column.cu; built on first use)
    bool csc_built = false;
    int32_t *d_c_ptr = nullptr;              // [n+1] by column (row id)
    int32_t *d_c_row = nullptr;              // dependent rows of each column
    void *d_c_val = nullptr;
    int32_t *d_count = nullptr;              // [n] SLFC dependency counters (reset from d_dp per solve)
    int32_t slfc_grid = 0;
    // synchronisation state
    int32_t *d_flags = nullptr;              // [n] per-row ready flags (epoch tagged)
    int32_t epoch = 0;
    unsigned *d_ctr = nullptr;               // [0] ticket, [1] exit count (self / mrhs)
    unsigned long long *d_bar = nullptr;     // level barrier counter (monotone)
    unsigned long long bar_base = 0;
    int32_t self_grid = 0, vf_grid = 0;       // resident grids (computed on first use)
    int32_t small_threads = 0;               // SMALL: CTA size (0: no plan yet)
    // in-place / host staging
    void *d_stage = nullptr;
    size_t stage_bytes = 0;
    void *d_scratch = nullptr;               // copy of b for in-place value-as-flag solves
    size_t scratch_bytes = 0;
    sptrsv::BlockPlan block;
    sptrsv::MrtPlan mrt;
    int mrhs_path = 0;                       // debug (sptrsv_dbg_mrhs_path): 0 auto, 1 never the tile kernel
    // spin watchdog of the BLOCK solve (sptrsv_get_solve_status)
    unsigned long long timeout_ns = 4000000000ull;
    int last_solve = 0;                      // 1: BLOCK, 2: multi-RHS tile (spin-wait kernels with a watchdog)
};

namespace sptrsv {
void keep_pool_memory(int dev);
extern int g_levels_mode;                    // analyze.cu (sptrsv_dbg_levels_mode)
sptrsv_status_t update_values_impl(sptrsv_handle_t h, const int32_t *rowptr, const int32_t *colidx,
                                   const void *vals, cudaStream_t s);                      // analyze.cu
// new values into every derived layout the handle has built (from its level-ordered layout)
sptrsv_status_t refresh_derived_values(sptrsv_handle_t h, cudaStream_t s);                 // solve.cu
sptrsv_status_t block_refresh_values(sptrsv_handle_t h, const int32_t *tri_ptr, const void *tri_val,
                                     cudaStream_t s);                                       // block.cu
sptrsv_status_t mrt_refresh_values(sptrsv_handle_t h, const int32_t *tri_ptr, const void *tri_val,
                                   cudaStream_t s);                                         // mrt.cu
sptrsv_status_t csc_refresh_values(sptrsv_handle_t h, cudaStream_t s);                      // column.cu
sptrsv_status_t analyze_impl(sptrsv_handle_t h, const int32_t *rowptr, const int32_t *colidx,
                             const void *vals, cudaStream_t s);
sptrsv_status_t solve_impl(sptrsv_handle_t h, const void *b, void *x, int32_t nrhs, cudaStream_t s);
sptrsv_status_t block_build(sptrsv_handle_t h, cudaStream_t s);
sptrsv_status_t block_solve(sptrsv_handle_t h, const void *b, void *x, cudaStream_t s);
sptrsv_status_t block_solve_status(sptrsv_handle_t h);
sptrsv_status_t build_tri_csr(sptrsv_handle_t h, DevArena &tmp, cudaStream_t s, int32_t **ptr, int32_t **col,
                              void **val);                                                   // block.cu
// multi-RHS tile solve (mrt.cu): plan built on the first eligible multi-RHS solve
bool mrt_eligible(sptrsv_handle_t h, const void *b, const void *x, int32_t nrhs);
sptrsv_status_t mrt_solve(sptrsv_handle_t h, const void *b, void *x, int32_t nrhs, cudaStream_t s);
sptrsv_status_t mrt_solve_status(sptrsv_handle_t h);
sptrsv_status_t column_solve(sptrsv_handle_t h, const void *b, void *x, cudaStream_t s);   // column.cu
sptrsv_status_t build_mr_any(sptrsv_handle_t h, cudaStream_t s);
sptrsv_status_t small_plan(sptrsv_handle_t h, bool explicit_request);                                              // solve.cu                            // solve.cu
// device scans (analyze.cu)
sptrsv_status_t exclusive_scan_i32(const int32_t *in, int32_t *out, int64_t n, DevArena &tmp, cudaStream_t s);
sptrsv_status_t exclusive_scan_i64(const int64_t *in, int64_t *out, int64_t n, DevArena &tmp, cudaStream_t s);
sptrsv_status_t radix_sort_pairs(const uint32_t *keys_in, const int32_t *vals_in, uint32_t *keys_out,
                                 int32_t *vals_out, int64_t n, uint32_t max_key, DevArena &tmp,
                                 cudaStream_t s);
}  // namespace sptrsv
