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

// Device allocation bookkeeping of one handle.
struct DevArena {
    std::vector<void *> ptrs;
    int64_t bytes = 0;
    sptrsv_status_t alloc(void **p, size_t nbytes);
    template <typename T> sptrsv_status_t alloc_n(T **p, size_t n) {
        return alloc(reinterpret_cast<void **>(p), n * sizeof(T));
    }
    void release_all();
};

// Block-schedule (SPTRSV_ALGO_BLOCK) device data; see block.cu.
struct BlockPlan {
    bool built = false;
    bool lean = false;        // k_block1 (one warp per tile) instead of k_block
    int32_t nblocks = 0;      // K co-resident CTAs
    int32_t wpc = 0;          // tiles per CTA
    int32_t nunits = 0;       // K x wpc tiles (a compute and a helper warp each)
    int32_t W = 0;            // EXT entries per record row (kernel instance)
    int32_t nst = 0;          // record ring per warp (steps)
    int32_t bb = 0;           // b lookahead (steps)
    int32_t d = 0;            // record lookahead (steps)
    int32_t r1 = 0, rr = 0;   // row-id lookahead / ring (steps)
    int32_t nsteps = 0;       // (warp, level) steps of <= 32 rows
    int32_t G = 0;            // global mailboxes (values read by another CTA)
    int32_t nslots = 0;       // shared slots per CTA (values read by another warp of the CTA)
    int32_t novf = 0, threads = 0, rec_bytes = 0;
    int32_t grid_nx = 0, grid_ny = 0, tile_w = 0, tile_h = 0;   // detected grid / warp tile (0 = natural)
    int64_t nent = 0;         // record bytes
    size_t smem = 0;
    void *kernel = nullptr;
    int32_t *d_unit_step0 = nullptr;  // [U+1] first step of every warp
    void *d_recs = nullptr;           // step records (see block.cu)
    int32_t *d_rows = nullptr;        // [nsteps][32] row ids (b gather addresses)
    int32_t *d_cta_g0 = nullptr;      // [K+1] mailbox range of every CTA
    int32_t *d_ovf_code = nullptr;    // overflow entries (rows with > W dependencies)
    void *d_ovf_val = nullptr;
    void *d_gmb = nullptr;            // [2][G] mailboxes (value-as-flag), roles swap per solve
    unsigned *d_ctr = nullptr;        // [0] solve epoch, [1] finished CTAs
    int32_t *d_unit = nullptr;        // [n] warp tile of every row (CTA = unit / wpc)
    // CTA-tile multi-RHS plan (built on the first multi-RHS BLOCK solve; see block.cu)
    bool tm_built = false;
    int32_t tm_K = 0;
    int32_t *d_tm_perm = nullptr;     // [n] position -> row, positions sorted by (CTA, level, row)
    void *d_tm_invd = nullptr;        // [n] 1/d by position
    int32_t *d_tm_ptr = nullptr;      // [n+1] CSR of the referenced strict triangle by position
    int32_t *d_tm_col = nullptr;
    void *d_tm_val = nullptr;
    int32_t *d_tm_off = nullptr;      // [K*nlev+1] first position of (CTA, level)
    int32_t *d_tm_dptr = nullptr;     // [K+1] producer-CTA lists
    int32_t *d_tm_dl = nullptr;
    unsigned long long *d_tm_done = nullptr;   // [K] levels completed (epoch based, monotone)
    unsigned long long tm_base = 0;
};

// CTA-tile level-synchronous plan (SPTRSV_ALGO_TILE); see tile.cu.
struct TilePlan {
    bool built = false;
    int32_t K = 0, threads = 0, maxr = 0;
    size_t smem = 0;
    void *kernel = nullptr;
    int4 *d_clist = nullptr;          // per CTA non-empty levels {level, first position, rows, 0}
    int32_t *d_cptr = nullptr;        // [K+1]
    int32_t *d_cpos = nullptr;        // [K+1] first position of every CTA
    int4 *d_ri = nullptr;             // [n] {row, code0..2}
    void *d_rv = nullptr;             // [n][4] {1/d, v0..v2}
    unsigned long long *d_done = nullptr;   // [K] level counters (epoch based)
    unsigned long long base = 0;
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
    int32_t self_grid = 0, level_grid = 0, mrhs_grid = 0;
    bool self_u16 = false;                   // k_self instance of self_grid (SPTRSV_WPR_U)
    // in-place / host staging
    void *d_stage = nullptr;
    size_t stage_bytes = 0;
    void *d_scratch = nullptr;               // copy of b for in-place value-as-flag solves
    size_t scratch_bytes = 0;
    sptrsv::BlockPlan block;
    sptrsv::TilePlan tile;
};

namespace sptrsv {
sptrsv_status_t analyze_impl(sptrsv_handle_t h, const int32_t *rowptr, const int32_t *colidx,
                             const void *vals, cudaStream_t s);
sptrsv_status_t solve_impl(sptrsv_handle_t h, const void *b, void *x, int32_t nrhs, cudaStream_t s);
sptrsv_status_t block_build(sptrsv_handle_t h, cudaStream_t s);
sptrsv_status_t block_solve(sptrsv_handle_t h, const void *b, void *x, cudaStream_t s);
sptrsv_status_t tile_mrhs_build(sptrsv_handle_t h, cudaStream_t s);
sptrsv_status_t tile_build(sptrsv_handle_t h, cudaStream_t s);
sptrsv_status_t tile_solve(sptrsv_handle_t h, const void *b, void *x, cudaStream_t s);
sptrsv_status_t column_solve(sptrsv_handle_t h, const void *b, void *x, cudaStream_t s);   // column.cu
sptrsv_status_t build_mr_any(sptrsv_handle_t h, cudaStream_t s);                            // solve.cu
// device scans (analyze.cu)
sptrsv_status_t exclusive_scan_i32(const int32_t *in, int32_t *out, int64_t n, DevArena &tmp, cudaStream_t s);
sptrsv_status_t exclusive_scan_i64(const int64_t *in, int64_t *out, int64_t n, DevArena &tmp, cudaStream_t s);
sptrsv_status_t radix_sort_pairs(const uint32_t *keys_in, const int32_t *vals_in, uint32_t *keys_out,
                                 int32_t *vals_out, int64_t n, uint32_t max_key, DevArena &tmp,
                                 cudaStream_t s);
}  // namespace sptrsv
