/*
 * sptrsv.h -- C ABI of the B200 (sm_100a) sparse triangular solve library.
 *
 * Operation (§3, Eq. (1)): solve  (L+D) x = f  or
 * (U+D) x = f  for a sparse lower or upper triangular matrix stored in CSR,
 * with a unit or non-unit diagonal, for one or many right-hand sides.
 *
 *   sptrsv_analyze  -- the setup phase (§4.4, Table 1): CSR
 *                      validation, dependency counts (DEP), level
 *                      sets (LEV), row reordering by level
 *                      (P:666-678); all on the GPU.
 *   sptrsv_solve    -- the solve phase: self-scheduled (Alg. 3 SLFR,
 *                      P:347-376) or level-scheduled (Alg. 1 LEVR,
 *                      P:272-285), single or multiple right-hand sides.
 *   sptrsv_destroy  -- frees the handle.
 *
 * Conventions
 *   - Indices are 0-based int32.  A CSR of order n is (rowptr[n+1],
 *     colidx[nnz], vals[nnz]) with nnz = rowptr[n] <= INT32_MAX.
 *   - Only the `uplo` triangle is referenced (BLAS trsv convention): entries
 *     of the other triangle are ignored and counted in
 *     sptrsv_info_t.ignored_entries.  With SPTRSV_UNIT the stored diagonal is
 *     not referenced and is taken as 1 (so one combined ILU(0) CSR serves as
 *     both the unit-lower L and the non-unit-upper U).
 *   - Levels are 0-based: lev(i) = 0 if row i has no dependency in the
 *     selected triangle, else 1 + max lev(j) over its dependencies j
 *     (backward: P:259-260).  nlev = 1 + max lev (0 for n = 0).
 *     jlev lists rows by ascending (lev, row id); ilev[l] is the position of
 *     level l's first row, ilev[nlev] = n.
 *   - Right-hand sides and solutions are ROW-MAJOR n x nrhs arrays: element
 *     (i, r) is at index i*nrhs + r (a contiguous torch (n, nrhs) tensor).
 *   - A stream is a cudaStream_t passed as an opaque pointer (NULL = the
 *     legacy default stream); the header needs no CUDA include.
 *   - Every entry point returns a status; none aborts the process.
 *
 * Thread-safety: a handle may be used by one host thread at a time.  Solves
 * on one handle must be stream-ordered (the handle's ready flags and epoch
 * counter are per-handle state); concurrent solves need separate handles.
 */
#ifndef SPTRSV_H
#define SPTRSV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sptrsv_handle_s *sptrsv_handle_t;
typedef void *sptrsv_stream_t;          /* cudaStream_t */

typedef enum { SPTRSV_LOWER = 0, SPTRSV_UPPER = 1 } sptrsv_uplo_t;
typedef enum { SPTRSV_NON_UNIT = 0, SPTRSV_UNIT = 1 } sptrsv_diag_t;
typedef enum { SPTRSV_F64 = 0, SPTRSV_F32 = 1 } sptrsv_dtype_t;

typedef enum {
    SPTRSV_ALGO_SELF = 0,   /* self-scheduled, per-row ready flags (SLFR) */
    SPTRSV_ALGO_LEVEL = 1,  /* level-scheduled, grid-wide barrier per level (LEVR) */
    SPTRSV_ALGO_BLOCK = 2,  /* self-scheduled over warp-owned row tiles, register/shared-memory
                               hand-offs.  Any matrix on a detected structured
                               grid; otherwise only if nnz_used <= 3 n (NOT_SUPPORTED above) */
    SPTRSV_ALGO_AUTO = 3,   /* BLOCK when the analysis detects a structured grid AND every row
                               has <= 3 dependencies (5-/7-point factors); else SMALL when the
                               triangle fits one CTA's shared memory (every level in one pass
                               of 32 warps); else SELF.  info.algo reports the choice */
    /* 4: retired (round-1 CTA-tile variant); sptrsv_set_algo(4) returns INVALID_VALUE */
    SPTRSV_ALGO_SLFC = 5,   /* column-wise self-scheduled (Alg. SLFC, kernel P:631-653):
                               per-column dependency counters, x updates pushed by L2
                               atomics; last-bit results vary run to run (atomic order).
                               nrhs > 1 solves use the self-scheduled row kernels */
    SPTRSV_ALGO_LEVC = 6,   /* column-wise level-scheduled (Alg. LEVC, kernel
                               P:536-552): atomics, grid-wide barrier per level.  nrhs > 1
                               solves use the level-scheduled row kernel */
    SPTRSV_ALGO_SMALL = 7   /* small systems: one CTA solves level by level (LEVR)
                               with the level-ordered triangle and x staged in shared memory.
                               NOT_SUPPORTED if the layout does not fit one CTA's shared
                               memory */
} sptrsv_algo_t;

typedef enum {
    SPTRSV_SUCCESS = 0,
    SPTRSV_ERR_INVALID_VALUE = 1,   /* NULL pointer with n > 0, n < 0, nrhs < 1, bad enum, NULL handle */
    SPTRSV_ERR_INVALID_MATRIX = 2,  /* a malformed row; see sptrsv_analyze */
    SPTRSV_ERR_ZERO_PIVOT = 3,      /* NON_UNIT: a row without a stored diagonal or with d(i) == 0 */
    SPTRSV_ERR_ALLOC = 4,           /* device or host allocation failed */
    SPTRSV_ERR_CUDA = 5,            /* a CUDA runtime call failed (message via sptrsv_last_cuda_error) */
    SPTRSV_ERR_NOT_SUPPORTED = 6,   /* no sm_100 device, or a size beyond the int32 index space */
    SPTRSV_ERR_TIMEOUT = 7          /* a BLOCK or multi-RHS tile solve gave up a spin wait (watchdog,
                                       default 4 s); reported by sptrsv_get_solve_status, x is invalid */
} sptrsv_status_t;

typedef struct {
    int32_t n;
    int32_t nlev;              /* number of levels */
    int32_t max_level_width;   /* max over levels of ilev[l+1] - ilev[l] */
    int32_t zero_pivot_row;    /* smallest zero-pivot row, or -1 */
    int32_t bad_row;           /* smallest malformed row, or -1 */
    int32_t uplo, diag, dtype, algo;
    int32_t max_row_deps;      /* max dependencies of one row */
    int64_t nnz_input;         /* rowptr[n] */
    int64_t nnz_used;          /* referenced off-diagonal entries (sum of dp) */
    int64_t ignored_entries;   /* stored but unreferenced entries */
    int32_t status;            /* the analysis status (sptrsv_status_t) */
    int32_t nblocks;           /* SPTRSV_ALGO_BLOCK: number of row blocks (0 if not built) */
    double analysis_ms;        /* wall time of sptrsv_analyze (host clock, includes the final sync) */
    int64_t device_bytes;      /* device memory owned by the handle */
} sptrsv_info_t;

/*
 * sptrsv_analyze -- setup phase.
 *   n        order of the matrix (n >= 0; n == 0 gives an empty handle).
 *   rowptr   DEVICE pointer, int32[n+1]; colidx DEVICE int32[nnz];
 *   vals     DEVICE pointer to nnz values of `dtype` (may be NULL only if
 *            diag == SPTRSV_UNIT and the triangle has no off-diagonal entry:
 *            else INVALID_VALUE).  Caller-owned; read during the call only.
 *   uplo, diag, dtype   as above.
 *   stream   stream for the analysis kernels; the call synchronizes it before
 *            returning, so the inputs may be freed afterwards.
 *   out      receives a new handle.  On SPTRSV_ERR_INVALID_MATRIX and
 *            SPTRSV_ERR_ZERO_PIVOT a handle IS returned (its info holds
 *            bad_row / zero_pivot_row, and sptrsv_solve on it returns the
 *            same status); on other errors *out is NULL.
 * Row i is MALFORMED iff rowptr[i] < 0, rowptr[i+1] < rowptr[i],
 * rowptr[i+1] > rowptr[n], (i == 0 and rowptr[0] != 0), or -- if its
 * pointers are sound -- a column lies outside [0, n) or its columns are not
 * strictly increasing.  Precedence: INVALID_VALUE, INVALID_MATRIX (smallest
 * malformed row), ZERO_PIVOT (smallest such row).
 * The handle owns: the level-ordered copy of the referenced triangle,
 * reciprocal diagonal, lev/ilev/jlev, dependency counts, ready flags, the
 * block schedule, and staging buffers for sptrsv_solve_host.
 */
sptrsv_status_t sptrsv_analyze(int32_t n, const int32_t *rowptr, const int32_t *colidx,
                               const void *vals, sptrsv_uplo_t uplo, sptrsv_diag_t diag,
                               sptrsv_dtype_t dtype, sptrsv_stream_t stream,
                               sptrsv_handle_t *out);

/*
 * sptrsv_solve -- x = T^{-1} b on `stream`.
 *   b, x   DEVICE pointers, row-major n x nrhs of the handle's dtype;
 *          x == b (in place, "x is first initialized as f") is allowed;
 *          other overlaps are not.  Caller-owned; valid until the stream
 *          work completes.  Alignment: the dtype's natural alignment.
 *   nrhs   >= 1, any width.  nrhs == 1 uses the handle's algorithm.  nrhs > 1
 *          (algorithm not LEVEL / LEVC): nrhs <= 16 the self-scheduled
 *          value-as-flag multi-RHS kernel; nrhs > 16 on factors with <= 4
 *          dependencies per row, with b, x 16-byte aligned and nrhs * sizeof
 *          a multiple of 16 bytes, the multi-RHS tile kernel (column blocks of
 *          <= 64; its plan is built on the first such solve); otherwise the
 *          level-scheduled multi-RHS kernel over independent column blocks of
 *          <= 128 (also for LEVEL / LEVC).
 * Arithmetic per (row, column): s = b(i); s = fma(-a(k), x(ja(k)), s) in CSR
 * storage order; x(i) = s * (1/d(i)) (s for UNIT).  This holds for BLOCK, for
 * every multi-RHS kernel and for SELF / LEVEL rows with <= 16 dependencies,
 * so those results are run-to-run bitwise reproducible and a column's result
 * does not depend on nrhs or the column block it is in.  SELF / LEVEL rows
 * with > 16 dependencies (warp per row) sum lane partials with a fixed
 * shuffle tree and compute b(i) - sum (reproducible, not storage order);
 * SLFC / LEVC accumulate with atomics (order varies run to run).
 * Asynchrony: no host synchronization, except on the first multi-RHS solve of
 * a handle (and the first tile-kernel solve), which builds the per-position
 * CSR or the tile plan (allocates, synchronizes `stream`).  In-place SELF and multi-RHS solves copy b into a handle-owned
 * scratch buffer (stream-ordered allocation, cudaMallocAsync) because x is
 * their flag array.  Run one multi-RHS solve before capturing a CUDA graph.
 * Returns INVALID_VALUE on bad arguments, the analysis status if the handle
 * holds an analysis error, CUDA on a launch failure.  A BLOCK solve whose spin
 * wait exceeded the watchdog (BLOCK, or the multi-RHS tile kernel) returns
 * SUCCESS here (it is asynchronous) and TIMEOUT from sptrsv_get_solve_status.
 */
sptrsv_status_t sptrsv_solve(sptrsv_handle_t h, const void *b, void *x, int32_t nrhs,
                             sptrsv_stream_t stream);

/*
 * sptrsv_solve_host -- the same solve with HOST buffers: copies b (n x nrhs)
 * into handle-owned device staging memory, solves, copies x back, all
 * enqueued on `stream`; the call then synchronizes the stream.  b and x may
 * be pageable or pinned (pinned gives asynchronous DMA).  x == b allowed.
 */
sptrsv_status_t sptrsv_solve_host(sptrsv_handle_t h, const void *b_host, void *x_host,
                                  int32_t nrhs, sptrsv_stream_t stream);

/*
 * sptrsv_update_values -- new values for the analyzed pattern (numerical
 * refactorization: the ILU factors of matrices with one sparsity
 * pattern share their triangular patterns, so the setup phase is reused).
 *   rowptr, colidx, vals   DEVICE pointers: the same CSR pattern as given to
 *          sptrsv_analyze (identical rowptr / colidx; vals may be NULL only
 *          for UNIT handles), caller-owned, read during the call only.
 * Validates with sptrsv_analyze's rules, then replaces the values of every
 * layout the handle holds (level-ordered rows, BLOCK records, multi-RHS and
 * column-wise layouts).  Synchronizes `stream` before returning.  Errors:
 * INVALID_MATRIX / ZERO_PIVOT as sptrsv_analyze; INVALID_VALUE if the
 * referenced pattern differs from the analyzed one; the handle then keeps
 * its old values.
 */
sptrsv_status_t sptrsv_update_values(sptrsv_handle_t h, const int32_t *rowptr, const int32_t *colidx,
                                     const void *vals, sptrsv_stream_t stream);

/* Frees the handle and its device memory.  NULL is a no-op.  Outstanding
 * solves on the handle must have completed. */
sptrsv_status_t sptrsv_destroy(sptrsv_handle_t h);

/* Selects the single-RHS algorithm (default SPTRSV_ALGO_SELF).  The BLOCK
 * schedule is built lazily on first use (BLOCK or AUTO; device kernels on the
 * default stream, synchronized).  Errors: INVALID_VALUE (NULL handle, bad
 * enum), NOT_SUPPORTED (BLOCK only: the plan does not fit the device), the
 * analysis status of a failed handle. */
sptrsv_status_t sptrsv_set_algo(sptrsv_handle_t h, sptrsv_algo_t algo);

/* Copies the handle's summary into *info (host pointer). */
sptrsv_status_t sptrsv_get_info(sptrsv_handle_t h, sptrsv_info_t *info);

/* Copies lev[n], ilev[nlev+1], jlev[n] to HOST buffers (any may be NULL). */
sptrsv_status_t sptrsv_get_levels(sptrsv_handle_t h, int32_t *lev, int32_t *ilev, int32_t *jlev);

/* Copies the dependency counts dp[n] to a HOST buffer. */
sptrsv_status_t sptrsv_get_dep_counts(sptrsv_handle_t h, int32_t *dp);

/*
 * sptrsv_get_solve_status -- synchronizes the device, then reports whether the
 * LAST solve on the handle completed: SUCCESS, or TIMEOUT if it was a BLOCK
 * or multi-RHS tile solve that gave up a spin wait (its x is invalid).  The
 * watchdog is per handle and per solve: the next solve starts clean.
 * (SPEC.md:259 timeout guard; the other kernels have no watchdog and always
 * report SUCCESS.)
 */
sptrsv_status_t sptrsv_get_solve_status(sptrsv_handle_t h);

/* Static string for a status code. */
const char *sptrsv_status_string(sptrsv_status_t s);

/* Message of the last CUDA error seen by the library on this thread ("" if none). */
const char *sptrsv_last_cuda_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SPTRSV_H */
