// block.cu -- SPTRSV_ALGO_BLOCK: self-scheduling over warp-owned row tiles
// (SURVEY.md §7 hard part H1).
//
// Why: the self-scheduled solve's time is its critical path, nlev dependent
// hand-offs (382 on cfg2).  A cross-SM hand-off costs an L2 round
// trip (~220 ns one way, profiles/microbench_r1.json), a warp shuffle ~25
// cycles.  So the rows are partitioned over warps such that almost every edge
// of the critical path stays inside one warp:
//
//   * structured grids (detected: every dependency is verified to be a 3x3x3
//     neighbour under the inferred nx, ny): a warp owns a tile of <= 32
//     z-columns (x, y), a CTA a rectangle of warp tiles; lane = column.  Warp
//     step t solves the tile's rows of its t-th level, so the dependencies of
//     a 7-point row on (x-1,y,z), (x,y-1,z), (x,y,z-1) were solved in the
//     previous step by this warp and arrive by __shfl_sync from registers.
//   * otherwise contiguous natural-order row blocks (correct for any matrix).
//
// A warp walks its steps in level order (every dependency has a
// lower level, so the lowest unfinished step can always proceed; all CTAs are
// co-resident by cooperative launch).  Per dependency term the analysis
// stores a 32-bit code, kind in bits 30-31:
//   SHFL(l)   solved by this warp in the previous step by lane l: __shfl_sync
//   SMEM(i)   solved by another warp of this CTA: shared slot i (value-as-flag,
//             slots filled with a NaN sentinel at kernel start, never reused)
//   GLOB(g)   solved by another CTA: global mailbox g (value-as-flag; two
//             mailbox arrays swap roles every solve -- device epoch -- and each
//             CTA re-arms its own range of the idle one)
//   NONE      padding (payload p > 0: the row's terms are in overflow list p-1)
//
// Row arithmetic = the paper's sweep with FMAs in STORAGE order:
//   s = b(i); s = fma(-a_k, x(j_k), s) for k in CSR order; x(i) = s * (1/d(i))
// -- the same sequence as SELF's thread-per-row rows and every multi-RHS
// kernel, so results are run-to-run bitwise reproducible and equal across
// algorithms that share it (reading Q8).
//
// One compute warp per tile; nothing on its per-step critical chain
// (shuffle -> select -> 3 FMA -> multiply) waits on global memory:
//   records   (codes, row ids, coefficients, publication targets): TMA bulk
//             copies into per-warp rings DC / DF blocks ahead (no L2 prefetch:
//             see SPTRSV_BLOCK_L2PF)
//   b(row)    cp.async gathers into a per-warp ring DG steps ahead
//   EXT       values of other warps / CTAs: shared-slot loads at the top of
//             the step (cluster peers store into them over DSMEM; values from
//             other clusters are copied in by kNf fetcher warps per compute
//             warp, which poll the global mailboxes)
// A value still holding the sentinel when its step comes is re-polled (the
// only wait).  A per-solve watchdog (timeout_ns) turns a hung wait into
// SPTRSV_ERR_TIMEOUT via sptrsv_get_solve_status instead of a hung GPU.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "internal.h"

namespace sptrsv {
namespace {

// ---------------------------------------------------------------- term codes
// A term code is a 32-bit word.  SHFL terms are the source lane itself
// (0..31), so `code < 32` decides SHFL in one compare and the code is the
// __shfl_sync lane operand.  Other kinds carry the kind in bits 30-31:
//   0 with payload 32      NONE (padding term)
//   0 with payload 33 + o  the row's terms are in overflow list o
//   2 (SMEM) slot index, 3 (GLOB) mailbox index (< 2^30)
constexpr unsigned kKNone = 0u, kKSmem = 2u, kKGlob = 3u;
constexpr int32_t kNoneCode = 32, kOvfBase = 33;
__host__ __device__ inline int32_t mk_code(unsigned kind, unsigned payload) {
    return (int32_t)((kind << 30) | (payload & 0x3FFFFFFFu));
}
__host__ __device__ inline unsigned code_kind(int32_t c) { return (unsigned)c >> 30; }
__host__ __device__ inline int code_idx(int32_t c) { return c & 0x3FFFFFFF; }
__host__ __device__ inline bool code_shfl(int32_t c) { return (unsigned)c < 32u; }
constexpr int32_t kOvfEnd = -1;          // overflow-list terminator (kind GLOB, payload all ones)
constexpr int kSH = 3;                   // terms per record row

// ---------------------------------------------------------------- records
// Two streams per (warp, step), SoA over 32 lanes, 16-byte aligned parts:
//   ctl  int4 {code0, code1, code2, row}[32]                               512 B
//        row: -1 on padding lanes
//   coef T = double: double2 {a0, a1}[32] | double2 {a2, 1/d}[32] | int4 pub[32]   1536 B
//        T = float : float4 {a0, a1, a2, 1/d}[32] | int4 pub[32]                    1024 B
//        pub = {shared slot, mailbox, remote 0, remote 1} (-1: none); remote =
//        rank << 24 | slot: a shared slot of another CTA of the cluster (DSMEM)
// The control stream is read further ahead (b gathers, GLOB prefetch) than
// the coefficients, so it has the deeper ring.  Every warp's steps are padded
// to a multiple of UNR with empty steps (no bounds checks in the loop).
constexpr int kCtlBytes = 512;
template <typename T> struct Coef;
template <> struct Coef<double> {
    static constexpr int BYTES = 1536, PUB = 1024;
    double a0, a1, a2, invd;
    __device__ __forceinline__ void load(const unsigned char *r, int lane) {
        const double2 c0 = reinterpret_cast<const double2 *>(r)[lane];
        const double2 c1 = reinterpret_cast<const double2 *>(r + 512)[lane];
        a0 = c0.x; a1 = c0.y; a2 = c1.x; invd = c1.y;
    }
    __device__ static void put(unsigned char *r, int lane, const double (&a)[3], double invd, int4 pub) {
        reinterpret_cast<double2 *>(r)[lane] = make_double2(a[0], a[1]);
        reinterpret_cast<double2 *>(r + 512)[lane] = make_double2(a[2], invd);
        reinterpret_cast<int4 *>(r + PUB)[lane] = pub;
    }
};
template <> struct Coef<float> {
    static constexpr int BYTES = 1024, PUB = 512;
    float a0, a1, a2, invd;
    __device__ __forceinline__ void load(const unsigned char *r, int lane) {
        const float4 c = reinterpret_cast<const float4 *>(r)[lane];
        a0 = c.x; a1 = c.y; a2 = c.z; invd = c.w;
    }
    __device__ static void put(unsigned char *r, int lane, const float (&a)[3], float invd, int4 pub) {
        reinterpret_cast<float4 *>(r)[lane] = make_float4(a[0], a[1], a[2], invd);
        reinterpret_cast<int4 *>(r + PUB)[lane] = pub;
    }
};

constexpr int kBuckets = kTprMax + 2;
__device__ __forceinline__ uint32_t bucket_of(int deps) { return deps > kTprMax ? 0u : (uint32_t)(kTprMax + 1 - deps); }

// ---------------------------------------------------------------- pipeline shape
// b(row) DG steps ahead goes to shared memory by cp.async, one commit group
// per step, so `cp.async.wait_group DG-1` waits for exactly the oldest step's
// load (register-ring loads would share counting scoreboards and wait for the
// newest ones too).  Values from other CTAs reach shared slots through the
// fetcher warps or DSMEM stores, so a step only reads shared memory: records
// two steps ahead (stage registers), EXT slots at the top of the step.  The
// next step's shuffles are issued right after a step's value, before its
// publication stores (whose addresses are computed ahead).  SHFL and NONE codes (< 32, 32) address
// the zero slots, so the EXT read of every term is one unconditional LDS.
// Per-step / publication timestamps (tools/block_trace2.py, crit_path.py) are
// compiled only into development builds: python tools/build_variant.py trace
// -DSPTRSV_BLOCK_TRACE=1 (they cost ~10% of a step in the release loop).
#ifndef SPTRSV_BLOCK_TRACE
#define SPTRSV_BLOCK_TRACE 0
#endif
// L2 prefetch of the record streams DP blocks ahead (cp.async.bulk.prefetch):
// off -- the TMA ring lookahead (DC = 7 blocks, ~28 steps) already covers the
// DRAM latency, and every bulk operation costs the SM's TMA issue path: without
// the prefetches one tile steps at 129 instead of 144 ns per level, cfg2 148.6
// instead of 157.7 us (profiles/bench_r2d.json).
#ifndef SPTRSV_BLOCK_L2PF
#define SPTRSV_BLOCK_L2PF 0
#endif
// EXT values (shared slots) read at the top of their own step instead of one
// step ahead: a consumer that has caught up with its producer finds the value
// landed more often (the LDS overlaps the step's shuffles)
#ifndef SPTRSV_BLOCK_EXT_LATE
#define SPTRSV_BLOCK_EXT_LATE 1
#endif
// Prologue stagger: a warp whose first row is at level L0 issues its ring
// prologue max(0, L0 * STAGGER_NS - STAGGER_MARGIN) ns after kernel entry, so
// the origin tile's first records are not queued behind every warp's (0: off)
#ifndef SPTRSV_BLOCK_STAGGER_NS
#define SPTRSV_BLOCK_STAGGER_NS 100
#endif
#ifndef SPTRSV_BLOCK_STAGGER_CAP
#define SPTRSV_BLOCK_STAGGER_CAP 16000
#endif
#ifndef SPTRSV_BLOCK_STAGGER_MARGIN
#define SPTRSV_BLOCK_STAGGER_MARGIN 4000
#endif
// The next step's shuffles issued right after this step's value (before its
// publication stores, whose addresses are computed ahead of the chain)
#ifndef SPTRSV_BLOCK_EARLY_SHFL
#define SPTRSV_BLOCK_EARLY_SHFL 1
#endif
// the idle mailbox array re-armed at the end of a solve (for the next one)
// instead of at its start (where the stores meet every warp's prologue)
#ifndef SPTRSV_BLOCK_REARM_END
#define SPTRSV_BLOCK_REARM_END 1
#endif
// Development builds with bounds checks of every record-driven index (shared
// slot, mailbox, cluster rank, row): a violation prints and traps.  Stands in
// for compute-sanitizer where the tool is not available
// (python tools/build_variant.py check -DSPTRSV_BLOCK_CHECK=1).
#ifndef SPTRSV_BLOCK_CHECK
#define SPTRSV_BLOCK_CHECK 0
#endif
#define SPTRSV_BCHECK(cond, what, v)                                                                             \
    do {                                                                                                         \
        if (SPTRSV_BLOCK_CHECK && !(cond)) {                                                                     \
            printf("k_block bounds check failed: %s = %d (block %d thread %d)\n", what, (int)(v), blockIdx.x,  \
                   threadIdx.x);                                                                                \
            __trap();                                                                                            \
        }                                                                                                        \
    } while (0)
#ifndef SPTRSV_BLOCK_UB
#define SPTRSV_BLOCK_UB 4
#define SPTRSV_BLOCK_DG 16
#define SPTRSV_BLOCK_DP 12
#endif
constexpr int UB = SPTRSV_BLOCK_UB;    // steps per TMA block
constexpr int NCB = 8, DC = 7;         // control ring (blocks) / TMA lookahead (blocks)
constexpr int NFB = 4, DF = 3;         // coefficient ring (blocks) / TMA lookahead (blocks)
constexpr int DP = SPTRSV_BLOCK_DP;    // L2 prefetch lookahead (blocks), both streams
constexpr int DG = SPTRSV_BLOCK_DG;    // b(row) loads in flight (steps): cp.async landing ring
#ifndef SPTRSV_BLOCK_UNR
#define SPTRSV_BLOCK_UNR 8
#endif
constexpr int UNR = SPTRSV_BLOCK_UNR;   // main-loop unroll = per-warp step padding
constexpr int XB = (DG + 1) / UB + 2;  // blocks staged past a warp's last step (lookahead)
constexpr int kPadSteps = (XB + 1) * UB;   // stream padding past the last warp
// fetcher warps per compute warp (each polls every kNf-th block of 32 items)
#ifndef SPTRSV_BLOCK_NF
#define SPTRSV_BLOCK_NF 2
#endif
constexpr int kNf = SPTRSV_BLOCK_NF;

constexpr int kZeroSlots = 64;         // shared slots 0..63 hold 0.0: the EXT read of a non-EXT term
static_assert(NCB > DC && NFB > DF && DG % UNR == 0 && UNR % UB == 0, "ring shapes");
static_assert((DG + 1 + UB - 1) / UB + 2 <= DC, "control records must land before their b gather");
static_assert((NCB * UB) % UNR == 0 && (NFB * UB) % UNR == 0, "ring offsets advance by whole iterations");

// per compute warp: control ring, coefficient ring, b landing [DG][32], barriers
template <typename T>
__host__ __device__ constexpr size_t warp_smem_bytes() {
    return ((size_t)NCB * UB * kCtlBytes + (size_t)NFB * UB * Coef<T>::BYTES + (size_t)DG * 32 * sizeof(T) +
            8 * (NCB + NFB) + 127) / 128 * 128;
}

// ---------------------------------------------------------------- build kernels
// natural-order CSR of the referenced strict triangle, from the chunk layout
template <typename T>
__global__ void k_tri_fill(int nchunks, const ChunkDesc *__restrict__ chunks, const int32_t *__restrict__ perm,
                           const int32_t *__restrict__ ecol, const T *__restrict__ eval,
                           const int32_t *__restrict__ tri_ptr, int32_t *__restrict__ tri_col, T *__restrict__ tri_val) {
    const int lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < nchunks; c += nwarps) {
        const ChunkDesc cd = chunks[c];
        const int width = chunk_width(cd.meta);
        if (!chunk_wpr(cd.meta)) {
            if (lane < chunk_nrows(cd.meta)) {
                const int row = perm[cd.pos + lane];
                const int base = tri_ptr[row];
                for (int k = 0; k < width; ++k) {
                    const int j = ecol[cd.eptr + (int64_t)k * 32 + lane];
                    if (j < 0) break;
                    tri_col[base + k] = j;
                    tri_val[base + k] = eval[cd.eptr + (int64_t)k * 32 + lane];
                }
            }
        } else {
            const int row = perm[cd.pos];
            const int base = tri_ptr[row];
            for (int k = lane; k < width; k += 32) {
                tri_col[base + k] = ecol[cd.eptr + k];
                tri_val[base + k] = eval[cd.eptr + k];
            }
        }
    }
}

// grid hypothesis check: every dependency must be a 3x3x3 neighbour
__global__ void k_grid_check(int n, int nx, int ny, const int32_t *__restrict__ tri_ptr,
                             const int32_t *__restrict__ tri_col, unsigned *bad) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int xi = i % nx, yi = (i / nx) % ny, zi = i / (nx * ny);
    bool ok = true;
    for (int k = tri_ptr[i]; k < tri_ptr[i + 1]; ++k) {
        const int j = tri_col[k];
        const int xj = j % nx, yj = (j / nx) % ny, zj = j / (nx * ny);
        ok &= abs(xi - xj) <= 1 && abs(yi - yj) <= 1 && abs(zi - zj) <= 1;
    }
    if (!ok) atomicAdd(bad, 1u);
}

// (x, y) tiles of tw x th columns; CTA = wx x wy tiles; unit = cta * wpc + warp.
// CTAs are numbered by clusters of csx x csy CTAs (rank = position inside).
// UPPER numbers the CTAs backwards so that every dependency points to a
// lower-numbered CTA in both cases.
__global__ void k_part_tiles(int n, int nx, int ny, int tw, int th, int wx, int wy, int cxn, int K, int upper,
                             int csx, int csy, int32_t *unit) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int x = i % nx, y = (i / nx) % ny;
    const int txi = x / tw, tyi = y / th;
    const int cx = txi / wx, cy = tyi / wy;
    int cta = ((cy / csy) * (cxn / csx) + cx / csx) * (csx * csy) + (cy % csy) * csx + cx % csx;
    int w = (tyi % wy) * wx + (txi % wx);
    if (upper) {
        cta = K - 1 - cta;
        w = wx * wy - 1 - w;
    }
    unit[i] = cta * (wx * wy) + w;
}

__global__ void k_part_natural(int n, int U, int uplo, int32_t *unit) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int t = uplo == SPTRSV_LOWER ? i : n - 1 - i;
    unit[i] = (int)((int64_t)t * U / n);
}

__global__ void k_unit_keys(int n, int nlev, const int32_t *unit, const int32_t *lev, const int32_t *dp,
                            uint32_t *keys) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) keys[i] = ((uint32_t)unit[i] * (uint32_t)nlev + (uint32_t)lev[i]) * kBuckets + bucket_of(dp[i]);
}

// head flags of groups (new (unit, level)); inverse permutation
__global__ void k_heads(const uint32_t *skeys, const int32_t *bperm, int n, int32_t *head, int32_t *pos) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const uint32_t s = skeys[p] / kBuckets;
    head[p] = (p == 0 || skeys[p - 1] / kBuckets != s) ? 1 : 0;
    pos[bperm[p]] = p;
}

__global__ void k_group_start(const int32_t *head, const int32_t *gid, int n, int ngroups, int32_t *gp0) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n && head[p]) gp0[gid[p]] = p;
    if (p == 0) gp0[ngroups] = n;
}

__global__ void k_group_sub(const int32_t *gp0, int ngroups, int32_t *nsub) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < ngroups) nsub[g] = (gp0[g + 1] - gp0[g] + 31) / 32;
    if (g == ngroups) nsub[g] = 0;
}

// per group: its 32-row steps (first position, rows); unit of each step
__global__ void k_steps(const int32_t *gp0, const int32_t *sub0, int ngroups, const int32_t *bperm,
                        const int32_t *unit, int2 *steps, int32_t *step_unit) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ngroups) return;
    const int a = gp0[g], e = gp0[g + 1];
    int s = sub0[g];
    const int u = unit[bperm[a]];
    for (int p0 = a; p0 < e; p0 += 32, ++s) {
        steps[s] = make_int2(p0, min(32, e - p0));
        step_unit[s] = u;
    }
}

__global__ void k_unit_step0(const int32_t *step_unit, int nsteps, int U, int32_t *unit_step0) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < nsteps && (s == 0 || step_unit[s - 1] != step_unit[s])) {
        const int uprev = (s == 0) ? -1 : step_unit[s - 1];
        for (int uu = uprev + 1; uu <= step_unit[s]; ++uu) unit_step0[uu] = s;
    }
    if (s == nsteps - 1)
        for (int uu = step_unit[s] + 1; uu <= U; ++uu) unit_step0[uu] = nsteps;
}

// position -> step
__global__ void k_pos_step(const int32_t *head, const int32_t *gid, const int32_t *gp0, const int32_t *sub0, int n,
                           int32_t *step_of) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int g = gid[p] + head[p] - 1;
    step_of[p] = sub0[g] + (p - gp0[g]) / 32;
}

// first position of every CTA (positions are sorted by unit, units by CTA)
__global__ void k_cta_p0(int K, int wpc, int nsteps, int n, const int32_t *unit_step0, const int2 *steps,
                         int32_t *cta_p0) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c > K) return;
    const int s = unit_step0[min(c, K) * wpc];
    cta_p0[c] = s < nsteps ? steps[s].x : n;
}

// Dependency classes: a dependency solved by the same warp in the previous
// step is SHFL; one solved by another warp of the CTA is read from a shared
// slot its producer writes (need bit 0); every other one is CROSS: its
// producer publishes it to a global mailbox (bit 1) and the consumer CTA's
// fetcher copies it into a shared slot (GLOB in the GL fallback).  noslot:
// that CTA's slots overflowed -> its intra-CTA dependencies are CROSS too.
// icnt[pos]: CROSS dependencies of the row at solve position pos.
__device__ __forceinline__ bool dep_shfl(int ui, int si, int uj, int sj) { return uj == ui && sj == si - 1; }
__global__ void k_need(int n, int wpc, const int32_t *__restrict__ tri_ptr, const int32_t *__restrict__ tri_col,
                       const int32_t *__restrict__ unit, const int32_t *__restrict__ pos,
                       const int32_t *__restrict__ step_of, const unsigned char *__restrict__ noslot, int32_t *need,
                       int32_t *icnt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) icnt[n] = 0;
    if (i >= n) return;
    const int ui = unit[i], pi = pos[i], si = step_of[pi];
    const bool ns = noslot[ui / wpc] != 0;
    int cross = 0;
    for (int k = tri_ptr[i]; k < tri_ptr[i + 1]; ++k) {
        const int j = tri_col[k];
        const int uj = unit[j], pj = pos[j];
        if (dep_shfl(ui, si, uj, step_of[pj])) continue;
        if (uj / wpc == ui / wpc && !ns) atomicOr(&need[pj], 1);
        else ++cross;
    }
    icnt[pi] = cross;
}

// CROSS dependencies, numbered q = iptr[pos] + r (r-th CROSS dependency of the
// row in storage order).  Each gets a shared slot of the consumer CTA (after
// its intra slots).  Delivery: the producer stores into it directly over
// DSMEM when both CTAs are in one cluster (<= 2 such targets per producer,
// rt[pos]); otherwise the producer publishes a mailbox (need bit 1) and the
// consumer CTA's fetcher copies it (an inbound item).  GL: every CROSS
// dependency polls the mailbox itself (no slot).
__global__ void k_cross(int n, int nlev, int wpc, int cs, int gl, const int32_t *__restrict__ bperm,
                        const int32_t *__restrict__ tri_ptr, const int32_t *__restrict__ tri_col,
                        const int32_t *__restrict__ unit, const int32_t *__restrict__ pos,
                        const int32_t *__restrict__ step_of, const int32_t *__restrict__ lev,
                        const int32_t *__restrict__ slot_scan, const int32_t *__restrict__ cta_p0,
                        const int32_t *__restrict__ iptr, int32_t *islot, int32_t *need, int32_t *rtc, int2 *rt,
                        unsigned char *fetch, uint32_t *ikey, int32_t *iprod) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int i = bperm[p];
    const int ui = unit[i], si = step_of[p], cc = ui / wpc;
    int q = iptr[p];
    const int intra = slot_scan[cta_p0[cc + 1]] - slot_scan[cta_p0[cc]];
    const int q0 = iptr[cta_p0[cc]];
    for (int k = tri_ptr[i]; k < tri_ptr[i + 1]; ++k) {
        const int j = tri_col[k];
        const int uj = unit[j], pj = pos[j], pc = uj / wpc;
        if (dep_shfl(ui, si, uj, step_of[pj]) || pc == cc) continue;    // (no noslot CTA outside GL)
        const int slot = kZeroSlots + intra + (q - q0);
        islot[q] = slot;
        bool f = true;
        if (!gl && cs > 1 && pc / cs == cc / cs) {
            const int r = atomicAdd(&rtc[pj], 1);
            if (r < 2) {
                const int code = ((cc % cs) << 24) | slot;
                if (r == 0) rt[pj].x = code;
                else rt[pj].y = code;
                f = false;
            }
        }
        if (f) atomicOr(&need[pj], 2);
        fetch[q] = f && !gl;
        ikey[q] = (uint32_t)ui * (uint32_t)nlev + (uint32_t)lev[i];      // (consumer warp, level)
        iprod[q] = pj;
        ++q;
    }
}

// GL fallback with noslot CTAs: their intra-CTA dependencies use mailboxes too
__global__ void k_need_gl(int n, int wpc, const int32_t *__restrict__ tri_ptr, const int32_t *__restrict__ tri_col,
                          const int32_t *__restrict__ unit, const int32_t *__restrict__ pos,
                          const int32_t *__restrict__ step_of, const unsigned char *__restrict__ noslot, int32_t *need) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int ui = unit[i], pi = pos[i], si = step_of[pi];
    const bool ns = noslot[ui / wpc] != 0;
    for (int k = tri_ptr[i]; k < tri_ptr[i + 1]; ++k) {
        const int j = tri_col[k];
        const int uj = unit[j], pj = pos[j];
        if (dep_shfl(ui, si, uj, step_of[pj])) continue;
        if (uj / wpc != ui / wpc || ns) atomicOr(&need[pj], 2);
    }
}

__global__ void k_flag_i32(int nq, const unsigned char *f, int32_t *out) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < nq) out[q] = f[q];
    if (q == nq) out[q] = 0;
}

// compact the fetched CROSS dependencies into items (key, mailbox, slot)
__global__ void k_item_compact(int nq, const unsigned char *fetch, const int32_t *fscan, const uint32_t *ikey,
                               const int32_t *iprod, const int32_t *islot, const int32_t *g_scan, uint32_t *key,
                               int2 *item) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq || !fetch[q]) return;
    const int o = fscan[q];
    key[o] = ikey[q];
    item[o] = make_int2(g_scan[iprod[q]], islot[q]);
}

__global__ void k_item_gather(int nitems, const int32_t *perm, const int2 *item, int2 *fitems) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o < nitems) fitems[o] = item[perm[o]];
}

// first item of every warp in the (warp, level)-sorted item list
__global__ void k_item_ptr(int nitems, int K, int nlev, const uint32_t *skey, int32_t *fptr) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o > nitems) return;
    const int c1 = o < nitems ? (int)(skey[o] / (uint32_t)nlev) : K;
    const int c0 = o > 0 ? (int)(skey[o - 1] / (uint32_t)nlev) : -1;
    for (int c = c0 + 1; c <= c1; ++c) fptr[c] = o;
}

__global__ void k_need_bits(int n, const int32_t *need, int bit, int32_t *out) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) out[p] = (need[p] >> bit) & 1;
    if (p == n) out[p] = 0;
}

// overflow-list length by position: rows with more than kSH terms (+ terminator)
__global__ void k_ovf_count(int n, const int32_t *bperm, const int32_t *dp, int32_t *cnt) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) {
        const int d = dp[bperm[p]];
        cnt[p] = d > kSH ? d + 1 : 0;
    }
    if (p == n) cnt[p] = 0;
}

// per CTA: number of shared slots it needs (intra-CTA, + inbound if iptr)
__global__ void k_cta_slots(int K, const int32_t *cta_p0, const int32_t *slot_scan, const int32_t *iptr, int32_t *cnt) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < K)
        cnt[c] = slot_scan[cta_p0[c + 1]] - slot_scan[cta_p0[c]] + (iptr ? iptr[cta_p0[c + 1]] - iptr[cta_p0[c]] : 0);
}

// mailbox range of every CTA
__global__ void k_cta_g0(int K, const int32_t *cta_p0, const int32_t *g_scan, int32_t *g0) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c <= K) g0[c] = g_scan[cta_p0[c]];
}

// every record of both streams = an empty step (all lanes padding)
template <typename T>
__global__ void k_pad_fill(int64_t nrec, unsigned char *__restrict__ ctl, unsigned char *__restrict__ coef) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nrec * 32) return;
    const int s = (int)(t >> 5), lane = (int)(t & 31);
    reinterpret_cast<int4 *>(ctl + (size_t)s * kCtlBytes)[lane] = make_int4(kNoneCode, kNoneCode, kNoneCode, -1);
    const T a[kSH] = {T(0), T(0), T(0)};
    Coef<T>::put(coef + (size_t)s * Coef<T>::BYTES, lane, a, T(0), make_int4(-1, -1, -1, -1));
}

// padded step index of every step: warp u's steps start at pstart[u]
__global__ void k_pad_map(int nsteps, const int32_t *step_unit, const int32_t *unit_step0, const int32_t *pstart,
                          int32_t *pmap) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nsteps) return;
    const int u = step_unit[s];
    pmap[s] = pstart[u] + (s - unit_step0[u]);
}

// level of every warp's first row: the smallest level among the rows of its
// first non-empty step (0 for a warp without rows)
__global__ void k_unit_lev0(int U, const int32_t *unit_step0, const unsigned char *ctl, const int32_t *lev,
                            int32_t *lev0) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= U) return;
    int best = 0x7fffffff;
    for (int t = unit_step0[u]; t < unit_step0[u + 1] && best == 0x7fffffff; ++t) {
        const int4 *c = reinterpret_cast<const int4 *>(ctl + (size_t)t * kCtlBytes);
        for (int l = 0; l < 32; ++l)
            if (c[l].w >= 0) best = min(best, lev[c[l].w]);
    }
    lev0[u] = best == 0x7fffffff ? 0 : best;
}
__global__ void k_pad_count(int U, const int32_t *unit_step0, int32_t *cnt) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u < U) cnt[u] = (unit_step0[u + 1] - unit_step0[u] + UNR - 1) / UNR * UNR;
    if (u == U) cnt[u] = 0;
}

// one thread per (step, lane): that lane's entries of both streams, at the
// step's padded position
template <typename T>
__global__ void k_rec_fill(int nsteps, int wpc, const int2 *__restrict__ steps, const int32_t *__restrict__ pmap,
                           const int32_t *__restrict__ bperm, const int32_t *__restrict__ pos,
                           const int32_t *__restrict__ step_of, const int32_t *__restrict__ unit,
                           const int32_t *__restrict__ tri_ptr, const int32_t *__restrict__ tri_col,
                           const T *__restrict__ tri_val, const T *__restrict__ invd_row, int unit_diag,
                           const unsigned char *__restrict__ noslot, const int32_t *__restrict__ need,
                           const int32_t *__restrict__ slot_scan, const int32_t *__restrict__ g_scan,
                           const int32_t *__restrict__ cta_p0, const int32_t *__restrict__ ovf_ptr,
                           const int32_t *__restrict__ iptr, const int32_t *__restrict__ islot, int gl,
                           const int2 *__restrict__ rt,
                           unsigned char *__restrict__ ctl, unsigned char *__restrict__ coef,
                           int32_t *__restrict__ ovf_code, T *__restrict__ ovf_val) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)nsteps * 32) return;
    const int s = (int)(t >> 5), lane = (int)(t & 31);
    const int2 st = steps[s];
    if (lane >= st.y) return;                       // padding lane: k_pad_fill's empty entry stays
    const size_t ps = (size_t)pmap[s];
    unsigned char *cr = ctl + ps * kCtlBytes;
    unsigned char *fr = coef + ps * Coef<T>::BYTES;
    T a[kSH] = {T(0), T(0), T(0)};
    const int p = st.x + lane;
    const int i = bperm[p];
    const int ui = unit[i], cta = ui / wpc;
    const bool ns = noslot[cta] != 0;
    const int si = step_of[p];
    const int ka = tri_ptr[i], ke = tri_ptr[i + 1];
    const int slot_base = slot_scan[cta_p0[cta]];
    int32_t code[kSH] = {kNoneCode, kNoneCode, kNoneCode};
    const bool ovf = ke - ka > kSH;
    int o = ovf ? ovf_ptr[p] : 0;
    if (ovf) code[0] = kOvfBase + o;
    int item = gl ? 0 : iptr[p];
    for (int k = ka, q = 0; k < ke; ++k, ++q) {
        const int j = tri_col[k];
        const int uj = unit[j], pj = pos[j];
        int32_t c;
        if (dep_shfl(ui, si, uj, step_of[pj])) c = pj - steps[si - 1].x;                  // SHFL: source lane
        else if (uj / wpc == cta && !ns) c = mk_code(kKSmem, (unsigned)(kZeroSlots + slot_scan[pj] - slot_base));
        else if (gl) c = mk_code(kKGlob, (unsigned)g_scan[pj]);
        else c = mk_code(kKSmem, (unsigned)islot[item++]);                                // inbound slot
        if (ovf) {
            ovf_code[o] = c;
            ovf_val[o] = tri_val[k];
            ++o;
        } else {
            code[q] = c;
            a[q] = tri_val[k];
        }
    }
    if (ovf) {
        ovf_code[o] = kOvfEnd;
        ovf_val[o] = T(0);
    }
    const int nd = need[p];
    reinterpret_cast<int4 *>(cr)[lane] = make_int4(code[0], code[1], code[2], i);
    const int2 r2 = rt[p];
    Coef<T>::put(fr, lane, a, unit_diag ? T(1) : invd_row[i],
                 make_int4((nd & 1) ? kZeroSlots + slot_scan[p] - slot_base : -1, (nd & 2) ? g_scan[p] : -1, r2.x, r2.y));
}

// new values into the records (NEXT-2 value update): every real lane of every
// step keeps its codes and publication targets; its coefficients (or its
// overflow list's values) and 1/d are re-read in storage order
template <typename T>
__global__ void k_rec_refill(int64_t npad, const unsigned char *__restrict__ ctl, unsigned char *__restrict__ coef,
                             const int32_t *__restrict__ tri_ptr, const T *__restrict__ tri_val,
                             const T *__restrict__ invd_row, int unit_diag, T *__restrict__ ovf_val) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= npad * 32) return;
    const int64_t st = t >> 5;
    const int lane = (int)(t & 31);
    const int4 c = reinterpret_cast<const int4 *>(ctl + (size_t)st * kCtlBytes)[lane];
    if (c.w < 0) return;                               // padding lane
    const int row = c.w, ka = tri_ptr[row], nd = tri_ptr[row + 1] - ka;
    T a[kSH] = {T(0), T(0), T(0)};
    if (nd > kSH) {
        const int o = c.x - kOvfBase;
        for (int q = 0; q < nd; ++q) ovf_val[o + q] = tri_val[ka + q];
    } else {
        for (int q = 0; q < nd; ++q) a[q] = tri_val[ka + q];
    }
    unsigned char *fr = coef + (size_t)st * Coef<T>::BYTES;
    const int4 pub = reinterpret_cast<const int4 *>(fr + Coef<T>::PUB)[lane];
    Coef<T>::put(fr, lane, a, unit_diag ? T(1) : invd_row[row], pub);
}

template <typename T>
__global__ void k_fill_sentinel(T *p, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (; i < n; i += stride) p[i] = Sentinel<T>::value();
}

// ------------------------------------------------------------------ solve
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ double lds_volatile(const double *p) {
    double v;
    asm volatile("ld.relaxed.cluster.shared::cta.f64 %0, [%1];" : "=d"(v) : "r"(smem_u32(p)));
    return v;
}
__device__ __forceinline__ float lds_volatile(const float *p) {
    float v;
    asm volatile("ld.relaxed.cluster.shared::cta.f32 %0, [%1];" : "=f"(v) : "r"(smem_u32(p)));
    return v;
}
// predicated value-as-flag loads (return 0 where !pred)
__device__ __forceinline__ double ldg_flag_if(const double *p, bool pred) {
    unsigned long long v = 0;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.relaxed.gpu.global.b64 %0, [%1];\n\t}"
                 : "+l"(v) : "l"(p), "r"((unsigned)pred));
    return __longlong_as_double((long long)v);
}
__device__ __forceinline__ float ldg_flag_if(const float *p, bool pred) {
    unsigned v = 0;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.relaxed.gpu.global.b32 %0, [%1];\n\t}"
                 : "+r"(v) : "l"(p), "r"((unsigned)pred));
    return __uint_as_float(v);
}
__device__ __forceinline__ double lds_flag_if(const double *p, bool pred) {
    unsigned long long v = 0;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.relaxed.cluster.shared::cta.b64 %0, [%1];\n\t}"
                 : "+l"(v) : "r"(smem_u32(p)), "r"((unsigned)pred));
    return __longlong_as_double((long long)v);
}
__device__ __forceinline__ float lds_flag_if(const float *p, bool pred) {
    unsigned v = 0;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.relaxed.cluster.shared::cta.b32 %0, [%1];\n\t}"
                 : "+r"(v) : "r"(smem_u32(p)), "r"((unsigned)pred));
    return __uint_as_float(v);
}
__device__ __forceinline__ void sts_flag(double *p, double v) {
    asm volatile("st.relaxed.cluster.shared::cta.f64 [%0], %1;" ::"r"(smem_u32(p)), "d"(v));
}
__device__ __forceinline__ void sts_flag(float *p, float v) {
    asm volatile("st.relaxed.cluster.shared::cta.f32 [%0], %1;" ::"r"(smem_u32(p)), "f"(v));
}
__device__ __forceinline__ void stg_flag(double *p, double v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"((unsigned long long)__double_as_longlong(v)));
}
__device__ __forceinline__ void stg_flag(float *p, float v) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(__float_as_uint(v)));
}
// base + idx (idx < 2^30 elements): one IMAD.WIDE.U32
template <typename T>
__device__ __forceinline__ T *elem(T *base, int32_t code) {
    T *r;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"((unsigned)code & 0x3FFFFFFFu), "r"((unsigned)sizeof(T)), "l"(base));
    return r;
}

// predicated loads merging into v (v unchanged where !pred)
__device__ __forceinline__ void ldg_flag_into(double &v, const double *p, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.relaxed.gpu.global.f64 %0, [%1];\n\t}"
                 : "+d"(v) : "l"(p), "r"((unsigned)pred));
}
__device__ __forceinline__ void ldg_flag_into(float &v, const float *p, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.relaxed.gpu.global.f32 %0, [%1];\n\t}"
                 : "+f"(v) : "l"(p), "r"((unsigned)pred));
}
__device__ __forceinline__ void lds_flag_into(double &v, const double *p, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.relaxed.cluster.shared::cta.f64 %0, [%1];\n\t}"
                 : "+d"(v) : "r"(smem_u32(p)), "r"((unsigned)pred));
}
__device__ __forceinline__ void lds_flag_into(float &v, const float *p, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.relaxed.cluster.shared::cta.f32 %0, [%1];\n\t}"
                 : "+f"(v) : "r"(smem_u32(p)), "r"((unsigned)pred));
}
__device__ __forceinline__ unsigned hi_word(double v) { return (unsigned)((unsigned long long)__double_as_longlong(v) >> 32); }
__device__ __forceinline__ unsigned hi_word(float v) { return __float_as_uint(v); }
template <typename T> __device__ __forceinline__ unsigned sent_hi();
template <> __device__ __forceinline__ unsigned sent_hi<double>() { return (unsigned)(Sentinel<double>::bits >> 32); }
template <> __device__ __forceinline__ unsigned sent_hi<float>() { return Sentinel<float>::bits; }

// the sentinel test on the high word only (finite values and arithmetic NaNs
// never carry the sentinel's high word)
__device__ __forceinline__ bool is_sent(double v) {
    return (unsigned)(__double_as_longlong(v) >> 32) == (unsigned)(Sentinel<double>::bits >> 32);
}
__device__ __forceinline__ bool is_sent(float v) { return Sentinel<float>::is(v); }

struct BlockArgs {
    const int32_t *unit_step0;    // [U+1] padded first step of every warp (multiples of UNR)
    const int32_t *unit_lev0;     // [U] level of every warp's first row
    const unsigned char *ctl;     // control stream [npad + kPadSteps][kCtlBytes]
    const unsigned char *coef;    // coefficient stream [npad + kPadSteps][Coef<T>::BYTES]
    const int32_t *cta_g0;        // [K+1] mailbox range of every CTA (values it publishes)
    const int2 *fitems;           // inbound items {mailbox, shared slot}, by (CTA, level)
    const int32_t *fptr;          // [K+1] inbound item range of every CTA
    const int32_t *ovf_code;
    const void *ovf_val;
    void *gmb;                    // [2][G] mailboxes
    unsigned *ctr;                // [0] solve epoch, [1] finished CTAs
    unsigned *status;             // [0] epoch + 1 of the last solve that timed out
    unsigned long long *trace;    // debug: per-warp %globaltimer at block starts (NULL: off)
    int trace_cap;
    unsigned long long *ftrace;   // debug: %globaltimer of every inbound item's delivery (NULL: off)
    unsigned long long *ptrace;   // debug: %globaltimer of every mailbox publication, by mailbox (NULL: off)
    const void *b;
    void *x;
    int G, nslots;                // nslots: shared slots per CTA including the kZeroSlots
    int n, cs;                    // rows, CTAs per cluster (bounds checks of development builds)
    unsigned long long timeout_ns;
};

// Watchdog of one wait: true once this solve is given up (this wait exceeded
// timeout_ns, or another one already did).
struct Watch {
    unsigned long long t0;
    unsigned it;
    __device__ bool expired(unsigned *status, unsigned long long timeout_ns, unsigned tag) {
        if (timeout_ns == 0) {               // test hook: give up the first wait
            st_relaxed(reinterpret_cast<int *>(status), (int)tag);
            return true;
        }
        if ((++it & 255u) != 0) return false;
        if (it == 256u) t0 = gtimer();
        if (ld_relaxed(reinterpret_cast<const int *>(status)) == (int)tag) return true;
        if (gtimer() - t0 > timeout_ns) {
            st_relaxed(reinterpret_cast<int *>(status), (int)tag);
            return true;
        }
        return false;
    }
};

// Indexed stores / copies predicated on index >= 0 (address and predicate
// computed inside: no branch, no separate predicate materialisation)
__device__ __forceinline__ void st_x(double *base, int k, double v) {         // x(k) = v, cache at L2
    asm volatile("{\n\t.reg .pred q;\n\t.reg .s64 a;\n\tsetp.ge.s32 q, %1, 0;\n\tmad.wide.s32 a, %1, 8, %0;\n\t"
                 "@q st.global.cg.f64 [a], %2;\n\t}" ::"l"(base), "r"(k), "d"(v));
}
__device__ __forceinline__ void st_x(float *base, int k, float v) {
    asm volatile("{\n\t.reg .pred q;\n\t.reg .s64 a;\n\tsetp.ge.s32 q, %1, 0;\n\tmad.wide.s32 a, %1, 4, %0;\n\t"
                 "@q st.global.cg.f32 [a], %2;\n\t}" ::"l"(base), "r"(k), "f"(v));
}
__device__ __forceinline__ void st_mb(double *base, int k, double v) {        // mailbox k (relaxed, gpu scope)
    asm volatile("{\n\t.reg .pred q;\n\t.reg .s64 a;\n\tsetp.ge.s32 q, %1, 0;\n\tmad.wide.s32 a, %1, 8, %0;\n\t"
                 "@q st.relaxed.gpu.global.f64 [a], %2;\n\t}" ::"l"(base), "r"(k), "d"(v));
}
__device__ __forceinline__ void st_mb(float *base, int k, float v) {
    asm volatile("{\n\t.reg .pred q;\n\t.reg .s64 a;\n\tsetp.ge.s32 q, %1, 0;\n\tmad.wide.s32 a, %1, 4, %0;\n\t"
                 "@q st.relaxed.gpu.global.f32 [a], %2;\n\t}" ::"l"(base), "r"(k), "f"(v));
}
__device__ __forceinline__ void st_slot(uint32_t base, int k, double v) {     // shared slot k (volatile)
    asm volatile("{\n\t.reg .pred q;\n\t.reg .u32 a;\n\tsetp.ge.s32 q, %1, 0;\n\tmad.lo.u32 a, %1, 8, %0;\n\t"
                 "@q st.relaxed.cluster.shared::cta.f64 [a], %2;\n\t}" ::"r"(base), "r"(k), "d"(v));
}
__device__ __forceinline__ void st_slot(uint32_t base, int k, float v) {
    asm volatile("{\n\t.reg .pred q;\n\t.reg .u32 a;\n\tsetp.ge.s32 q, %1, 0;\n\tmad.lo.u32 a, %1, 4, %0;\n\t"
                 "@q st.relaxed.cluster.shared::cta.f32 [a], %2;\n\t}" ::"r"(base), "r"(k), "f"(v));
}
// slot read of a term code: SHFL / NONE codes land in the zero slots; SMEM
// codes (kind bits shifted out by the scale) in their slot
__device__ __forceinline__ double ld_code(uint32_t base, int c, double) {
    double v;
    asm volatile("{\n\t.reg .u32 a;\n\tmad.lo.u32 a, %1, 8, %2;\n\tld.relaxed.cluster.shared::cta.f64 %0, [a];\n\t}"
                 : "=d"(v) : "r"(c), "r"(base));
    return v;
}
__device__ __forceinline__ float ld_code(uint32_t base, int c, float) {
    float v;
    asm volatile("{\n\t.reg .u32 a;\n\tmad.lo.u32 a, %1, 4, %2;\n\tld.relaxed.cluster.shared::cta.f32 %0, [a];\n\t}"
                 : "=f"(v) : "r"(c), "r"(base));
    return v;
}
// cp.async of b(k) (k < 0: zero-fill, nothing read)
__device__ __forceinline__ void cp_b(uint32_t dst, const double *base, int k) {
    asm volatile("{\n\t.reg .pred q;\n\t.reg .s64 a;\n\t.reg .u32 z;\n\tsetp.ge.s32 q, %2, 0;\n\t"
                 "mad.wide.s32 a, %2, 8, %1;\n\tselp.u32 z, 8, 0, q;\n\tcp.async.ca.shared.global [%0], [a], 8, z;\n\t}" ::"r"(
                     dst), "l"(base), "r"(k)
                 : "memory");
}
__device__ __forceinline__ void cp_b(uint32_t dst, const float *base, int k) {
    asm volatile("{\n\t.reg .pred q;\n\t.reg .s64 a;\n\t.reg .u32 z;\n\tsetp.ge.s32 q, %2, 0;\n\t"
                 "mad.wide.s32 a, %2, 4, %1;\n\tselp.u32 z, 4, 0, q;\n\tcp.async.ca.shared.global [%0], [a], 4, z;\n\t}" ::"r"(
                     dst), "l"(base), "r"(k)
                 : "memory");
}
// TMA bulk copy issued by one lane (predicate), no branch
__device__ __forceinline__ void tma_if(void *dst, const void *src, uint32_t bytes, uint64_t *bar, bool pred) {
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %4, 0;\n\t"
        "@q mbarrier.arrive.expect_tx.shared::cta.b64 _, [%3], %2;\n\t"
        "@q cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n\t}" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "r"((unsigned)pred)
        : "memory");
}
__device__ __forceinline__ void l2pf_if(const void *src, uint32_t bytes, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q cp.async.bulk.prefetch.L2.global [%0], %1;\n\t}" ::"l"(
                     src), "r"(bytes), "r"((unsigned)pred)
                 : "memory");
}

// EXT value of one term in the GL / OVF instances: shared slot (SMEM),
// mailbox polled directly (GLOB, GL only); 0 for other kinds
template <typename T, bool GL>
__device__ __forceinline__ T ext_load(int32_t c, const T *slots, const T *gm) {
    T v = T(0);
    lds_flag_into(v, slots + code_idx(c), code_kind(c) == kKSmem);
    if (GL) ldg_flag_into(v, elem(gm, c), code_kind(c) == kKGlob);
    return v;
}

// Re-poll the EXT values of a step that are still the sentinel (warp-uniform
// loop; out of line: the common case never gets here).  By value / through
// the kernel parameters: nothing of the caller's state becomes addressable.
template <typename T> struct E3 { T e0, e1, e2; };
template <typename T, bool GL>
__device__ __noinline__ E3<T> repoll(E3<T> e, int c0, int c1, int c2, const BlockArgs *pa, unsigned tag) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int wpc = blockDim.x / (32 * (1 + kNf));
    const T *slots = reinterpret_cast<const T *>(smem_raw + (size_t)wpc * warp_smem_bytes<T>());
    const T *gm = static_cast<const T *>(pa->gmb) + (size_t)((tag - 1u) & 1u) * pa->G;
    Watch wd{0, 0};
    for (;;) {
        const bool p0 = is_sent(e.e0), p1 = is_sent(e.e1), p2 = is_sent(e.e2);
        if (!__any_sync(0xffffffffu, p0 || p1 || p2) || wd.expired(pa->status, pa->timeout_ns, tag)) break;
#if SPTRSV_BLOCK_RSLEEP
        __nanosleep(SPTRSV_BLOCK_RSLEEP);    // dev: spinning warps off the shared-memory pipe
#endif
        if (p0) e.e0 = ext_load<T, GL>(c0, slots, gm);
        if (p1) e.e1 = ext_load<T, GL>(c1, slots, gm);
        if (p2) e.e2 = ext_load<T, GL>(c2, slots, gm);
    }
    return e;
}

// overflow row (> kSH terms): warp-uniform walk of the lists of the lanes
// that have one, in storage order, polling SMEM / GLOB values
template <typename T>
__device__ __noinline__ T ovf_terms(T acc, int o, T xprev, const BlockArgs *pa, unsigned tag) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int wpc = blockDim.x / (32 * (1 + kNf));
    const T *slots = reinterpret_cast<const T *>(smem_raw + (size_t)wpc * warp_smem_bytes<T>());
    const T *gm = static_cast<const T *>(pa->gmb) + (size_t)((tag - 1u) & 1u) * pa->G;
    const int32_t *oc = pa->ovf_code;
    const T *ov = static_cast<const T *>(pa->ovf_val);
    for (;;) {
        const int32_t c = o >= 0 ? oc[o] : kOvfEnd;
        const bool live = c != kOvfEnd;
        if (!__any_sync(0xffffffffu, live)) break;
        const T sh = __shfl_sync(0xffffffffu, xprev, c & 31);
        if (live) {
            const unsigned k = code_shfl(c) ? kKNone : code_kind(c);
            T v = sh;
            if (k == kKSmem || k == kKGlob) {
                Watch w{0, 0};
                for (;;) {
                    v = k == kKSmem ? lds_volatile(slots + code_idx(c)) : ld_relaxed_val(elem(gm, c));
                    if (!is_sent(v) || w.expired(pa->status, pa->timeout_ns, tag)) break;
                }
            }
            acc = fnma(ov[o], v, acc);
            ++o;
        }
    }
    return acc;
}

// The fetchers (kNf warps per compute warp): copy the warp's inbound values
// (written to global mailboxes by CTAs of other clusters) into their shared
// slots, in the order the warp's steps need them.  Fetcher p, lane l owns the
// items 32 p + l + 32 kNf j; it keeps kFw of them polled at once (relaxed
// loads) and refills each window entry as soon as its value arrived (no
// head-of-line blocking).  Two fetchers with one item per lane measured best
// (cfg2 118 vs 130 us with one fetcher of four: a refill then waits for one
// item-list load, not for a round of four polls).
#ifndef SPTRSV_BLOCK_RSLEEP
#define SPTRSV_BLOCK_RSLEEP 0
#endif
#ifndef SPTRSV_BLOCK_FW
#define SPTRSV_BLOCK_FW 1
#endif
#ifndef SPTRSV_BLOCK_FSLEEP
#define SPTRSV_BLOCK_FSLEEP 128
#endif
constexpr int kFw = SPTRSV_BLOCK_FW;
constexpr unsigned kFsleep = SPTRSV_BLOCK_FSLEEP;      // ns between unproductive poll rounds
template <typename T>
__device__ void fetcher(const int2 *items, int f0, int f1, const T *gm, T *slots, unsigned *status,
                        unsigned long long tmo, unsigned tag, unsigned long long *ftrace, int part, int G,
                        int nslots) {
    const int lane = threadIdx.x & 31;
    Watch wd{0, 0};
    int2 d[kFw];
    int id[kFw];
    int nxt = f0 + 32 * part + lane;          // next item of this lane (fetcher part of kNf: items in blocks of 32)
#pragma unroll
    for (int k = 0; k < kFw; ++k) {
        d[k] = nxt < f1 ? items[nxt] : make_int2(-1, 0);
        id[k] = nxt;
        nxt += 32 * kNf;
    }
    for (;;) {
        bool live = false;
#pragma unroll
        for (int k = 0; k < kFw; ++k) live |= d[k].x >= 0;
        if (!__any_sync(0xffffffffu, live)) break;
        T v[kFw];
#pragma unroll
        for (int k = 0; k < kFw; ++k) v[k] = d[k].x >= 0 ? ld_relaxed_val(gm + d[k].x) : T(0);
        bool got = false;
#pragma unroll
        for (int k = 0; k < kFw; ++k)
            if (d[k].x >= 0 && !is_sent(v[k])) {
                SPTRSV_BCHECK(d[k].x < G && d[k].y >= kZeroSlots && d[k].y < nslots, "fetched item", d[k].x);
                st_slot(smem_u32(slots), d[k].y, v[k]);
                if (ftrace != nullptr) ftrace[id[k]] = gtimer();
                d[k] = nxt < f1 ? items[nxt] : make_int2(-1, 0);
                id[k] = nxt;
                nxt += 32 * kNf;
                got = true;
            }
        if (!__any_sync(0xffffffffu, got)) {      // nothing arrived: back off (polls load L2 for everyone)
            if (kFsleep) __nanosleep(kFsleep);
            if (wd.expired(status, tmo, tag)) return;
        }
    }
}

// Record fields of one step (loaded two steps before the step runs)
template <typename T>
struct Stage {
    int4 c;          // term codes, row
    int4 pub;        // shared slot, mailbox, remote targets
    Coef<T> f;
};

// DSMEM store into shared slot (r & 0xFFFFFF) of cluster rank r >> 24 (r >= 0)
__device__ __forceinline__ void st_remote(uint32_t slots, int r, double v) {
    asm volatile("{\n\t.reg .pred q;\n\t.reg .u32 a, ra, rk;\n\tsetp.ge.s32 q, %1, 0;\n\t"
                 "and.b32 a, %1, 0xFFFFFF;\n\tmad.lo.u32 a, a, 8, %0;\n\tshr.u32 rk, %1, 24;\n\t"
                 "@q mapa.shared::cluster.u32 ra, a, rk;\n\t@q st.relaxed.cluster.shared::cluster.f64 [ra], %2;\n\t}" ::"r"(
                     slots), "r"(r), "d"(v)
                 : "memory");
}
__device__ __forceinline__ void st_remote(uint32_t slots, int r, float v) {
    asm volatile("{\n\t.reg .pred q;\n\t.reg .u32 a, ra, rk;\n\tsetp.ge.s32 q, %1, 0;\n\t"
                 "and.b32 a, %1, 0xFFFFFF;\n\tmad.lo.u32 a, a, 4, %0;\n\tshr.u32 rk, %1, 24;\n\t"
                 "@q mapa.shared::cluster.u32 ra, a, rk;\n\t@q st.relaxed.cluster.shared::cluster.f32 [ra], %2;\n\t}" ::"r"(
                     slots), "r"(r), "f"(v)
                 : "memory");
}
// Publication targets of one step with their addresses computed ahead (off
// the chain), and the predicated stores that use them right after the step's
// value is known.
struct PubA {
    uint32_t sa, r0, r1;         // shared slot, DSMEM slots of cluster peers (shared::cluster addresses)
    unsigned ps, p0, p1, pm, px; // predicates (0 / 1)
    const void *mb;              // mailbox
    const void *xp;              // x(row)
};
template <typename T>
__device__ __forceinline__ PubA pub_addr(const int4 &pub, int row, uint32_t slots, T *gm, T *x) {
    PubA P;
    P.ps = pub.x >= 0;
    P.sa = slots + (uint32_t)pub.x * (uint32_t)sizeof(T);
    P.pm = pub.y >= 0;
    P.mb = gm + (P.pm ? pub.y : 0);
    P.p0 = pub.z >= 0;
    P.p1 = pub.w >= 0;
    const uint32_t a0 = slots + (uint32_t)(pub.z & 0xFFFFFF) * (uint32_t)sizeof(T);
    const uint32_t a1 = slots + (uint32_t)(pub.w & 0xFFFFFF) * (uint32_t)sizeof(T);
    const uint32_t k0 = P.p0 ? ((uint32_t)pub.z >> 24) : 0u, k1 = P.p1 ? ((uint32_t)pub.w >> 24) : 0u;
    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(P.r0) : "r"(a0), "r"(k0));
    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(P.r1) : "r"(a1), "r"(k1));
    P.px = row >= 0;
    P.xp = x + (P.px ? row : 0);
    return P;
}
__device__ __forceinline__ void pub_store(const PubA &P, double v, bool cl) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.relaxed.cluster.shared::cta.f64 [%0], %1;\n\t}"
                 ::"r"(P.sa), "d"(v), "r"(P.ps) : "memory");
    if (cl) {
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.relaxed.cluster.shared::cluster.f64 [%0], %1;\n\t}"
                     ::"r"(P.r0), "d"(v), "r"(P.p0) : "memory");
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.relaxed.cluster.shared::cluster.f64 [%0], %1;\n\t}"
                     ::"r"(P.r1), "d"(v), "r"(P.p1) : "memory");
    }
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.relaxed.gpu.global.f64 [%0], %1;\n\t}"
                 ::"l"(P.mb), "d"(v), "r"(P.pm) : "memory");
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.global.cg.f64 [%0], %1;\n\t}"
                 ::"l"(P.xp), "d"(v), "r"(P.px) : "memory");
}
__device__ __forceinline__ void pub_store(const PubA &P, float v, bool cl) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.relaxed.cluster.shared::cta.f32 [%0], %1;\n\t}"
                 ::"r"(P.sa), "f"(v), "r"(P.ps) : "memory");
    if (cl) {
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.relaxed.cluster.shared::cluster.f32 [%0], %1;\n\t}"
                     ::"r"(P.r0), "f"(v), "r"(P.p0) : "memory");
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.relaxed.cluster.shared::cluster.f32 [%0], %1;\n\t}"
                     ::"r"(P.r1), "f"(v), "r"(P.p1) : "memory");
    }
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.relaxed.gpu.global.f32 [%0], %1;\n\t}"
                 ::"l"(P.mb), "f"(v), "r"(P.pm) : "memory");
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.global.cg.f32 [%0], %1;\n\t}"
                 ::"l"(P.xp), "f"(v), "r"(P.px) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// OVF: the plan has rows with more than kSH terms (overflow lists).  GL: the
// plan keeps GLOB terms (mailboxes polled by the consumer itself: shared
// slots did not fit); otherwise every cross-CTA value reaches its consumer
// through the CTA's fetcher warp and a shared slot.  The common instance
// (no OVF, no GL) carries no code for either.
template <typename T, bool UNIT, bool OVF, bool GL, bool CL>
__global__ void __launch_bounds__(128 * (1 + kNf), 1) k_block(const __grid_constant__ BlockArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ unsigned s_epoch;
    constexpr int CB = Coef<T>::BYTES;
    constexpr int CR = NCB * UB, FR = NFB * UB;      // ring lengths (steps), powers of two
    static_assert((CR & (CR - 1)) == 0 && (FR & (FR - 1)) == 0, "power-of-two rings");
    constexpr size_t WS = warp_smem_bytes<T>();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int wpc = blockDim.x / (32 * (1 + kNf));   // compute warps 0..wpc-1; warps wpc + g + wpc p fetch for warp g
#if SPTRSV_BLOCK_TRACE
    const unsigned long long t_entry = gtimer();      // dev: kernel entry (stored at trace[cap - 2])
#endif
    unsigned char *ctlring = smem_raw + (size_t)w * WS;                                // [CR][kCtlBytes]
    unsigned char *coefring = ctlring + (size_t)CR * kCtlBytes;                         // [FR][CB]
    T *bland = reinterpret_cast<T *>(coefring + (size_t)FR * CB);                      // [DG][32]
    uint64_t *cbar = reinterpret_cast<uint64_t *>(bland + DG * 32);                     // [NCB]
    uint64_t *fbar = cbar + NCB;                                                        // [NFB]
    T *slots = reinterpret_cast<T *>(smem_raw + (size_t)wpc * WS);                     // [nslots]
    const uint32_t slots_u32 = smem_u32(slots);
    const T *b = static_cast<const T *>(a.b);
    T *x = static_cast<T *>(a.x);

    for (int i = threadIdx.x; i < a.nslots; i += blockDim.x) slots[i] = i < kZeroSlots ? T(0) : Sentinel<T>::value();
    if (lane == 0 && w < wpc) {
        for (int i = 0; i < NCB + NFB; ++i) mbar_init(&cbar[i], 1);
        fence_mbar_init();
    }
    if (threadIdx.x == 0) s_epoch = (unsigned)ld_relaxed(reinterpret_cast<const int *>(a.ctr));
    if (CL) cluster_sync_all();      // every CTA of the cluster armed its slots before any DSMEM store
    else __syncthreads();
    const unsigned epoch = s_epoch;
    const unsigned tag = epoch + 1u;
    T *gm = static_cast<T *>(a.gmb) + (size_t)(epoch & 1u) * a.G;
    if (!SPTRSV_BLOCK_REARM_END) {   // re-arm this CTA's mailboxes of the idle array (written by the previous solve)
        T *go = static_cast<T *>(a.gmb) + (size_t)((epoch & 1u) ^ 1u) * a.G;
        for (int i = a.cta_g0[blockIdx.x] + threadIdx.x; i < a.cta_g0[blockIdx.x + 1]; i += blockDim.x)
            go[i] = Sentinel<T>::value();
    }

    if (w >= wpc) {
        const int fu = blockIdx.x * wpc + (w - wpc) % wpc;   // the compute warp whose items this warp fetches
        if (!GL) fetcher<T>(a.fitems, a.fptr[fu], a.fptr[fu + 1], gm, slots, a.status, a.timeout_ns, tag,
                          a.ftrace, (w - wpc) / wpc, a.G, a.nslots);
    } else {
    const int u = blockIdx.x * wpc + w;
    const int s0 = a.unit_step0[u], n = a.unit_step0[u + 1] - s0;    // n: a multiple of UNR
    if (n > 0) {
        const int nbx = n / UB + XB;             // blocks staged: this warp's + lookahead past its end
        const unsigned char *gctl = a.ctl + (size_t)s0 * kCtlBytes;
        const unsigned char *gcoef = a.coef + (size_t)s0 * CB;
        unsigned long long *trc = a.trace != nullptr ? a.trace + (size_t)u * a.trace_cap : nullptr;
        const bool l0 = lane == 0;
        const uint32_t bland_u32 = smem_u32(bland) + lane * (uint32_t)sizeof(T);
        auto issue = [&](int kb) {              // lane 0: TMA of both streams' blocks kb+DC / kb+DF, L2 prefetch
            const int kc = kb + DC, kf = kb + DF, kp = kb + DP;
            tma_if(ctlring + (size_t)(kc % NCB) * UB * kCtlBytes, gctl + (size_t)kc * UB * kCtlBytes,
                   UB * kCtlBytes, &cbar[kc % NCB], l0 && kc >= 0 && kc < nbx);
            tma_if(coefring + (size_t)((kf + NFB) % NFB) * UB * CB, gcoef + (size_t)kf * UB * CB, UB * CB,
                   &fbar[(kf + NFB) % NFB], l0 && kf >= 0 && kf < nbx);
            if (SPTRSV_BLOCK_L2PF) {
                l2pf_if(gctl + (size_t)kp * UB * kCtlBytes, UB * kCtlBytes, l0 && kp >= DP && kp < nbx);
                l2pf_if(gcoef + (size_t)kp * UB * CB, UB * CB, l0 && kp >= DP && kp < nbx);
            }
        };
        auto wait_bar = [&](uint64_t *bar, uint32_t ph) {
            Watch wd{0, 0};
            while (!mbar_try_wait(bar, ph))
                if (wd.expired(a.status, a.timeout_ns, tag)) break;
        };
        auto try_ctl = [&](int kb) { return kb >= nbx || mbar_try_wait(&cbar[kb % NCB], (uint32_t)((kb / NCB) & 1)); };
        auto try_coef = [&](int kb) { return kb >= nbx || mbar_try_wait(&fbar[kb % NFB], (uint32_t)((kb / NFB) & 1)); };
        auto wait_ctl = [&](int kb) { if (kb < nbx) wait_bar(&cbar[kb % NCB], (uint32_t)((kb / NCB) & 1)); };
        auto wait_coef = [&](int kb) { if (kb < nbx) wait_bar(&fbar[kb % NFB], (uint32_t)((kb / NFB) & 1)); };
        auto ctl_at = [&](int t) -> const int4 * {
            return reinterpret_cast<const int4 *>(ctlring + (size_t)(t & (CR - 1)) * kCtlBytes) + lane;
        };
        auto load_stage = [&](int t, Stage<T> &S) {
            S.c = *ctl_at(t);
            const unsigned char *fr = coefring + (size_t)(t & (FR - 1)) * CB;
            S.f.load(fr, lane);
            S.pub = reinterpret_cast<const int4 *>(fr + Coef<T>::PUB)[lane];
        };
        auto load_ext = [&](const Stage<T> &S, E3<T> &E) {
            if (OVF || GL) {
                E.e0 = ext_load<T, GL>(S.c.x, slots, gm);
                E.e1 = ext_load<T, GL>(S.c.y, slots, gm);
                E.e2 = ext_load<T, GL>(S.c.z, slots, gm);
            } else {
                E.e0 = ld_code(slots_u32, S.c.x, T(0));
                E.e1 = ld_code(slots_u32, S.c.y, T(0));
                E.e2 = ld_code(slots_u32, S.c.z, T(0));
            }
        };
        // cp.async of b(row) of step t, one commit group per step
        auto far_load = [&](int t, int row) {
            cp_b(bland_u32 + (uint32_t)((t & (DG - 1)) * 32 * sizeof(T)), b, row);
            cp_async_commit();
        };

        // ---- prologue
        if (SPTRSV_BLOCK_STAGGER_NS > 0) {
            // capped: the prologue burst is the first microseconds' problem, and a
            // deep factor (a chain) must never start a warp after its wave arrived
            const long long d = min((long long)a.unit_lev0[u] * SPTRSV_BLOCK_STAGGER_NS - SPTRSV_BLOCK_STAGGER_MARGIN,
                                    (long long)SPTRSV_BLOCK_STAGGER_CAP);
            if (d > 0) {
                const unsigned long long te = gtimer();
                while (gtimer() - te < (unsigned long long)d) __nanosleep(500);
            }
        }
        if (l0)
            for (int kb = 0; kb < min(nbx, DP); ++kb) {
                l2pf_if(gctl + (size_t)kb * UB * kCtlBytes, UB * kCtlBytes, true);
                l2pf_if(gcoef + (size_t)kb * UB * CB, UB * CB, true);
            }
        for (int kb = -DC; kb < 0; ++kb) issue(kb);     // control blocks 0..DC-1, coefficient blocks 0..DF-1
        for (int kb = 0; kb <= (DG + UB) / UB; ++kb) wait_ctl(kb);
        wait_coef(0);
        __syncwarp();
#pragma unroll 1
        for (int j = 0; j < DG; ++j) far_load(j, ctl_at(j)->w);
        Stage<T> S0, S1;
        load_stage(0, S0);
        load_stage(1, S1);
        E3<T> E0;
        if (!SPTRSV_BLOCK_EXT_LATE) load_ext(S0, E0);
        cp_async_wait<DG - 1>();
        T b0 = bland[lane];
        int nrow = ctl_at(DG)->w;               // row of the next far step
        T xprev = T(0);
        T hc0 = T(0), hc1 = T(0), hc2 = T(0);    // EARLY_SHFL: this step's shuffled values
#if SPTRSV_BLOCK_TRACE
        unsigned n_c = 0, n_f = 0, n_p = 0;            // dev: steps that found a ring block / an EXT value late
        long long cyc_b = 0, cyc_s = 0, cyc_0 = clock64();   // dev: cycles in the b wait / the slow path / total
#endif

        // ---- main loop: UNR steps per iteration.  A step is one basic block:
        // the chain runs speculatively on this step's EXT values while the next
        // steps' loads are issued; the readiness check (and any ring wait)
        // comes last, and its rare slow path redoes the chain.
#pragma unroll 1
        for (int t0 = 0; t0 < n; t0 += UNR) {
#pragma unroll
            for (int j = 0; j < UNR; ++j) {
                const int t = t0 + j;
                bool okc = true, okf = true;
                if (j % UB == 0) {          // block start: refill the rings, test the next blocks
                    const int kb = t / UB;
                    issue(kb);                           // ring slots of block kb-1 (read >= 3 steps ago)
                    okc = try_ctl(kb + (DG + UB) / UB);  // read from the next step on
                    okf = try_coef(kb + 1);
                }
                // ---- the chain on this step's values
                if (SPTRSV_BLOCK_EXT_LATE) load_ext(S0, E0);
                const T h0 = SPTRSV_BLOCK_EARLY_SHFL ? hc0 : __shfl_sync(0xffffffffu, xprev, S0.c.x);
                const T h1 = SPTRSV_BLOCK_EARLY_SHFL ? hc1 : __shfl_sync(0xffffffffu, xprev, S0.c.y);
                const T h2 = SPTRSV_BLOCK_EARLY_SHFL ? hc2 : __shfl_sync(0xffffffffu, xprev, S0.c.z);
                T acc = b0;
                acc = fnma(S0.f.a0, code_shfl(S0.c.x) ? h0 : E0.e0, acc);
                acc = fnma(S0.f.a1, code_shfl(S0.c.y) ? h1 : E0.e1, acc);
                acc = fnma(S0.f.a2, code_shfl(S0.c.z) ? h2 : E0.e2, acc);
                // ---- loads of later steps (independent of the chain)
                far_load(t + DG, nrow);
#if SPTRSV_BLOCK_TRACE
                const long long cw0 = clock64();
                cp_async_wait<DG - 1>();
                cyc_b += clock64() - cw0;
#else
                cp_async_wait<DG - 1>();
#endif
                const T b1 = bland[((t + 1) & (DG - 1)) * 32 + lane];
                E3<T> E1;
                if (!SPTRSV_BLOCK_EXT_LATE) load_ext(S1, E1);
                const int nrow1 = ctl_at(t + 1 + DG)->w;
                Stage<T> S2;
                load_stage(t + 2, S2);
                const PubA P = pub_addr<T>(S0.pub, S0.c.w, slots_u32, gm, x);
                if (SPTRSV_BLOCK_CHECK) {
                    SPTRSV_BCHECK(S0.pub.x < a.nslots && (S0.pub.x < 0 || S0.pub.x >= kZeroSlots), "pub slot", S0.pub.x);
                    SPTRSV_BCHECK(S0.pub.y < a.G, "pub mailbox", S0.pub.y);
                    SPTRSV_BCHECK(S0.pub.z < 0 || (!CL ? false : ((S0.pub.z >> 24) < a.cs && (S0.pub.z & 0xFFFFFF) < a.nslots)), "pub remote0", S0.pub.z);
                    SPTRSV_BCHECK(S0.pub.w < 0 || (!CL ? false : ((S0.pub.w >> 24) < a.cs && (S0.pub.w & 0xFFFFFF) < a.nslots)), "pub remote1", S0.pub.w);
                    SPTRSV_BCHECK(S0.c.w < a.n, "row", S0.c.w);
                    SPTRSV_BCHECK(OVF || GL || code_shfl(S0.c.x) || S0.c.x == kNoneCode || (code_kind(S0.c.x) == kKSmem && code_idx(S0.c.x) < a.nslots), "code0", S0.c.x);
                    SPTRSV_BCHECK(OVF || GL || code_shfl(S0.c.y) || S0.c.y == kNoneCode || (code_kind(S0.c.y) == kKSmem && code_idx(S0.c.y) < a.nslots), "code1", S0.c.y);
                    SPTRSV_BCHECK(OVF || GL || code_shfl(S0.c.z) || S0.c.z == kNoneCode || (code_kind(S0.c.z) == kKSmem && code_idx(S0.c.z) < a.nslots), "code2", S0.c.z);
                }
                // ---- readiness (value-as-flag; non-EXT terms hold 0) and ring waits
                const unsigned sh = sent_hi<T>();
                const bool pend = (hi_word(E0.e0) == sh) | (hi_word(E0.e1) == sh) | (hi_word(E0.e2) == sh);
#if SPTRSV_BLOCK_TRACE
                const long long cs0 = clock64();
#endif
                if (__any_sync(0xffffffffu, pend || !okc || !okf)) {
#if SPTRSV_BLOCK_TRACE
                    n_c += !okc;
                    n_f += !okf;
                    n_p += __any_sync(0xffffffffu, pend);
#endif
                    if (!okc) wait_ctl(t / UB + (DG + UB) / UB);
                    if (!okf) wait_coef(t / UB + 1);
                    if (__any_sync(0xffffffffu, pend)) {
                        E0 = repoll<T, GL>(E0, S0.c.x, S0.c.y, S0.c.z, &a, tag);
                        acc = b0;
                        acc = fnma(S0.f.a0, code_shfl(S0.c.x) ? h0 : E0.e0, acc);
                        acc = fnma(S0.f.a1, code_shfl(S0.c.y) ? h1 : E0.e1, acc);
                        acc = fnma(S0.f.a2, code_shfl(S0.c.z) ? h2 : E0.e2, acc);
                    }
                }
#if SPTRSV_BLOCK_TRACE
                cyc_s += clock64() - cs0;
                if (trc != nullptr && l0 && t < a.trace_cap - 1) trc[t] = gtimer();   // step t's inputs present
#endif
                if (OVF) {
                    const bool ovf = S0.c.x >= kOvfBase && code_kind(S0.c.x) == kKNone;
                    if (__any_sync(0xffffffffu, ovf))
                        acc = ovf_terms<T>(acc, ovf ? S0.c.x - kOvfBase : -1, xprev, &a, tag);
                }
                const T xi = UNIT ? Sentinel<T>::scrub(acc) : acc * S0.f.invd;   // a product is never the sentinel
                if (SPTRSV_BLOCK_EARLY_SHFL) {
                    hc0 = __shfl_sync(0xffffffffu, xi, S1.c.x);
                    hc1 = __shfl_sync(0xffffffffu, xi, S1.c.y);
                    hc2 = __shfl_sync(0xffffffffu, xi, S1.c.z);
                    pub_store(P, xi, CL);
                } else {
                    st_slot(slots_u32, S0.pub.x, xi);
                    st_mb(gm, S0.pub.y, xi);
                    if (CL) {
                        st_remote(slots_u32, S0.pub.z, xi);
                        st_remote(slots_u32, S0.pub.w, xi);
                    }
                    st_x(x, S0.c.w, xi);
                }
#if SPTRSV_BLOCK_TRACE
                if (trc != nullptr && a.ptrace != nullptr && S0.pub.y >= 0) a.ptrace[S0.pub.y] = gtimer();
#endif
                xprev = xi;
                S0 = S1;
                S1 = S2;
                if (!SPTRSV_BLOCK_EXT_LATE) E0 = E1;
                b0 = b1;
                nrow = nrow1;
            }
        }
        cp_async_wait<0>();
        if (trc != nullptr && l0) trc[a.trace_cap - 1] = gtimer();
#if SPTRSV_BLOCK_TRACE
        if (trc != nullptr && l0) {
            trc[a.trace_cap - 2] = t_entry;
            trc[a.trace_cap - 3] = n_c;
            trc[a.trace_cap - 4] = n_f;
            trc[a.trace_cap - 5] = n_p;
            trc[a.trace_cap - 6] = cyc_b;
            trc[a.trace_cap - 7] = cyc_s;
            trc[a.trace_cap - 8] = clock64() - cyc_0;
        }
#endif
    }
    }

    if (SPTRSV_BLOCK_REARM_END) {    // re-arm this CTA's mailboxes of the idle array for the next solve
        T *go = static_cast<T *>(a.gmb) + (size_t)((epoch & 1u) ^ 1u) * a.G;
        for (int i = a.cta_g0[blockIdx.x] + threadIdx.x; i < a.cta_g0[blockIdx.x + 1]; i += blockDim.x)
            go[i] = Sentinel<T>::value();
    }
    if (CL) cluster_sync_all();      // no CTA leaves while a cluster peer may still store into it
    else __syncthreads();
    if (threadIdx.x == 0) {      // the last CTA to finish advances the mailbox epoch
        __threadfence();
        if (atomicAdd(&a.ctr[1], 1u) == gridDim.x - 1) {
            atomicExch(&a.ctr[1], 0u);
            __threadfence();
            atomicAdd(&a.ctr[0], 1u);
        }
    }
}

template <typename T, bool UNIT>
void *pick_kernel_u(bool ovf, bool gl, bool cl) {
    if (gl) return ovf ? (void *)k_block<T, UNIT, true, true, false> : (void *)k_block<T, UNIT, false, true, false>;
    if (cl) return ovf ? (void *)k_block<T, UNIT, true, false, true> : (void *)k_block<T, UNIT, false, false, true>;
    return ovf ? (void *)k_block<T, UNIT, true, false, false> : (void *)k_block<T, UNIT, false, false, false>;
}
template <typename T>
void *pick_kernel(int diag, bool ovf, bool gl, bool cl) {
    return diag == SPTRSV_UNIT ? pick_kernel_u<T, true>(ovf, gl, cl) : pick_kernel_u<T, false>(ovf, gl, cl);
}

// Structured-grid detection: candidates (nx, nx*ny) from the dependency
// offsets of an interior row, each verified on every dependency on the GPU.
// 2-D grids are reported as (nx, 1): their y axis plays the role of z.
sptrsv_status_t detect_grid(sptrsv_handle_t h, const int32_t *tri_ptr, const int32_t *tri_col, DevArena &tmp,
                            cudaStream_t s, int &nx_out, int &ny_out) {
    nx_out = ny_out = 0;
    const int n = h->n;
    if (n < 64) return SPTRSV_SUCCESS;
    const int mid = h->uplo == SPTRSV_LOWER ? n - 1 - n / 3 : n / 3;
    int32_t rp[2];
    SPTRSV_CUDA(cudaMemcpyAsync(rp, tri_ptr + mid, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    const int deg = rp[1] - rp[0];
    if (deg <= 0 || deg > 64) return SPTRSV_SUCCESS;
    std::vector<int32_t> cols(deg);
    SPTRSV_CUDA(cudaMemcpyAsync(cols.data(), tri_col + rp[0], deg * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    std::vector<int64_t> offs;
    for (int c : cols) offs.push_back(std::abs((int64_t)mid - c));
    std::sort(offs.begin(), offs.end());
    std::vector<std::pair<int, int>> cand3, cand2;
    for (int64_t av : offs)
        for (int da = -1; da <= 1; ++da) {
            const int64_t nx = av + da;
            if (nx < 2 || nx >= n) continue;
            if (n % nx == 0 && n / nx >= 2) cand2.emplace_back((int)nx, 1);
            for (int64_t c : offs)
                for (int dc = -1; dc <= 1; ++dc)
                    for (int dn = -1; dn <= 1; ++dn) {
                        const int64_t nxy = c + dc + dn * nx;
                        if (nxy <= nx || nxy % nx != 0 || n % nxy != 0 || n / nxy < 2) continue;
                        cand3.emplace_back((int)nx, (int)(nxy / nx));
                    }
        }
    for (auto *cv : {&cand3, &cand2}) {
        std::sort(cv->begin(), cv->end());
        cv->erase(std::unique(cv->begin(), cv->end()), cv->end());
        if (cv->size() > 24) cv->resize(24);
    }
    unsigned *bad = nullptr;
    sptrsv_status_t st;
    if ((st = tmp.alloc_n(&bad, 1)) != SPTRSV_SUCCESS) return st;
    for (auto *cv : {&cand3, &cand2})
        for (auto &c : *cv) {
            SPTRSV_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned), s));
            k_grid_check<<<(n + 255) / 256, 256, 0, s>>>(n, c.first, c.second, tri_ptr, tri_col, bad);
            unsigned hb = 1;
            SPTRSV_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
            SPTRSV_CUDA(cudaStreamSynchronize(s));
            if (hb == 0) {
                nx_out = c.first;
                ny_out = c.second;
                return SPTRSV_SUCCESS;
            }
        }
    return SPTRSV_SUCCESS;
}

// K CTAs of `threads` threads and `smem` dynamic shared memory, in clusters
// of cs: co-resident?  (Checked on the slot-mode instance, the largest.)
bool clusters_fit(sptrsv_handle_t h, bool f64, int cs, int K, int threads, size_t smem) {
    void *kn = f64 ? (void *)k_block<double, false, false, false, true> : (void *)k_block<float, false, false, false, true>;
    if (cudaFuncSetAttribute(kn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)K);
    cfg.blockDim = dim3((unsigned)threads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, kn, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    (void)h;
    return (int64_t)nc * cs >= K;
}

int i32_at(const int32_t *d, int64_t i, cudaStream_t s, sptrsv_status_t &st) {
    int32_t v = 0;
    cudaError_t e = cudaMemcpyAsync(&v, d + i, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) st = cuda_fail(e, "i32_at");
    return v;
}

}  // namespace

// Natural-order CSR (ptr[n+1], col, val) of the referenced strict triangle, in
// each row's storage order, rebuilt from the chunk layout into `tmp`.
sptrsv_status_t build_tri_csr(sptrsv_handle_t h, DevArena &tmp, cudaStream_t s, int32_t **ptr_out, int32_t **col_out,
                              void **val_out) {
    const int n = h->n;
    const size_t es = h->esize;
    sptrsv_status_t st;
    int32_t *tri_ptr = nullptr, *tri_col = nullptr;
    void *tri_val = nullptr;
    const int64_t nnz = h->info.nnz_used;
    if ((st = tmp.alloc_n(&tri_ptr, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&tri_col, (size_t)std::max<int64_t>(nnz, 1))) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc(&tri_val, (size_t)std::max<int64_t>(nnz, 1) * es)) != SPTRSV_SUCCESS) return st;
    {
        int32_t *dpx = nullptr;
        if ((st = tmp.alloc_n(&dpx, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
        SPTRSV_CUDA(cudaMemcpyAsync(dpx, h->d_dp, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
        SPTRSV_CUDA(cudaMemsetAsync(dpx + n, 0, sizeof(int32_t), s));
        if ((st = exclusive_scan_i32(dpx, tri_ptr, (int64_t)n + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    }
    const int cgrid = std::max(1, std::min((h->nchunks * 32 + 255) / 256, h->num_sms * 16));
    if (h->dtype == SPTRSV_F64)
        k_tri_fill<double><<<cgrid, 256, 0, s>>>(h->nchunks, h->d_chunks, h->d_perm, h->d_ecol,
                                                 (const double *)h->d_eval, tri_ptr, tri_col, (double *)tri_val);
    else
        k_tri_fill<float><<<cgrid, 256, 0, s>>>(h->nchunks, h->d_chunks, h->d_perm, h->d_ecol,
                                                (const float *)h->d_eval, tri_ptr, tri_col, (float *)tri_val);
    SPTRSV_CUDA(cudaGetLastError());
    *ptr_out = tri_ptr;
    *col_out = tri_col;
    *val_out = tri_val;
    return SPTRSV_SUCCESS;
}

sptrsv_status_t block_build(sptrsv_handle_t h, cudaStream_t s) {
    ArenaStream as_{h->arena, s};     // the handle's allocations in this call: stream-ordered on s
    BlockPlan &B = h->block;
    const int n = h->n;
    const int nlev = h->info.nlev;
    DevArena tmp(s);
    struct Guard {
        DevArena &a;
        ~Guard() { a.release_all(); }
    } guard{tmp};
    sptrsv_status_t st = SPTRSV_SUCCESS;
    const size_t es = h->esize;
    const bool f64 = h->dtype == SPTRSV_F64;
    int max_smem = 0;
    SPTRSV_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
    const int eg = (n + 255) / 256;
    const int CB = f64 ? Coef<double>::BYTES : Coef<float>::BYTES;
    const size_t wsb = f64 ? warp_smem_bytes<double>() : warp_smem_bytes<float>();

    // ---- 1. natural-order CSR of the triangle
    int32_t *tri_ptr = nullptr, *tri_col = nullptr;
    void *tri_val = nullptr;
    if ((st = build_tri_csr(h, tmp, s, &tri_ptr, &tri_col, &tri_val)) != SPTRSV_SUCCESS) return st;

    const size_t budget = (size_t)max_smem - 1024;          // static smem + slack

    // ---- 2. partition rows over U = K x wpc warps of K co-resident CTAs
    int32_t *unit = nullptr;
    if ((st = h->arena.alloc_n(&unit, n)) != SPTRSV_SUCCESS) return st;
    B.d_unit = unit;
    int gnx = 0, gny = 0;
    if (n >= 64) {
        if ((st = detect_grid(h, tri_ptr, tri_col, tmp, s, gnx, gny)) != SPTRSV_SUCCESS) return st;
    }
    int K = 1, wpc = 4;
    B.cs = 1;
    B.grid_nx = B.grid_ny = B.tile_w = B.tile_h = 0;
    if (gnx > 0) {
        // warp tile tw x th columns (<= 32: one step per level), CTA = wx x wy
        // tiles; the fewest warps per CTA that fit all CTAs on the SMs
        int tw = std::min(gny == 1 ? 32 : 8, gnx);
        int th = std::max(1, std::min(32 / std::max(tw, 1), gny));
        static const int shapes[][2] = {{1, 1}, {2, 1}, {1, 2}, {2, 2}};
        int wx = 0, wy = 0;
        for (int grow = 0; grow < 8 && wx == 0; ++grow) {
            const int ntx = (gnx + tw - 1) / tw, nty = (gny + th - 1) / th;
            for (auto &sh : shapes) {
                if (sh[0] > ntx && sh[0] > 1) continue;
                if (sh[1] > nty && sh[1] > 1) continue;
                const int k = ((ntx + sh[0] - 1) / sh[0]) * ((nty + sh[1] - 1) / sh[1]);
                if (k <= h->num_sms) {
                    wx = sh[0];
                    wy = sh[1];
                    break;
                }
            }
            if (wx == 0) {          // tiles too small for the SM count: grow them
                if (th < gny) th *= 2;
                else tw *= 2;
            }
        }
        if (wx > 0) {
            const int ntx = (gnx + tw - 1) / tw, nty = (gny + th - 1) / th;
            const int cxn = (ntx + wx - 1) / wx, cyn = (nty + wy - 1) / wy;
            K = cxn * cyn;
            wpc = wx * wy;
            if (K > h->num_sms) return SPTRSV_ERR_NOT_SUPPORTED;
            // clusters of CTAs (DSMEM hand-offs): the largest csx x csy <= 8 that
            // tiles the CTA grid and can be co-resident
            int csx = 1, csy = 1;
            static const int cshapes[][2] = {{2, 4}, {4, 2}, {2, 2}, {4, 1}, {1, 4}, {2, 1}, {1, 2}};
            for (auto &c : cshapes) {
                if (cxn % c[0] || cyn % c[1]) continue;
                if (!clusters_fit(h, f64, c[0] * c[1], K, 32 * (1 + kNf) * wpc, budget)) continue;
                csx = c[0];
                csy = c[1];
                break;
            }
            B.cs = csx * csy;
            B.csx = csx;
            k_part_tiles<<<eg, 256, 0, s>>>(n, gnx, gny, tw, th, wx, wy, cxn, K, h->uplo == SPTRSV_UPPER, csx, csy,
                                            unit);
            B.grid_nx = gnx;
            B.grid_ny = gny;
            B.tile_w = tw;
            B.tile_h = th;
        } else {
            gnx = 0;
        }
    }
    if (gnx == 0) {
        K = (int)std::max<int64_t>(1, std::min<int64_t>(h->num_sms, n / 8192));
        wpc = 4;
        while (wpc > 1 && (size_t)wpc * wsb + 2048 * es > budget) wpc /= 2;
        k_part_natural<<<eg, 256, 0, s>>>(n, K * wpc, h->uplo, unit);
    }
    SPTRSV_CUDA(cudaGetLastError());
    const int U = K * wpc;
    B.nblocks = K;
    B.wpc = wpc;
    B.nunits = U;
    if ((uint64_t)U * (uint64_t)std::max(nlev, 1) * kBuckets >= (1ull << 32)) return SPTRSV_ERR_NOT_SUPPORTED;

    // ---- 3. order (unit, level, decreasing deps, row); groups (unit, level) -> 32-row steps
    uint32_t *keys = nullptr, *skeys = nullptr;
    int32_t *pos = nullptr, *head = nullptr, *gid = nullptr, *bperm = nullptr;
    if ((st = tmp.alloc_n(&keys, n)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&skeys, n)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&pos, n)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&head, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&gid, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&bperm, n)) != SPTRSV_SUCCESS) return st;
    k_unit_keys<<<eg, 256, 0, s>>>(n, nlev, unit, h->d_lev, h->d_dp, keys);
    if ((st = radix_sort_pairs(keys, nullptr, skeys, bperm, n, (uint32_t)((uint64_t)U * nlev * kBuckets - 1), tmp,
                               s)) != SPTRSV_SUCCESS)
        return st;
    SPTRSV_CUDA(cudaMemsetAsync(head + n, 0, sizeof(int32_t), s));
    k_heads<<<eg, 256, 0, s>>>(skeys, bperm, n, head, pos);
    if ((st = exclusive_scan_i32(head, gid, (int64_t)n + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    const int32_t ngroups = i32_at(gid, n, s, st);
    if (st != SPTRSV_SUCCESS) return st;
    int32_t *gp0 = nullptr, *nsub = nullptr, *sub0 = nullptr;
    if ((st = tmp.alloc_n(&gp0, (size_t)ngroups + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&nsub, (size_t)ngroups + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&sub0, (size_t)ngroups + 1)) != SPTRSV_SUCCESS) return st;
    const int gg = (ngroups + 1 + 255) / 256;
    k_group_start<<<eg, 256, 0, s>>>(head, gid, n, ngroups, gp0);
    k_group_sub<<<gg, 256, 0, s>>>(gp0, ngroups, nsub);
    if ((st = exclusive_scan_i32(nsub, sub0, (int64_t)ngroups + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    const int32_t nsteps = i32_at(sub0, ngroups, s, st);
    if (st != SPTRSV_SUCCESS) return st;
    B.nsteps = nsteps;
    int2 *steps = nullptr;
    int32_t *step_unit = nullptr, *step_of = nullptr, *cta_p0 = nullptr;
    if ((st = tmp.alloc_n(&steps, (size_t)nsteps + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&step_unit, (size_t)nsteps + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&step_of, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&cta_p0, (size_t)K + 1)) != SPTRSV_SUCCESS) return st;
    int32_t *unit_step0 = nullptr, *pcnt = nullptr, *pmap = nullptr;
    if ((st = tmp.alloc_n(&unit_step0, (size_t)U + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&pcnt, (size_t)U + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&pmap, (size_t)nsteps + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&B.d_unit_step0, (size_t)U + 1)) != SPTRSV_SUCCESS) return st;
    k_steps<<<gg, 256, 0, s>>>(gp0, sub0, ngroups, bperm, unit, steps, step_unit);
    k_unit_step0<<<(nsteps + 255) / 256, 256, 0, s>>>(step_unit, nsteps, U, unit_step0);
    k_pos_step<<<eg, 256, 0, s>>>(head, gid, gp0, sub0, n, step_of);
    k_cta_p0<<<(K + 1 + 255) / 256, 256, 0, s>>>(K, wpc, nsteps, n, unit_step0, steps, cta_p0);
    // every warp's steps padded to a multiple of UNR (empty steps): padded starts, step -> padded step
    k_pad_count<<<(U + 1 + 255) / 256, 256, 0, s>>>(U, unit_step0, pcnt);
    if ((st = exclusive_scan_i32(pcnt, B.d_unit_step0, (int64_t)U + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    k_pad_map<<<(nsteps + 255) / 256, 256, 0, s>>>(nsteps, step_unit, unit_step0, B.d_unit_step0, pmap);
    const int32_t npad = i32_at(B.d_unit_step0, U, s, st);
    if (st != SPTRSV_SUCCESS) return st;
    B.npad = npad;
    SPTRSV_CUDA(cudaGetLastError());

    // ---- 4. shared-memory budget, dependency classes, inbound items
    const size_t fixed = (size_t)wpc * wsb;
    if (fixed > budget) return SPTRSV_ERR_NOT_SUPPORTED;
    const int cap = (int)((budget - fixed) / es) - kZeroSlots;
    unsigned char *noslot = nullptr;
    int32_t *need = nullptr, *bits = nullptr, *slot_scan = nullptr, *g_scan = nullptr, *ccnt = nullptr;
    int32_t *icnt = nullptr, *iptr = nullptr;
    if ((st = tmp.alloc_n(&noslot, (size_t)K)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&need, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&bits, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&slot_scan, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&g_scan, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&ccnt, (size_t)K)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&icnt, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&iptr, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemsetAsync(noslot, 0, (size_t)K, s));
    // intra-CTA slots (need bit 0), CROSS dependencies per position
    SPTRSV_CUDA(cudaMemsetAsync(need, 0, sizeof(int32_t) * ((size_t)n + 1), s));
    k_need<<<eg, 256, 0, s>>>(n, wpc, tri_ptr, tri_col, unit, pos, step_of, noslot, need, icnt);
    k_need_bits<<<(n + 1 + 255) / 256, 256, 0, s>>>(n, need, 0, bits);
    if ((st = exclusive_scan_i32(bits, slot_scan, (int64_t)n + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    if ((st = exclusive_scan_i32(icnt, iptr, (int64_t)n + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    k_cta_slots<<<(K + 255) / 256, 256, 0, s>>>(K, cta_p0, slot_scan, iptr, ccnt);
    SPTRSV_CUDA(cudaGetLastError());
    std::vector<int32_t> hcnt((size_t)K);
    SPTRSV_CUDA(cudaMemcpyAsync(hcnt.data(), ccnt, sizeof(int32_t) * K, cudaMemcpyDeviceToHost, s));
    const int32_t ncross = i32_at(iptr, n, s, st);      // (synchronizes)
    if (st != SPTRSV_SUCCESS) return st;
    // every CTA's intra + CROSS slots fit: slot mode; else the GL instance
    // (CROSS terms poll mailboxes), and CTAs whose intra slots do not fit use
    // mailboxes for those too
    bool gl = false;
    int max_slots = 0;
    for (int c = 0; c < K; ++c) {
        gl |= hcnt[c] > cap;
        max_slots = std::max(max_slots, hcnt[c]);
    }
    if (gl) {
        k_cta_slots<<<(K + 255) / 256, 256, 0, s>>>(K, cta_p0, slot_scan, nullptr, ccnt);   // intra only
        SPTRSV_CUDA(cudaMemcpyAsync(hcnt.data(), ccnt, sizeof(int32_t) * K, cudaMemcpyDeviceToHost, s));
        SPTRSV_CUDA(cudaStreamSynchronize(s));
        std::vector<unsigned char> hns(K, 0);
        bool over = false;
        max_slots = 0;
        for (int c = 0; c < K; ++c) {
            if (hcnt[c] > cap) hns[c] = 1, over = true;
            else max_slots = std::max(max_slots, hcnt[c]);
        }
        if (over) {
            SPTRSV_CUDA(cudaMemcpyAsync(noslot, hns.data(), (size_t)K, cudaMemcpyHostToDevice, s));
            SPTRSV_CUDA(cudaMemsetAsync(need, 0, sizeof(int32_t) * ((size_t)n + 1), s));
            k_need<<<eg, 256, 0, s>>>(n, wpc, tri_ptr, tri_col, unit, pos, step_of, noslot, need, icnt);
            k_need_bits<<<(n + 1 + 255) / 256, 256, 0, s>>>(n, need, 0, bits);
            if ((st = exclusive_scan_i32(bits, slot_scan, (int64_t)n + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
        }
        k_need_gl<<<eg, 256, 0, s>>>(n, wpc, tri_ptr, tri_col, unit, pos, step_of, noslot, need);
    }
    B.gl = gl;
    const int cs = gl ? 1 : B.cs;
    if (gl) B.cs = 1;
    // CROSS dependencies: slots, DSMEM targets, fetch flags, mailbox bits
    int32_t *islot = nullptr, *rtc = nullptr, *iprod = nullptr, *fscan = nullptr;
    int2 *rt = nullptr;
    unsigned char *fetch = nullptr;
    uint32_t *ikey = nullptr;
    const size_t nq = (size_t)std::max(ncross, 1);
    if ((st = tmp.alloc_n(&islot, nq)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&iprod, nq)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&fscan, nq + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&ikey, nq)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&fetch, nq)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&rtc, (size_t)n)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&rt, (size_t)n)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemsetAsync(rtc, 0, sizeof(int32_t) * (size_t)n, s));
    SPTRSV_CUDA(cudaMemsetAsync(rt, 0xFF, sizeof(int2) * (size_t)n, s));
    if (!gl && ncross > 0)
        k_cross<<<eg, 256, 0, s>>>(n, nlev, wpc, cs, 0, bperm, tri_ptr, tri_col, unit, pos, step_of, h->d_lev,
                                   slot_scan, cta_p0, iptr, islot, need, rtc, rt, fetch, ikey, iprod);
    k_need_bits<<<(n + 1 + 255) / 256, 256, 0, s>>>(n, need, 1, bits);
    if ((st = exclusive_scan_i32(bits, g_scan, (int64_t)n + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    const int32_t G = i32_at(g_scan, n, s, st);
    if (st != SPTRSV_SUCCESS) return st;
    B.G = (G + 3) / 4 * 4;             // mailbox array stride (16-byte aligned arrays)
    B.nslots = kZeroSlots + max_slots;
    if ((st = h->arena.alloc_n(&B.d_cta_g0, (size_t)K + 1)) != SPTRSV_SUCCESS) return st;
    k_cta_g0<<<(K + 1 + 255) / 256, 256, 0, s>>>(K, cta_p0, g_scan, B.d_cta_g0);
    // inbound items {mailbox, slot} of the fetched CROSS dependencies, sorted by (CTA, level)
    int32_t nitems = 0;
    if (!gl && ncross > 0) {
        int32_t *fl = nullptr;
        if ((st = tmp.alloc_n(&fl, nq + 1)) != SPTRSV_SUCCESS) return st;
        k_flag_i32<<<(int)((nq + 1 + 255) / 256), 256, 0, s>>>(ncross, fetch, fl);
        if ((st = exclusive_scan_i32(fl, fscan, (int64_t)ncross + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
        nitems = i32_at(fscan, ncross, s, st);
        if (st != SPTRSV_SUCCESS) return st;
    }
    if ((st = h->arena.alloc_n(&B.d_fptr, (size_t)U + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&B.d_fitems, (size_t)std::max(nitems, 1) + 2)) != SPTRSV_SUCCESS) return st;   // + L2-prefetch tail padding
    SPTRSV_CUDA(cudaMemsetAsync(B.d_fptr, 0, sizeof(int32_t) * ((size_t)U + 1), s));
    if (nitems > 0) {
        uint32_t *key = nullptr, *skey = nullptr;
        int2 *item = nullptr;
        int32_t *perm = nullptr;
        if ((st = tmp.alloc_n(&key, nitems)) != SPTRSV_SUCCESS) return st;
        if ((st = tmp.alloc_n(&skey, nitems)) != SPTRSV_SUCCESS) return st;
        if ((st = tmp.alloc_n(&item, nitems)) != SPTRSV_SUCCESS) return st;
        if ((st = tmp.alloc_n(&perm, nitems)) != SPTRSV_SUCCESS) return st;
        k_item_compact<<<(ncross + 255) / 256, 256, 0, s>>>(ncross, fetch, fscan, ikey, iprod, islot, g_scan, key, item);
        if ((st = radix_sort_pairs(key, nullptr, skey, perm, nitems, (uint32_t)((uint64_t)U * nlev - 1), tmp, s)) !=
            SPTRSV_SUCCESS)
            return st;
        k_item_gather<<<(nitems + 255) / 256, 256, 0, s>>>(nitems, perm, item, B.d_fitems);
        if ((st = h->arena.alloc_n(&B.d_fkey, (size_t)nitems)) != SPTRSV_SUCCESS) return st;   // (tools)
        SPTRSV_CUDA(cudaMemcpyAsync(B.d_fkey, skey, sizeof(uint32_t) * nitems, cudaMemcpyDeviceToDevice, s));
        k_item_ptr<<<(nitems + 1 + 255) / 256, 256, 0, s>>>(nitems, U, nlev, skey, B.d_fptr);
        SPTRSV_CUDA(cudaGetLastError());
    }
    B.nitems = nitems;

    // ---- 5. overflow lists and records
    int32_t *ocnt = nullptr, *ovf_ptr = nullptr;
    if ((st = tmp.alloc_n(&ocnt, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&ovf_ptr, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    k_ovf_count<<<(n + 1 + 255) / 256, 256, 0, s>>>(n, bperm, h->d_dp, ocnt);
    if ((st = exclusive_scan_i32(ocnt, ovf_ptr, (int64_t)n + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    const int32_t novf = i32_at(ovf_ptr, n, s, st);
    if (st != SPTRSV_SUCCESS) return st;
    B.novf = novf;
    // + kPadSteps: a warp's last block of records / row ids is copied whole
    const size_t nrec = (size_t)npad + kPadSteps;
    if ((st = h->arena.alloc(&B.d_ctl, nrec * kCtlBytes)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc(&B.d_coef, nrec * CB)) != SPTRSV_SUCCESS) return st;
    {
        const int fgp = (int)std::max<int64_t>(1, ((int64_t)nrec * 32 + 255) / 256);
        if (f64) k_pad_fill<double><<<fgp, 256, 0, s>>>((int64_t)nrec, (unsigned char *)B.d_ctl, (unsigned char *)B.d_coef);
        else k_pad_fill<float><<<fgp, 256, 0, s>>>((int64_t)nrec, (unsigned char *)B.d_ctl, (unsigned char *)B.d_coef);
    }
    if ((st = h->arena.alloc_n(&B.d_ovf_code, (size_t)std::max(novf, 1))) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc(&B.d_ovf_val, (size_t)std::max(novf, 1) * es)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc(&B.d_gmb, (size_t)2 * std::max(B.G, 4) * es)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&B.d_ctr, 4)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemsetAsync(B.d_ctr, 0, 4 * sizeof(unsigned), s));
    const int pg = (int)std::max<int64_t>(1, ((int64_t)nsteps * 32 + 255) / 256);
    const int fg = std::max(1, std::min((int)((2 * (int64_t)std::max(B.G, 4) + 255) / 256), h->num_sms * 8));
    if (f64) {
        k_rec_fill<double><<<pg, 256, 0, s>>>(nsteps, wpc, steps, pmap, bperm, pos, step_of, unit, tri_ptr, tri_col,
                                              (const double *)tri_val, (const double *)h->d_invd_row,
                                              h->diag == SPTRSV_UNIT, noslot, need, slot_scan, g_scan, cta_p0,
                                              ovf_ptr, iptr, islot, (int)gl, rt, (unsigned char *)B.d_ctl, (unsigned char *)B.d_coef, B.d_ovf_code,
                                              (double *)B.d_ovf_val);
        k_fill_sentinel<double><<<fg, 256, 0, s>>>((double *)B.d_gmb, 2 * (int64_t)std::max(B.G, 4));
    } else {
        k_rec_fill<float><<<pg, 256, 0, s>>>(nsteps, wpc, steps, pmap, bperm, pos, step_of, unit, tri_ptr, tri_col,
                                             (const float *)tri_val, (const float *)h->d_invd_row,
                                             h->diag == SPTRSV_UNIT, noslot, need, slot_scan, g_scan, cta_p0,
                                             ovf_ptr, iptr, islot, (int)gl, rt, (unsigned char *)B.d_ctl, (unsigned char *)B.d_coef, B.d_ovf_code,
                                             (float *)B.d_ovf_val);
        k_fill_sentinel<float><<<fg, 256, 0, s>>>((float *)B.d_gmb, 2 * (int64_t)std::max(B.G, 4));
    }
    if ((st = h->arena.alloc_n(&B.d_unit_lev0, (size_t)U)) != SPTRSV_SUCCESS) return st;
    k_unit_lev0<<<(U + 127) / 128, 128, 0, s>>>(U, B.d_unit_step0, (const unsigned char *)B.d_ctl, h->d_lev,
                                               B.d_unit_lev0);
    SPTRSV_CUDA(cudaGetLastError());

    // ---- launch configuration: K co-resident CTAs of wpc warps
    void *kn = f64 ? pick_kernel<double>(h->diag, novf > 0, gl, B.cs > 1)
                   : pick_kernel<float>(h->diag, novf > 0, gl, B.cs > 1);
    const size_t smem = fixed + (size_t)B.nslots * es;
    SPTRSV_CUDA(cudaFuncSetAttribute(kn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    SPTRSV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kn, 32 * (1 + kNf) * wpc, smem));
    if (per_sm * h->num_sms < K) return SPTRSV_ERR_NOT_SUPPORTED;
    B.kernel = kn;
    B.smem = smem;
    B.threads = 32 * (1 + kNf) * wpc;    // wpc compute warps + kNf fetcher warps each
    B.rec_bytes = kCtlBytes + CB;
    B.nent = (int64_t)npad * (kCtlBytes + CB);
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    B.built = true;
    return SPTRSV_SUCCESS;
}

sptrsv_status_t block_refresh_values(sptrsv_handle_t h, const int32_t *tri_ptr, const void *tri_val, cudaStream_t s) {
    const BlockPlan &B = h->block;
    const int64_t npad = B.npad;
    if (npad == 0) return SPTRSV_SUCCESS;
    const int g = (int)((npad * 32 + 255) / 256);
    if (h->dtype == SPTRSV_F64)
        k_rec_refill<double><<<g, 256, 0, s>>>(npad, (const unsigned char *)B.d_ctl, (unsigned char *)B.d_coef, tri_ptr,
                                               (const double *)tri_val, (const double *)h->d_invd_row,
                                               h->diag == SPTRSV_UNIT, (double *)B.d_ovf_val);
    else
        k_rec_refill<float><<<g, 256, 0, s>>>(npad, (const unsigned char *)B.d_ctl, (unsigned char *)B.d_coef, tri_ptr,
                                              (const float *)tri_val, (const float *)h->d_invd_row,
                                              h->diag == SPTRSV_UNIT, (float *)B.d_ovf_val);
    SPTRSV_CUDA(cudaGetLastError());
    return SPTRSV_SUCCESS;
}

sptrsv_status_t block_solve(sptrsv_handle_t h, const void *b, void *x, cudaStream_t s) {
    BlockPlan &B = h->block;
    if (!B.built) return SPTRSV_ERR_NOT_SUPPORTED;
    BlockArgs a;
    a.unit_step0 = B.d_unit_step0;
    a.unit_lev0 = B.d_unit_lev0;
    a.ctl = (const unsigned char *)B.d_ctl;
    a.coef = (const unsigned char *)B.d_coef;
    a.cta_g0 = B.d_cta_g0;
    a.fitems = B.d_fitems;
    a.fptr = B.d_fptr;
    a.ovf_code = B.d_ovf_code;
    a.ovf_val = B.d_ovf_val;
    a.gmb = B.d_gmb;
    a.ctr = B.d_ctr;
    a.status = B.d_ctr + 2;
    a.trace = static_cast<unsigned long long *>(B.trace);
    a.trace_cap = B.trace_cap;
    a.ftrace = static_cast<unsigned long long *>(B.ftrace);
    a.ptrace = static_cast<unsigned long long *>(B.ptrace);
    a.b = b;
    a.x = x;
    a.G = B.G;
    a.n = h->n;
    a.cs = B.cs;
    a.nslots = B.nslots;
    a.timeout_ns = h->timeout_ns;
    void *args[] = {(void *)&a};
    if (B.cs <= 1) {
        SPTRSV_CUDA(cudaLaunchCooperativeKernel(B.kernel, B.nblocks, B.threads, args, B.smem, s));
    } else {
        // clusters of B.cs CTAs; co-residency of all K CTAs was checked at
        // build time (cudaOccupancyMaxActiveClusters)
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)B.nblocks);
        cfg.blockDim = dim3((unsigned)B.threads);
        cfg.dynamicSmemBytes = B.smem;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)B.cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        SPTRSV_CUDA(cudaLaunchKernelExC(&cfg, B.kernel, args));
    }
    h->last_solve = 1;
    return SPTRSV_SUCCESS;
}

// TIMEOUT iff the last BLOCK solve on the handle gave up a wait: its status
// word holds the solve's epoch + 1 and the epoch counter has advanced past it.
sptrsv_status_t block_solve_status(sptrsv_handle_t h) {
    BlockPlan &B = h->block;
    if (!B.built) return SPTRSV_SUCCESS;
    unsigned c[4] = {0, 0, 0, 0};
    SPTRSV_CUDA(cudaMemcpy(c, B.d_ctr, sizeof(c), cudaMemcpyDeviceToHost));
    return (c[2] != 0 && c[2] == c[0]) ? SPTRSV_ERR_TIMEOUT : SPTRSV_SUCCESS;
}

}  // namespace sptrsv
