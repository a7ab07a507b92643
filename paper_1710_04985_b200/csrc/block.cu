// block.cu -- SPTRSV_ALGO_BLOCK: self-scheduling over WARP-owned row tiles
// (SURVEY.md §7 hard part H1, lever (a)).
//
// Why: on B200 a cross-SM handoff costs >= one L2 round trip (~220 ns,
// profiles/microbench_r1.json), a CTA-wide barrier step ~55-130 ns, while a
// shared-memory load is ~30 cycles and __syncwarp a few.  The paper's SLFR
// pays the L2 price on every edge of the critical path (nlev = 382 on cfg2).
// Here the rows are partitioned over U = K x WPC warps (K co-resident CTAs,
// WPC warps each).  Warp u walks the GLOBAL levels of its own rows
// in order, one lane per row and __syncwarp between levels; every result goes
// to a shared-memory slot (and to x).  Dependencies are read
//   * from the warp's own slots (ordered by __syncwarp),
//   * from another warp's slots in the same CTA by value-as-flag polling of
//     shared memory (slots prefilled with a NaN sentinel),
//   * from another CTA by value-as-flag polling of x in global memory (x
//     prefilled with the sentinel), loaded speculatively two levels ahead.
// No CTA-wide barrier runs during the solve: each warp self-schedules.
// The partition keeps long dependency chains inside a warp and a CTA:
//   * structured grids (detected: every dependency verified to be a 3x3x3
//     neighbour under the inferred nx, ny) -> (x, y) tiles x all z, 2x2 tiles
//     per CTA, so z-chains stay in one warp and a path crosses few CTAs;
//   * otherwise contiguous topological blocks.
// Progress: all CTAs are co-resident (cooperative launch) and every warp
// processes its levels in increasing order, so the lowest unfinished level
// always advances.
//
// Step records: one fixed-size record per (warp, level) step of <= 32 rows
// (lane = row), contiguous per warp, streamed into a per-warp shared-memory
// ring by TMA bulk copies (cp.async.bulk + mbarrier), nst records in flight:
//   int32 rows[32] (-1 = padding lane) | int32 cols[W][32] | T invd[32] | T vals[W][32]
//   cols >= 0: global column (another CTA, or a value that left the ring);
//   cols < 0: shared slot -1-cols (slot Z = the zero slot pads short rows).
//   W = min(max dependencies per row, kTprMax); the rest: ovf_* (CSR by position).
// Every per-step address is a constant offset, so the step loop is short.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "internal.h"

namespace sptrsv {
namespace {

constexpr int kWPC = 4;          // warps (tiles) per CTA
constexpr int kBuckets = kTprMax + 2;
constexpr int kLead = 2;         // register lead of b / speculative external x (3 register sets)
constexpr int kPrefB = 6;        // L2 prefetch lead of b
constexpr int kSleepSmemNs = 40;    // poll back-off: a spinning warp must not starve its SM's LSU pipe
constexpr int kSleepGlobalNs = 80;
constexpr int kMinStages = 8;    // records in flight per warp (> kPrefB, or the lookahead deadlocks)
static_assert(kMinStages > kPrefB && kMinStages > kLead + 1, "record ring shorter than the lookahead");

__device__ __forceinline__ uint32_t bucket_of(int deps) { return deps > kTprMax ? 0u : (uint32_t)(kTprMax + 1 - deps); }
// fixed record geometry: rows | cols[W] | invd | vals[W], 32 lanes each
__host__ __device__ __forceinline__ int rec_bytes(int W, int es) { return 32 * (4 + 4 * W + es + es * W); }
__host__ __device__ __forceinline__ int rec_cols(int) { return 32 * 4; }
__host__ __device__ __forceinline__ int rec_invd(int W) { return 32 * 4 * (1 + W); }
__host__ __device__ __forceinline__ int rec_vals(int W, int es) { return 32 * (4 * (1 + W) + es); }

// -------------------------------------------------------------- build kernels
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

// (x, y) tiles: CTA (cx, cy) owns the 2x2 tiles (2cx..2cx+1, 2cy..2cy+1);
// a tile is a set of z-columns, so the z-chains stay inside one warp
__global__ void k_part_tiles(int n, int nx, int ny, int cxn, int cyn, int32_t *unit) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int x = i % nx, y = (i / nx) % ny;
    const int tx = (int)((int64_t)x * (2 * cxn) / nx), ty = (int)((int64_t)y * (2 * cyn) / ny);
    const int cta = (tx >> 1) * cyn + (ty >> 1);
    unit[i] = cta * kWPC + (tx & 1) * 2 + (ty & 1);
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

// position -> step; padded position of each row inside its warp's step stream
__global__ void k_pos_step(const int32_t *head, const int32_t *gid, const int32_t *gp0, const int32_t *sub0,
                           const int2 *steps, const int32_t *bperm, const int32_t *unit,
                           const int32_t *unit_step0, int n, int32_t *step_of, int32_t *ppos) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int g = gid[p] + head[p] - 1;
    const int s = sub0[g] + (p - gp0[g]) / 32;
    step_of[p] = s;
    const int row = bperm[p];
    ppos[row] = (s - unit_step0[unit[row]]) * 32 + (p - steps[s].x);
}

__global__ void k_ovf_count(int n, const int32_t *bperm, const int32_t *dp, int W, int32_t *ocnt) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) ocnt[p] = max(0, dp[bperm[p]] - W);
    if (p == n) ocnt[p] = 0;
}

// padding lanes of every step: row -1, zero-slot columns, zero values
template <typename T>
__global__ void k_rec_pad(int nsteps, int W, int Z, const int2 *steps, unsigned char *recs) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)nsteps * 32) return;
    const int s = (int)(t >> 5), lane = (int)(t & 31);
    if (lane < steps[s].y) return;
    unsigned char *base = recs + (size_t)s * rec_bytes(W, sizeof(T));
    reinterpret_cast<int32_t *>(base)[lane] = -1;
    int32_t *cols = reinterpret_cast<int32_t *>(base + rec_cols(W));
    T *vals = reinterpret_cast<T *>(base + rec_vals(W, sizeof(T)));
    for (int k = 0; k < W; ++k) {
        cols[k * 32 + lane] = -1 - Z;
        vals[k * 32 + lane] = T(0);
    }
    reinterpret_cast<T *>(base + rec_invd(W))[lane] = T(0);
}

template <typename T>
__global__ void k_rec_fill(int n, int Wu, int W, int Z, const int32_t *__restrict__ unit,
                           const int32_t *__restrict__ unit_step0, const int32_t *__restrict__ step_of,
                           const int32_t *__restrict__ bperm, const int32_t *__restrict__ ppos,
                           const int2 *__restrict__ steps, const int32_t *__restrict__ tri_ptr,
                           const int32_t *__restrict__ tri_col, const T *__restrict__ tri_val,
                           const T *__restrict__ invd_row, const int32_t *__restrict__ ovf_ptr,
                           unsigned char *__restrict__ recs, int32_t *__restrict__ ovf_col, T *__restrict__ ovf_val) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int s = step_of[p];
    const int lane = p - steps[s].x;
    const int row = bperm[p];
    const int u = unit[row];
    unsigned char *base = recs + (size_t)s * rec_bytes(W, sizeof(T));
    reinterpret_cast<int32_t *>(base)[lane] = row;
    reinterpret_cast<T *>(base + rec_invd(W))[lane] = invd_row[row];
    int32_t *cols = reinterpret_cast<int32_t *>(base + rec_cols(W));
    T *vals = reinterpret_cast<T *>(base + rec_vals(W, sizeof(T)));
    const int step_end_pp = (s - unit_step0[u] + 1) * 32;        // padded end of the consumer's step
    int k = 0;
    for (int kk = tri_ptr[row]; kk < tri_ptr[row + 1]; ++kk, ++k) {
        const int j = tri_col[kk];
        const int uj = unit[j];
        int code = j;                                    // global: another CTA, or left the ring
        if (uj / kWPC == u / kWPC) {
            const int pj = ppos[j];
            const bool ring_ok = (uj == u) ? (pj + Wu >= step_end_pp)            // overwritten later than now
                                           : ((unit_step0[uj + 1] - unit_step0[uj]) * 32 <= Wu);   // never overwritten
            if (ring_ok) code = -1 - ((uj % kWPC) * Wu + (pj & (Wu - 1)));
        }
        if (k < W) {
            cols[k * 32 + lane] = code;
            vals[k * 32 + lane] = tri_val[kk];
        } else {
            const int o = ovf_ptr[p] + (k - W);
            ovf_col[o] = code;
            ovf_val[o] = tri_val[kk];
        }
    }
    for (; k < W; ++k) {
        cols[k * 32 + lane] = -1 - Z;
        vals[k * 32 + lane] = T(0);
    }
}

// ------------------------------------------------------------------ solve
__device__ __forceinline__ double lds_volatile(const double *p) {
    double v;
    asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"(smem_u32(p)));
    return v;
}
__device__ __forceinline__ float lds_volatile(const float *p) {
    float v;
    asm volatile("ld.volatile.shared.f32 %0, [%1];" : "=f"(v) : "r"(smem_u32(p)));
    return v;
}

// Spin watchdog: a wait that exceeds ~4 s (a scheduling bug, never expected
// on valid input) sets g_watchdog and gives up instead of hanging the GPU.
__device__ unsigned g_watchdog = 0;
__device__ __forceinline__ unsigned long long wd_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __noinline__ bool wd_expired(unsigned long long t0) {
    if (*(volatile unsigned *)&g_watchdog) return true;      // another wait already gave up
    if (wd_now() - t0 > 4000000000ull) {
        atomicExch(&g_watchdog, 1u);
        return true;
    }
    return false;
}

template <typename T>
__device__ __noinline__ T poll_smem_slow(const T *p) {
    const unsigned long long t0 = wd_now();
    T v = lds_volatile(p);
    unsigned it = 0;
    while (Sentinel<T>::is(v)) {
        __nanosleep(kSleepSmemNs);       // leave the shared-memory pipe to the working warps
        v = lds_volatile(p);
        if ((++it & 1023u) == 0 && wd_expired(t0)) break;
    }
    return v;
}
template <typename T>
__device__ __noinline__ T poll_global_slow(const T *p) {
    const unsigned long long t0 = wd_now();
    T v = ld_relaxed_val(p);
    unsigned it = 0;
    while (Sentinel<T>::is(v)) {
        __nanosleep(kSleepGlobalNs);
        v = ld_relaxed_val(p);
        if ((++it & 1023u) == 0 && wd_expired(t0)) break;
    }
    return v;
}

// Debug-only timeline hook (sptrsv_dbg_block_trace): lane 0 of every warp
// records %globaltimer at its first `cap` - 1 steps and at the end.
__device__ unsigned long long *g_trace = nullptr;
__device__ int g_trace_cap = 0;
__device__ unsigned long long *g_phase = nullptr;     // TRACE build: warp 0, 5 clock64 stamps x 128 steps
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <typename T, int MAXW>
struct Lead {
    int row;
    T bv;
    T xv[MAXW];
};

// One warp = one tile of rows; lane = row of the current step.  Per step s:
//   lead   (record s+2 is here) row, b and the speculative external x of step
//          s+2 into a register set; 3 sets rotate by unrolling, never by moves;
//   ring   lane 0 refills the record ring (TMA, record s+nst-1); b of step
//          s+6 is prefetched into L2 if its record has landed;
//   solve  deps from shared slots (polled: written by this warp before the
//          last __syncwarp, or by a neighbour warp) or the speculative value
//          (re-polled from L2 only if it was still the sentinel); FMA chain;
//          result to the warp's slot and to x; __syncwarp.
template <typename T, bool UNIT, int MAXW, bool TRACE>
__global__ void __launch_bounds__(32 * kWPC, 1)
    k_block(int Wu, int W, int nst, const int32_t *__restrict__ unit_step0, const unsigned char *__restrict__ recs,
            const int32_t *__restrict__ ovf_ptr, const int32_t *__restrict__ ovf_col,
            const T *__restrict__ ovf_val, const int32_t *__restrict__ ovf_pos, const T *b, T *x) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int REC = rec_bytes(W, sizeof(T));
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw) + warp * nst;
    unsigned char *ring = smem_raw + 8 * (size_t)kWPC * nst + (size_t)warp * nst * REC;
    T *xs = reinterpret_cast<T *>(smem_raw + 8 * (size_t)kWPC * nst + (size_t)kWPC * nst * REC);
    for (int i = threadIdx.x; i <= kWPC * Wu; i += blockDim.x) xs[i] = (i == kWPC * Wu) ? T(0) : Sentinel<T>::value();
    const int u = blockIdx.x * kWPC + warp;
    const int s0 = unit_step0[u], s1 = unit_step0[u + 1];
    if (lane == 0) {
        for (int i = 0; i < nst; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (s0 == s1) return;
    T *myslots = xs + warp * Wu;
    const int cW = rec_cols(W), iW = rec_invd(W), vW = rec_vals(W, sizeof(T));
    auto slot_of = [&](int s) { return ring + (size_t)((s - s0) & (nst - 1)) * REC; };
    auto issue = [&](int s) {     // lane 0
        uint64_t *bar = &bars[(s - s0) & (nst - 1)];
        mbar_arrive_expect_tx(bar, (uint32_t)REC);
        bulk_g2s(slot_of(s), recs + (size_t)s * REC, (uint32_t)REC, bar);
    };
    auto wait = [&](int s) {
        const int i = s - s0;
        uint64_t *bar = &bars[i & (nst - 1)];
        const uint32_t par = (uint32_t)((i / nst) & 1);
        if (!mbar_try_wait(bar, par)) {
            const unsigned long long t0 = wd_now();
            while (!mbar_try_wait(bar, par))
                if (wd_expired(t0)) break;
        }
    };
    auto lead = [&](Lead<T, MAXW> &L, int s) {          // record s has landed
        const unsigned char *r = slot_of(s);
        L.row = reinterpret_cast<const int32_t *>(r)[lane];
        if (L.row >= 0) L.bv = ld_cg(b + L.row);
        const int32_t *cols = reinterpret_cast<const int32_t *>(r + cW);
#pragma unroll
        for (int k = 0; k < MAXW; ++k) {
            if (k < W) {
                const int c = cols[k * 32 + lane];
                if (c >= 0) L.xv[k] = ld_relaxed_val(x + c);
            }
        }
    };
    auto solve = [&](const Lead<T, MAXW> &L, int s) {
        const unsigned char *r = slot_of(s);
        if (L.row >= 0) {
            const int32_t *cols = reinterpret_cast<const int32_t *>(r + cW);
            const T *vals = reinterpret_cast<const T *>(r + vW);
            T acc = L.bv;
#pragma unroll
            for (int k = 0; k < MAXW; ++k) {
                if (k < W) {
                    const int c = cols[k * 32 + lane];
                    T v;
                    if (c < 0) {
                        v = lds_volatile(xs - 1 - c);
                        if (Sentinel<T>::is(v)) v = poll_smem_slow(xs - 1 - c);
                    } else {
                        v = L.xv[k];
                        if (Sentinel<T>::is(v)) v = poll_global_slow(x + c);
                    }
                    acc = fnma(vals[k * 32 + lane], v, acc);
                }
            }
            if (MAXW >= kTprMax && W == kTprMax) {
                const int p = ovf_pos[L.row];
                for (int o = ovf_ptr[p]; o < ovf_ptr[p + 1]; ++o) {
                    const int c = ovf_col[o];
                    T v = c < 0 ? lds_volatile(xs - 1 - c) : ld_relaxed_val(x + c);
                    if (Sentinel<T>::is(v)) v = c < 0 ? poll_smem_slow(xs - 1 - c) : poll_global_slow(x + c);
                    acc = fnma(ovf_val[o], v, acc);
                }
            }
            const T res = Sentinel<T>::scrub(UNIT ? acc : acc * reinterpret_cast<const T *>(r + iW)[lane]);
            myslots[(((s - s0) << 5) + lane) & (Wu - 1)] = res;
            st_relaxed_val(x + L.row, res);
        }
        __syncwarp();
    };
    if (lane == 0)
        for (int s = s0; s < min(s1, s0 + nst - 1); ++s) issue(s);
    Lead<T, MAXW> L0, L1, L2;
    wait(s0);
    lead(L0, s0);
    if (s0 + 1 < s1) {
        wait(s0 + 1);
        lead(L1, s0 + 1);
    }
#define SPTRSV_BLOCK_STEP(CUR, NXT, OFF)                                                        \
    {                                                                                           \
        const int ss = s + (OFF);                                                               \
        if (ss >= s1) break;                                                                    \
        if (TRACE && lane == 0 && ss - s0 < g_trace_cap - 1)                                    \
            g_trace[(size_t)u * g_trace_cap + (ss - s0)] = gtimer();                            \
        unsigned long long *ph = (TRACE && g_phase && u == 0 && lane == 0 && ss - s0 < 128)     \
                                     ? g_phase + 5 * (ss - s0) : nullptr;                       \
        if (ph) ph[0] = clock64();                                                              \
        if (ss + kLead < s1) {                                                                  \
            wait(ss + kLead);                                                                   \
            if (ph) ph[1] = clock64();                                                          \
            lead(NXT, ss + kLead);                                                              \
        }                                                                                       \
        if (ph) ph[2] = clock64();                                                              \
        if (lane == 0 && ss + nst - 1 < s1) issue(ss + nst - 1);                                \
        if (ph) ph[3] = clock64();                                                              \
        if (ss + kPrefB < s1) {                                                                 \
            const int i6 = ss + kPrefB - s0;                                                    \
            if (mbar_test_wait(&bars[i6 & (nst - 1)], (uint32_t)((i6 / nst) & 1))) {            \
                const int rw = reinterpret_cast<const int32_t *>(slot_of(ss + kPrefB))[lane];   \
                if (rw >= 0) prefetch_l2(b + rw);                                               \
            }                                                                                   \
        }                                                                                       \
        solve(CUR, ss);                                                                         \
        if (ph) ph[4] = clock64();                                                              \
    }
    for (int s = s0; s < s1; s += 3) {
        SPTRSV_BLOCK_STEP(L0, L2, 0)
        SPTRSV_BLOCK_STEP(L1, L0, 1)
        SPTRSV_BLOCK_STEP(L2, L1, 2)
    }
#undef SPTRSV_BLOCK_STEP
    if (TRACE && lane == 0) g_trace[(size_t)u * g_trace_cap + min(s1 - s0, g_trace_cap - 1)] = gtimer();
}

template <typename T>
__global__ void k_bprefill(T *x, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (; i < n; i += stride) x[i] = Sentinel<T>::value();
}

int env_int(const char *name, int dflt) {
    const char *v = getenv(name);
    return (v && *v) ? atoi(v) : dflt;
}

template <typename T, bool UNIT>
void *pick_kernel(int W, bool trace) {
    if (trace) {
        if (W <= 4) return (void *)k_block<T, UNIT, 4, true>;
        if (W <= 8) return (void *)k_block<T, UNIT, 8, true>;
        return (void *)k_block<T, UNIT, kTprMax, true>;
    }
    if (W <= 4) return (void *)k_block<T, UNIT, 4, false>;
    if (W <= 8) return (void *)k_block<T, UNIT, 8, false>;
    return (void *)k_block<T, UNIT, kTprMax, false>;
}
bool g_host_trace = false;

// Structured-grid detection: candidates (nx, nx*ny) from the dependency
// offsets of an interior row, each verified on every dependency on the GPU.
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
    std::vector<std::pair<int, int>> cand;
    for (int64_t a : offs)
        for (int da = -1; da <= 1; ++da) {
            const int64_t nx = a + da;
            if (nx < 2 || nx >= n) continue;
            for (int64_t c : offs)
                for (int dc = -1; dc <= 1; ++dc)
                    for (int dn = -1; dn <= 1; ++dn) {
                        const int64_t nxy = c + dc + dn * nx;
                        if (nxy <= nx || nxy % nx != 0 || n % nxy != 0) continue;
                        cand.emplace_back((int)nx, (int)(nxy / nx));
                    }
        }
    std::sort(cand.begin(), cand.end());
    cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
    if (cand.size() > 24) cand.resize(24);
    unsigned *bad = nullptr;
    sptrsv_status_t st;
    if ((st = tmp.alloc_n(&bad, 1)) != SPTRSV_SUCCESS) return st;
    for (auto &c : cand) {
        const int nz = n / (c.first * c.second);
        if (nz < 2 || c.second < 2) continue;
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

}  // namespace

sptrsv_status_t block_build(sptrsv_handle_t h, cudaStream_t s) {
    BlockPlan &B = h->block;
    const int n = h->n;
    const int nlev = h->info.nlev;
    DevArena tmp;
    struct Guard {
        DevArena &a;
        ~Guard() { a.release_all(); }
    } guard{tmp};
    sptrsv_status_t st;
    const size_t es = h->esize;
    int max_smem = 0;
    SPTRSV_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
    const int eg = (n + 255) / 256;

    // ---- 1. natural-order CSR of the triangle
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

    // ---- 2. partition rows over U = K x kWPC warps of K co-resident CTAs
    int32_t *unit = nullptr;
    if ((st = tmp.alloc_n(&unit, n)) != SPTRSV_SUCCESS) return st;
    int Kmax = env_int("SPTRSV_BLOCK_K", 0);
    const int min_rows = env_int("SPTRSV_BLOCK_MIN_ROWS", 8192);
    if (Kmax <= 0) Kmax = (int)std::max<int64_t>(1, std::min<int64_t>(h->num_sms, n / std::max(1, min_rows)));
    Kmax = std::min(Kmax, h->num_sms);
    int K = Kmax;
    int gnx = 0, gny = 0;
    if (Kmax > 1 && !env_int("SPTRSV_BLOCK_NO_GRID", 0)) {
        if ((st = detect_grid(h, tri_ptr, tri_col, tmp, s, gnx, gny)) != SPTRSV_SUCCESS) return st;
    }
    if (gnx > 0) {
        // CTA grid cxn x cyn (2x2 tiles each): prefer tiles of <= 32 columns (one
        // step per level), then more CTAs, then square tiles
        int best = -1, bcx = 0, bcy = 0;
        double bscore = -1e30;
        for (int cx = 1; cx <= std::min(Kmax, gnx / 2); ++cx)
            for (int cy = 1; cy <= std::min(Kmax / cx, gny / 2); ++cy) {
                const int tw = (gnx + 2 * cx - 1) / (2 * cx), th = (gny + 2 * cy - 1) / (2 * cy);
                const bool fits = tw * th <= 32;
                const double score = (fits ? 1e6 : 0.0) + cx * cy * 10.0 - std::fabs(std::log((double)tw / th));
                if (score > bscore) {
                    bscore = score;
                    best = 1;
                    bcx = cx;
                    bcy = cy;
                }
            }
        if (best < 0) {
            gnx = 0;
        } else {
            K = bcx * bcy;
            k_part_tiles<<<eg, 256, 0, s>>>(n, gnx, gny, bcx, bcy, unit);
            B.grid_nx = gnx;
            B.grid_ny = gny;
            B.tiles_x = 2 * bcx;
            B.tiles_y = 2 * bcy;
        }
    }
    const int U = K * kWPC;
    if (gnx == 0) k_part_natural<<<eg, 256, 0, s>>>(n, U, h->uplo, unit);
    SPTRSV_CUDA(cudaGetLastError());
    B.nblocks = K;
    B.nunits = U;
    if ((uint64_t)U * (uint64_t)nlev * kBuckets >= (1ull << 32)) return SPTRSV_ERR_NOT_SUPPORTED;

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
    int32_t ngroups = 0;
    SPTRSV_CUDA(cudaMemcpyAsync(&ngroups, gid + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    int32_t *gp0 = nullptr, *nsub = nullptr, *sub0 = nullptr;
    if ((st = tmp.alloc_n(&gp0, (size_t)ngroups + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&nsub, (size_t)ngroups + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&sub0, (size_t)ngroups + 1)) != SPTRSV_SUCCESS) return st;
    const int gg = (ngroups + 1 + 255) / 256;
    k_group_start<<<eg, 256, 0, s>>>(head, gid, n, ngroups, gp0);
    k_group_sub<<<gg, 256, 0, s>>>(gp0, ngroups, nsub);
    if ((st = exclusive_scan_i32(nsub, sub0, (int64_t)ngroups + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    int32_t nsteps = 0;
    SPTRSV_CUDA(cudaMemcpyAsync(&nsteps, sub0 + ngroups, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    B.nsteps = nsteps;
    int2 *steps = nullptr;
    int32_t *step_unit = nullptr, *step_of = nullptr, *ppos = nullptr;
    if ((st = tmp.alloc_n(&steps, (size_t)nsteps + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&step_unit, (size_t)nsteps + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&step_of, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&ppos, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&B.d_unit_step0, (size_t)U + 1)) != SPTRSV_SUCCESS) return st;
    k_steps<<<gg, 256, 0, s>>>(gp0, sub0, ngroups, bperm, unit, steps, step_unit);
    k_unit_step0<<<(nsteps + 255) / 256, 256, 0, s>>>(step_unit, nsteps, U, B.d_unit_step0);
    k_pos_step<<<eg, 256, 0, s>>>(head, gid, gp0, sub0, steps, bperm, unit, B.d_unit_step0, n, step_of, ppos);
    SPTRSV_CUDA(cudaGetLastError());

    // ---- 4. record geometry, shared memory (mbarriers | record rings | x slots)
    const int W = std::max(1, std::min(h->info.max_row_deps, kTprMax));
    const int REC = rec_bytes(W, (int)es);
    int nst = 16;
    while (nst > kMinStages && (size_t)kWPC * nst * REC > (size_t)max_smem / 2) nst /= 2;
    const size_t fixed = 8 * (size_t)kWPC * nst + (size_t)kWPC * nst * REC;
    if (fixed + (size_t)(kWPC * 64 + 1) * es > (size_t)max_smem) return SPTRSV_ERR_NOT_SUPPORTED;
    int Wu = 32;
    while ((size_t)(kWPC * 2 * Wu + 1) * es + fixed <= (size_t)max_smem) Wu *= 2;
    const int Wenv = env_int("SPTRSV_BLOCK_SLOTS", 0);
    if (Wenv > 0) {
        int w2 = 32;
        while (w2 * 2 <= Wenv) w2 *= 2;
        Wu = std::min(Wu, w2);
    }
    const int Z = kWPC * Wu;
    B.W = Wu;
    B.nst = nst;
    B.maxw = W;
    B.rec_max = REC;
    B.nent = (int64_t)nsteps * REC;

    // overflow CSR (entries beyond W), by position; row -> position
    int32_t *ocnt = nullptr;
    if ((st = tmp.alloc_n(&ocnt, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&B.d_ovf_ptr, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&B.d_ovf_pos, (size_t)n)) != SPTRSV_SUCCESS) return st;
    k_ovf_count<<<(n + 1 + 255) / 256, 256, 0, s>>>(n, bperm, h->d_dp, W, ocnt);
    if ((st = exclusive_scan_i32(ocnt, B.d_ovf_ptr, (int64_t)n + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemcpyAsync(B.d_ovf_pos, pos, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
    int32_t novf = 0;
    SPTRSV_CUDA(cudaMemcpyAsync(&novf, B.d_ovf_ptr + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    B.novf = novf;

    // ---- 5. records
    if ((st = h->arena.alloc(&B.d_recs, (size_t)std::max<int64_t>((int64_t)nsteps * REC, 16))) != SPTRSV_SUCCESS)
        return st;
    if ((st = h->arena.alloc_n(&B.d_ovf_col, (size_t)std::max(novf, 1))) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc(&B.d_ovf_val, (size_t)std::max(novf, 1) * es)) != SPTRSV_SUCCESS) return st;
    const int pg = (int)(((int64_t)nsteps * 32 + 255) / 256);
    if (h->dtype == SPTRSV_F64) {
        k_rec_pad<double><<<pg, 256, 0, s>>>(nsteps, W, Z, steps, (unsigned char *)B.d_recs);
        k_rec_fill<double><<<eg, 256, 0, s>>>(n, Wu, W, Z, unit, B.d_unit_step0, step_of, bperm, ppos, steps, tri_ptr,
                                             tri_col, (const double *)tri_val, (const double *)h->d_invd_row,
                                             B.d_ovf_ptr, (unsigned char *)B.d_recs, B.d_ovf_col,
                                             (double *)B.d_ovf_val);
    } else {
        k_rec_pad<float><<<pg, 256, 0, s>>>(nsteps, W, Z, steps, (unsigned char *)B.d_recs);
        k_rec_fill<float><<<eg, 256, 0, s>>>(n, Wu, W, Z, unit, B.d_unit_step0, step_of, bperm, ppos, steps, tri_ptr,
                                            tri_col, (const float *)tri_val, (const float *)h->d_invd_row,
                                            B.d_ovf_ptr, (unsigned char *)B.d_recs, B.d_ovf_col,
                                            (float *)B.d_ovf_val);
    }
    SPTRSV_CUDA(cudaGetLastError());

    // ---- launch configuration: K co-resident CTAs of kWPC warps
    const size_t smem = fixed + (size_t)(kWPC * Wu + 1) * es;
    void *kn = nullptr;
    for (int tr = 1; tr >= 0; --tr) {
        if (h->dtype == SPTRSV_F64)
            kn = h->diag == SPTRSV_UNIT ? pick_kernel<double, true>(W, tr) : pick_kernel<double, false>(W, tr);
        else
            kn = h->diag == SPTRSV_UNIT ? pick_kernel<float, true>(W, tr) : pick_kernel<float, false>(W, tr);
        SPTRSV_CUDA(cudaFuncSetAttribute(kn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        if (tr) B.kernel_trace = kn;
    }
    int per_sm = 0;
    SPTRSV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kn, 32 * kWPC, smem));
    if (per_sm * h->num_sms < K) return SPTRSV_ERR_NOT_SUPPORTED;
    B.kernel = kn;
    B.smem = smem;
    B.threads = 32 * kWPC;
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    B.built = true;
    return SPTRSV_SUCCESS;
}

sptrsv_status_t block_solve(sptrsv_handle_t h, const void *b, void *x, cudaStream_t s) {
    BlockPlan &B = h->block;
    if (!B.built) return SPTRSV_ERR_NOT_SUPPORTED;
    const size_t bytes = (size_t)h->n * h->esize;
    if (b == x) {   // in place: keep b aside, x becomes the flag array
        if (h->scratch_bytes < bytes) {
            if (h->d_scratch) {
                SPTRSV_CUDA(cudaStreamSynchronize(s));
                cudaFree(h->d_scratch);
            }
            h->d_scratch = nullptr;
            h->scratch_bytes = 0;
            SPTRSV_CUDA(cudaMalloc(&h->d_scratch, bytes));
            h->scratch_bytes = bytes;
        }
        SPTRSV_CUDA(cudaMemcpyAsync(h->d_scratch, b, bytes, cudaMemcpyDeviceToDevice, s));
        b = h->d_scratch;
    }
    if (h->dtype == SPTRSV_F64)
        k_bprefill<double><<<h->num_sms * 4, 512, 0, s>>>((double *)x, h->n);
    else
        k_bprefill<float><<<h->num_sms * 4, 512, 0, s>>>((float *)x, h->n);
    SPTRSV_CUDA(cudaGetLastError());
    int Wu = B.W, W = B.maxw, nst = B.nst;
    const unsigned char *recs = (const unsigned char *)B.d_recs;
    void *args[] = {(void *)&Wu, (void *)&W, (void *)&nst, (void *)&B.d_unit_step0, (void *)&recs,
                    (void *)&B.d_ovf_ptr, (void *)&B.d_ovf_col, (void *)&B.d_ovf_val, (void *)&B.d_ovf_pos,
                    (void *)&b, (void *)&x};
    SPTRSV_CUDA(cudaLaunchCooperativeKernel(g_host_trace ? B.kernel_trace : B.kernel, B.nblocks, B.threads, args,
                                            B.smem, s));
    return SPTRSV_SUCCESS;
}

}  // namespace sptrsv

// Debug hook (not part of include/sptrsv.h): install a device trace buffer of
// (#warps) x cap uint64 timestamps for SPTRSV_ALGO_BLOCK solves (NULL disables).
extern "C" int sptrsv_dbg_block_phase(void *dev_buf) {
    unsigned long long *p = (unsigned long long *)dev_buf;
    return cudaMemcpyToSymbol(sptrsv::g_phase, &p, sizeof(p)) == cudaSuccess ? 0 : 5;
}

extern "C" int sptrsv_dbg_block_trace(void *dev_buf, int cap) {
    unsigned long long *p = (unsigned long long *)dev_buf;
    if (cudaMemcpyToSymbol(sptrsv::g_trace, &p, sizeof(p)) != cudaSuccess) return 5;
    if (cudaMemcpyToSymbol(sptrsv::g_trace_cap, &cap, sizeof(int)) != cudaSuccess) return 5;
    sptrsv::g_host_trace = (dev_buf != nullptr);
    return 0;
}

// Debug hook: returns and clears the spin-watchdog flag (1 = a wait gave up).
extern "C" int sptrsv_dbg_watchdog(void) {
    unsigned v = 0, z = 0;
    cudaMemcpyFromSymbol(&v, sptrsv::g_watchdog, sizeof(v));
    cudaMemcpyToSymbol(sptrsv::g_watchdog, &z, sizeof(z));
    return (int)v;
}
