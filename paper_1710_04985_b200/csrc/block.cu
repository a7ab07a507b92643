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
// Step records (global, 16-byte aligned), streamed per warp into a shared-memory
// ring by TMA bulk copies (cp.async.bulk + mbarrier), nst records in flight:
//   int4 {p0, nr, w, bytes} | int4 {off_lo, off_hi, bytes, 0} of the record
//   this warp fetches when it consumes this one | int32 rows[nr] |
//   int32 cols[w][nr] | T invd[nr] | T vals[w][nr]   (arrays padded to 16 B)
//   cols >= 0: global column; cols < 0: shared slot -1-cols (the warp's
//   zero slot pads short rows).  Entries beyond kTprMax: ovf_* (CSR by position).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "internal.h"

namespace sptrsv {
namespace {

constexpr int kWPC = 4;          // warps (tiles) per CTA
constexpr int kBuckets = kTprMax + 2;
constexpr int kAheadB = 6;       // lead of the b loads (steps)
constexpr int kAheadX = 2;       // lead of the speculative external x loads
constexpr int kBRing = kAheadB + 2;   // per-warp shared ring of b values [kBRing][32]
constexpr int kXRing = kAheadX + 2;   // per-warp shared ring of speculative x [kXRing][MAXW][32]
constexpr int kMinStages = 8;    // records in flight per warp (> kAheadB + 1, or the lookahead deadlocks)
static_assert(kMinStages >= kAheadB + 2 && kMinStages >= kAheadX + 2, "record ring shorter than the lookahead");

__device__ __forceinline__ uint32_t bucket_of(int deps) { return deps > kTprMax ? 0u : (uint32_t)(kTprMax + 1 - deps); }
__host__ __device__ __forceinline__ int64_t a16(int64_t v) { return (v + 15) & ~(int64_t)15; }
__host__ __device__ __forceinline__ int64_t rec_bytes(int nr, int w, int es) {
    return 32 + a16(4ll * nr) + a16(4ll * w * nr) + a16((int64_t)es * nr) + a16((int64_t)es * w * nr);
}

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

// (x, y) tiles: CTA (cx, cy) owns the 2x2 tiles (2cx..2cx+1, 2cy..2cy+1)
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

// head flags of groups (new (unit, level)); inverse permutation; unit sizes
__global__ void k_heads(const uint32_t *skeys, const int32_t *bperm, const int32_t *unit, int n, int32_t *head,
                        int32_t *pos, int32_t *unit_rows) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const uint32_t s = skeys[p] / kBuckets;
    head[p] = (p == 0 || skeys[p - 1] / kBuckets != s) ? 1 : 0;
    pos[bperm[p]] = p;
    atomicAdd(&unit_rows[unit[bperm[p]]], 1);
}

__global__ void k_group_start(const int32_t *head, const int32_t *gid, int n, int ngroups, int32_t *gp0) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n && head[p]) gp0[gid[p]] = p;
    if (p == 0) gp0[ngroups] = n;
}

__global__ void k_group_sub(const int32_t *gp0, int ngroups, int rc, int32_t *nsub) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < ngroups) nsub[g] = (gp0[g + 1] - gp0[g] + rc - 1) / rc;
    if (g == ngroups) nsub[g] = 0;
}

// per group: its 32-row sub-steps {p0, nr, w}; unit of each step
__global__ void k_steps(const int32_t *gp0, const int32_t *sub0, int ngroups, int rc, const int32_t *bperm,
                        const int32_t *dp, const int32_t *unit, int4 *steps, int32_t *step_unit, int *maxw) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ngroups) return;
    const int a = gp0[g], e = gp0[g + 1];
    int s = sub0[g];
    const int u = unit[bperm[a]];
    int wmax = 0;
    for (int p0 = a; p0 < e; p0 += rc, ++s) {
        const int w = min(dp[bperm[p0]], kTprMax);      // first row has the most deps
        steps[s] = make_int4(p0, min(rc, e - p0), w, 0);
        step_unit[s] = u;
        wmax = max(wmax, w);
    }
    atomicMax(maxw, wmax);
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

__global__ void k_rec_sizes(const int4 *steps, int nsteps, int es, int64_t *rb, int *rec_max) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < nsteps) {
        const int64_t v = rec_bytes(steps[s].y, steps[s].z, es);
        rb[s] = v;
        atomicMax(rec_max, (int)v);
    }
    if (s == nsteps) rb[s] = 0;
}

__global__ void k_pos_step(const int32_t *head, const int32_t *gid, const int32_t *gp0, const int32_t *sub0, int n,
                           int rc, int32_t *step_of) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int g = gid[p] + head[p] - 1;
    step_of[p] = sub0[g] + (p - gp0[g]) / rc;
}

__global__ void k_ovf_count(int n, const int32_t *bperm, const int32_t *dp, int32_t *ocnt) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) ocnt[p] = max(0, dp[bperm[p]] - kTprMax);
    if (p == n) ocnt[p] = 0;
}

// slot of a produced value: warp-local ring of Wu (power of two) slots
__host__ __device__ __forceinline__ int slot_index(int u, int local, int Wu) {
    return (u % kWPC) * (Wu + 1) + (local & (Wu - 1));
}

template <typename T>
__global__ void k_rec_fill(int n, int Wu, int nst, const int32_t *__restrict__ unit,
                           const int32_t *__restrict__ unit_rows, const int32_t *__restrict__ step_of,
                           const int32_t *__restrict__ bperm, const int32_t *__restrict__ pos,
                           const int4 *__restrict__ steps, const int64_t *__restrict__ rec_off,
                           const int32_t *__restrict__ unit_step0, const int32_t *__restrict__ tri_ptr,
                           const int32_t *__restrict__ tri_col, const T *__restrict__ tri_val,
                           const T *__restrict__ invd_row, const int32_t *__restrict__ ovf_ptr,
                           unsigned char *__restrict__ recs, int32_t *__restrict__ ovf_col, T *__restrict__ ovf_val) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int s = step_of[p];
    const int4 st = steps[s];
    const int nr = st.y, w = st.z, j = p - st.x;
    unsigned char *base = recs + rec_off[s];
    const int row = bperm[p];
    const int u = unit[row];
    if (j == 0) {
        *reinterpret_cast<int4 *>(base) = make_int4(st.x, nr, w, (int)(rec_off[s + 1] - rec_off[s]));
        const int sn = s + nst - 1;
        int4 nx = make_int4(0, 0, 0, 0);
        if (sn < unit_step0[u + 1]) {
            const int64_t off = rec_off[sn];
            nx = make_int4((int)(off & 0xffffffffll), (int)(off >> 32), (int)(rec_off[sn + 1] - off), 0);
        }
        *reinterpret_cast<int4 *>(base + 16) = nx;
    }
    unsigned char *q = base + 32;
    int32_t *rows = reinterpret_cast<int32_t *>(q);
    q += a16(4ll * nr);
    int32_t *cols = reinterpret_cast<int32_t *>(q);
    q += a16(4ll * w * nr);
    T *invd = reinterpret_cast<T *>(q);
    q += a16((int64_t)sizeof(T) * nr);
    T *vals = reinterpret_cast<T *>(q);
    rows[j] = row;
    invd[j] = invd_row[row];
    const int u_p0 = steps[unit_step0[u]].x;
    const int step_end_local = st.x + nr - u_p0;
    int k = 0;
    for (int kk = tri_ptr[row]; kk < tri_ptr[row + 1]; ++kk, ++k) {
        const int jj = tri_col[kk];
        const int uj = unit[jj];
        int code = jj;                                   // global (another CTA, or left the ring)
        if (uj / kWPC == u / kWPC) {
            const int pj = pos[jj];
            const int uj_p0 = steps[unit_step0[uj]].x;
            const int lj = pj - uj_p0;
            if (uj == u) {
                if (lj + Wu >= step_end_local) code = -1 - slot_index(uj, lj, Wu);
            } else if (unit_rows[uj] <= Wu) {            // no slot reuse in the producer warp
                code = -1 - slot_index(uj, lj, Wu);
            }
        }
        if (k < w) {
            cols[k * nr + j] = code;
            vals[k * nr + j] = tri_val[kk];
        } else {
            const int o = ovf_ptr[p] + (k - w);
            ovf_col[o] = code;
            ovf_val[o] = tri_val[kk];
        }
    }
    for (; k < w; ++k) {
        cols[k * nr + j] = -1 - ((u % kWPC) * (Wu + 1) + Wu);    // the warp's zero slot
        vals[k * nr + j] = T(0);
    }
}

// ------------------------------------------------------------------ solve
template <typename T>
struct RecView {
    int4 hdr;
    int4 nxt;
    const int32_t *rows;
    const int32_t *cols;
    const T *invd;
    const T *vals;
    RecView() = default;
    __device__ __forceinline__ RecView(const unsigned char *base) {
        hdr = *reinterpret_cast<const int4 *>(base);
        nxt = *reinterpret_cast<const int4 *>(base + 16);
        const int nr = hdr.y, w = hdr.z;
        const unsigned char *q = base + 32;
        rows = reinterpret_cast<const int32_t *>(q);
        q += a16(4ll * nr);
        cols = reinterpret_cast<const int32_t *>(q);
        q += a16(4ll * w * nr);
        invd = reinterpret_cast<const T *>(q);
        q += a16((int64_t)sizeof(T) * nr);
        vals = reinterpret_cast<const T *>(q);
    }
};

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
__device__ __forceinline__ T poll_smem(const T *p) {
    T v = lds_volatile(p);
    if (Sentinel<T>::is(v)) {
        const unsigned long long t0 = wd_now();
        unsigned it = 0;
        while (Sentinel<T>::is(v)) {
            v = lds_volatile(p);
            if ((++it & 4095u) == 0 && wd_expired(t0)) break;
        }
    }
    return v;
}
template <typename T>
__device__ __forceinline__ T poll_global(const T *p, T v) {
    if (Sentinel<T>::is(v)) {
        const unsigned long long t0 = wd_now();
        unsigned it = 0;
        while (Sentinel<T>::is(v)) {
            __nanosleep(8);
            v = ld_relaxed_val(p);
            if ((++it & 1023u) == 0 && wd_expired(t0)) break;
        }
    }
    return v;
}

// Debug-only timeline hook (sptrsv_dbg_block_trace): lane 0 of every warp
// records %globaltimer at its first `cap` - 1 steps and at the end.
__device__ unsigned long long *g_trace = nullptr;
__device__ int g_trace_cap = 0;
__device__ unsigned long long *g_phase = nullptr;     // TRACE build: warp 0, 4 clock64 stamps x 128 steps

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Register state of one step, loaded two steps ahead (record view, b, and
// the speculative external x).  The loop is unrolled by two over two such
// sets, so no register is ever moved and no load latency lands on the step.
template <typename T, int MAXW>
struct StepRegs {
    RecView<T> r;
    T bv;
    T xv[MAXW];
};

// Per warp, per step s (lane = row of the step):
//   lookahead  record s+2 (wait), issue b and speculative external x loads of
//              step s+2 into the other register set; L2-prefetch b of step
//              s+6 if its record has landed; lane 0 refills the record ring;
//   solve      deps from shared slots (polled) or the speculative value
//              (re-polled from L2 only if still the sentinel); FMA chain;
//              result to this warp's slot and to x; __syncwarp.
template <typename T, bool UNIT, int MAXW, bool TRACE>
__global__ void __launch_bounds__(32 * kWPC, 1)
    k_block(int Wu, int nst, int rec_max, const int32_t *__restrict__ unit_step0, const int64_t *__restrict__ rec_off,
            const unsigned char *__restrict__ recs, const int32_t *__restrict__ ovf_ptr,
            const int32_t *__restrict__ ovf_col, const T *__restrict__ ovf_val, const T *b, T *x) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw) + warp * nst;
    unsigned char *ring = smem_raw + 8 * (size_t)kWPC * nst + (size_t)warp * nst * rec_max;
    T *xs = reinterpret_cast<T *>(smem_raw + 8 * (size_t)kWPC * nst + (size_t)kWPC * nst * rec_max);
    // sentinel-prefill every slot (zero slot = 0), then make it CTA-visible
    for (int i = threadIdx.x; i < kWPC * (Wu + 1); i += blockDim.x)
        xs[i] = (i % (Wu + 1) == Wu) ? T(0) : Sentinel<T>::value();
    const int u = blockIdx.x * kWPC + warp;
    const int s0 = unit_step0[u], s1 = unit_step0[u + 1];
    if (lane == 0) {
        for (int i = 0; i < nst; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (s0 == s1) return;
    auto issue_at = [&](int s, int64_t off, uint32_t bytes) {     // lane 0 only
        const int slot = (s - s0) & (nst - 1);
        mbar_arrive_expect_tx(&bars[slot], bytes);
        bulk_g2s(ring + (size_t)slot * rec_max, recs + off, bytes, &bars[slot]);
    };
    auto wait_rec = [&](int s) {
        const int i = s - s0;
        uint64_t *bar = &bars[i & (nst - 1)];
        const uint32_t par = (uint32_t)((i / nst) & 1);
        if (!mbar_try_wait(bar, par)) {
            const unsigned long long t0 = wd_now();
            while (!mbar_try_wait(bar, par))
                if (wd_expired(t0)) break;
        }
        return RecView<T>(ring + (size_t)(i & (nst - 1)) * rec_max);
    };
    auto load_regs = [&](StepRegs<T, MAXW> &R, int s) {
        R.r = wait_rec(s);
        if (lane < R.r.hdr.y) {
            R.bv = ld_cg(b + R.r.rows[lane]);
#pragma unroll
            for (int k = 0; k < MAXW; ++k) {
                if (k < R.r.hdr.z) {
                    const int c = R.r.cols[k * R.r.hdr.y + lane];
                    if (c >= 0) R.xv[k] = ld_relaxed_val(x + c);
                }
            }
        }
    };
    auto prefetch_b = [&](int s) {      // L2 warm-up of b, only if the record already landed
        const int i = s - s0;
        if (mbar_test_wait(&bars[i & (nst - 1)], (uint32_t)((i / nst) & 1))) {
            const unsigned char *base = ring + (size_t)(i & (nst - 1)) * rec_max;
            const int nr = reinterpret_cast<const int4 *>(base)->y;
            if (lane < nr) prefetch_l2(b + reinterpret_cast<const int32_t *>(base + 32)[lane]);
        }
    };
    if (lane == 0)
        for (int s = s0; s < min(s1, s0 + nst - 1); ++s) issue_at(s, rec_off[s], (uint32_t)(rec_off[s + 1] - rec_off[s]));
    const int u_p0 = wait_rec(s0).hdr.x;
    auto solve = [&](StepRegs<T, MAXW> &R, int s) {
        const RecView<T> &r = R.r;
        if (lane == 0 && r.nxt.z != 0) {
            // slot (s-1) % nst: every lane finished reading it before the last __syncwarp
            issue_at(s + nst - 1, (int64_t)(uint32_t)r.nxt.x | ((int64_t)r.nxt.y << 32), (uint32_t)r.nxt.z);
        }
        const int nr = r.hdr.y, w = r.hdr.z;
        if (lane < nr) {
            T acc = R.bv;
#pragma unroll
            for (int k = 0; k < MAXW; ++k) {
                if (k < w) {
                    const int c = r.cols[k * nr + lane];
                    const T v = c < 0 ? poll_smem(xs - 1 - c) : poll_global(x + c, R.xv[k]);
                    acc = fnma(r.vals[k * nr + lane], v, acc);
                }
            }
            const int p = r.hdr.x + lane;
            if (MAXW >= kTprMax && w == kTprMax) {
                for (int o = ovf_ptr[p]; o < ovf_ptr[p + 1]; ++o) {
                    const int c = ovf_col[o];
                    const T v = c < 0 ? poll_smem(xs - 1 - c) : poll_global(x + c, ld_relaxed_val(x + c));
                    acc = fnma(ovf_val[o], v, acc);
                }
            }
            const T res = Sentinel<T>::scrub(UNIT ? acc : acc * r.invd[lane]);
            xs[slot_index(u, p - u_p0, Wu)] = res;
            st_relaxed_val(x + r.rows[lane], res);
        }
        __syncwarp();
    };
    // three register sets with fixed roles in a 3x unrolled loop (lead 2, no moves)
    StepRegs<T, MAXW> X0, X1, X2;
    load_regs(X0, s0);
    if (s0 + 1 < s1) load_regs(X1, s0 + 1);
#define SPTRSV_BLOCK_STEP(CUR, NXT, OFF)                                                              \
    {                                                                                                 \
        const int ss = s + (OFF);                                                                     \
        if (ss >= s1) break;                                                                          \
        if (TRACE && lane == 0 && ss - s0 < g_trace_cap - 1)                                          \
            g_trace[(size_t)u * g_trace_cap + (ss - s0)] = gtimer();                                  \
        unsigned long long *ph = (TRACE && g_phase && u == 0 && lane == 0 && ss - s0 < 128)            \
                                     ? g_phase + 4 * (ss - s0) : nullptr;                             \
        if (ph) ph[0] = clock64();                                                                    \
        if (ss + 2 < s1) load_regs(NXT, ss + 2);                                                      \
        if (ph) ph[1] = clock64();                                                                    \
        if (ss + 6 < s1) prefetch_b(ss + 6);                                                          \
        if (ph) ph[2] = clock64();                                                                    \
        solve(CUR, ss);                                                                               \
        if (ph) ph[3] = clock64();                                                                    \
    }
    for (int s = s0; s < s1; s += 3) {
        SPTRSV_BLOCK_STEP(X0, X2, 0)
        SPTRSV_BLOCK_STEP(X1, X0, 1)
        SPTRSV_BLOCK_STEP(X2, X1, 2)
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
void *pick_kernel(int maxw, bool trace) {
    if (trace) {
        if (maxw <= 4) return (void *)k_block<T, UNIT, 4, true>;
        if (maxw <= 8) return (void *)k_block<T, UNIT, 8, true>;
        return (void *)k_block<T, UNIT, kTprMax, true>;
    }
    if (maxw <= 4) return (void *)k_block<T, UNIT, 4, false>;
    if (maxw <= 8) return (void *)k_block<T, UNIT, 8, false>;
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
    int K = env_int("SPTRSV_BLOCK_K", 0);
    const int min_rows = env_int("SPTRSV_BLOCK_MIN_ROWS", 8192);
    if (K <= 0) K = (int)std::max<int64_t>(1, std::min<int64_t>(h->num_sms, n / std::max(1, min_rows)));
    K = std::min(K, h->num_sms);
    int gnx = 0, gny = 0;
    if (K > 1 && !env_int("SPTRSV_BLOCK_NO_GRID", 0)) {
        if ((st = detect_grid(h, tri_ptr, tri_col, tmp, s, gnx, gny)) != SPTRSV_SUCCESS) return st;
    }
    if (gnx > 0) {
        // cxn x cyn CTAs (each 2x2 tiles), tiles of aspect ~1
        const int cxn = std::max(1, std::min(gnx / 2, (int)std::sqrt((double)K * gnx / gny)));
        const int cyn = std::max(1, std::min(gny / 2, K / cxn));
        if (2 * cxn > gnx || 2 * cyn > gny) {
            gnx = 0;
        } else {
            K = cxn * cyn;
            k_part_tiles<<<eg, 256, 0, s>>>(n, gnx, gny, cxn, cyn, unit);
            B.grid_nx = gnx;
            B.grid_ny = gny;
            B.tiles_x = 2 * cxn;
            B.tiles_y = 2 * cyn;
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
    int32_t *pos = nullptr, *head = nullptr, *gid = nullptr, *bperm = nullptr, *unit_rows = nullptr;
    if ((st = tmp.alloc_n(&keys, n)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&skeys, n)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&pos, n)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&head, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&gid, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&bperm, n)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&unit_rows, (size_t)U + 1)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemsetAsync(unit_rows, 0, sizeof(int32_t) * ((size_t)U + 1), s));
    k_unit_keys<<<eg, 256, 0, s>>>(n, nlev, unit, h->d_lev, h->d_dp, keys);
    if ((st = radix_sort_pairs(keys, nullptr, skeys, bperm, n, (uint32_t)((uint64_t)U * nlev * kBuckets - 1), tmp,
                               s)) != SPTRSV_SUCCESS)
        return st;
    SPTRSV_CUDA(cudaMemsetAsync(head + n, 0, sizeof(int32_t), s));
    k_heads<<<eg, 256, 0, s>>>(skeys, bperm, unit, n, head, pos, unit_rows);
    if ((st = exclusive_scan_i32(head, gid, (int64_t)n + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    int32_t ngroups = 0;
    SPTRSV_CUDA(cudaMemcpyAsync(&ngroups, gid + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    int32_t *gp0 = nullptr, *nsub = nullptr, *sub0 = nullptr;
    int *d_stats = nullptr;     // [0] max width, [1] max record bytes
    if ((st = tmp.alloc_n(&gp0, (size_t)ngroups + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&nsub, (size_t)ngroups + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&sub0, (size_t)ngroups + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&d_stats, 4)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemsetAsync(d_stats, 0, 4 * sizeof(int), s));
    const int gg = (ngroups + 1 + 255) / 256;
    k_group_start<<<eg, 256, 0, s>>>(head, gid, n, ngroups, gp0);
    // rows per step: 32 (one per lane) unless the records would not leave room
    // for >= kMinStages of them per warp in half the shared memory
    const int maxw_all = std::min(h->info.max_row_deps, kTprMax);
    int rc = 32;
    while (rc > 4 && (size_t)kWPC * kMinStages * a16(rec_bytes(rc, maxw_all, (int)es)) > (size_t)max_smem / 2) rc /= 2;
    B.rows_per_step = rc;
    k_group_sub<<<gg, 256, 0, s>>>(gp0, ngroups, rc, nsub);
    if ((st = exclusive_scan_i32(nsub, sub0, (int64_t)ngroups + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    int32_t nsteps = 0;
    SPTRSV_CUDA(cudaMemcpyAsync(&nsteps, sub0 + ngroups, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    B.nsteps = nsteps;
    int4 *steps = nullptr;
    int32_t *step_unit = nullptr, *step_of = nullptr;
    int64_t *rb = nullptr;
    if ((st = tmp.alloc_n(&steps, (size_t)nsteps + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&step_unit, (size_t)nsteps + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&step_of, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&rb, (size_t)nsteps + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&B.d_unit_step0, (size_t)U + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&B.d_rec_off, (size_t)nsteps + 1)) != SPTRSV_SUCCESS) return st;
    k_steps<<<gg, 256, 0, s>>>(gp0, sub0, ngroups, rc, bperm, h->d_dp, unit, steps, step_unit, d_stats);
    k_unit_step0<<<(nsteps + 255) / 256, 256, 0, s>>>(step_unit, nsteps, U, B.d_unit_step0);
    k_rec_sizes<<<(nsteps + 1 + 255) / 256, 256, 0, s>>>(steps, nsteps, (int)es, rb, d_stats + 1);
    if ((st = exclusive_scan_i64(rb, B.d_rec_off, (int64_t)nsteps + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    k_pos_step<<<eg, 256, 0, s>>>(head, gid, gp0, sub0, n, rc, step_of);
    SPTRSV_CUDA(cudaGetLastError());
    int64_t rec_total = 0;
    int hstats[4];
    SPTRSV_CUDA(cudaMemcpyAsync(&rec_total, B.d_rec_off + nsteps, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SPTRSV_CUDA(cudaMemcpyAsync(hstats, d_stats, 4 * sizeof(int), cudaMemcpyDeviceToHost, s));
    std::vector<int32_t> hunit_rows((size_t)U);
    SPTRSV_CUDA(cudaMemcpyAsync(hunit_rows.data(), unit_rows, sizeof(int32_t) * U, cudaMemcpyDeviceToHost, s));
    // overflow CSR (entries beyond kTprMax), by position
    int32_t *ocnt = nullptr;
    if ((st = tmp.alloc_n(&ocnt, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&B.d_ovf_ptr, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    k_ovf_count<<<(n + 1 + 255) / 256, 256, 0, s>>>(n, bperm, h->d_dp, ocnt);
    if ((st = exclusive_scan_i32(ocnt, B.d_ovf_ptr, (int64_t)n + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    int32_t novf = 0;
    SPTRSV_CUDA(cudaMemcpyAsync(&novf, B.d_ovf_ptr + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    const int maxw = hstats[0];
    const int rec_max = (int)a16(hstats[1]);
    B.maxw = maxw;
    B.rec_max = rec_max;
    B.nent = rec_total;
    B.novf = novf;
    int max_unit_rows = 0;
    for (int v : hunit_rows) max_unit_rows = std::max(max_unit_rows, v);
    B.max_unit_rows = max_unit_rows;

    // ---- 4. shared memory: mbarriers | per-warp record rings | per-warp x slot rings
    int nst = 16;
    while (nst > kMinStages && (size_t)kWPC * nst * rec_max > (size_t)max_smem / 2) nst /= 2;
    const size_t fixed = 8 * (size_t)kWPC * nst + (size_t)kWPC * nst * rec_max;
    if (fixed + (size_t)kWPC * (64 + (kBRing + kXRing * kTprMax) * 32) * es > (size_t)max_smem)
        return SPTRSV_ERR_NOT_SUPPORTED;
    const int maxw_t = maxw <= 4 ? 4 : (maxw <= 8 ? 8 : kTprMax);
    const size_t rings = (size_t)kWPC * (kBRing * 32 + (size_t)kXRing * maxw_t * 32) * es;
    int Wu = 1;
    while ((size_t)kWPC * (2 * Wu + 1) * es + fixed + rings <= (size_t)max_smem) Wu *= 2;
    const int Wenv = env_int("SPTRSV_BLOCK_SLOTS", 0);
    if (Wenv > 0) {
        int w2 = 1;
        while (w2 * 2 <= Wenv) w2 *= 2;
        Wu = std::min(Wu, w2);
    }
    B.W = Wu;
    B.nst = nst;
    if ((st = h->arena.alloc(&B.d_recs, (size_t)std::max<int64_t>(rec_total, 16))) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&B.d_ovf_col, (size_t)std::max(novf, 1))) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc(&B.d_ovf_val, (size_t)std::max(novf, 1) * es)) != SPTRSV_SUCCESS) return st;
    if (h->dtype == SPTRSV_F64)
        k_rec_fill<double><<<eg, 256, 0, s>>>(n, Wu, nst, unit, unit_rows, step_of, bperm, pos, steps, B.d_rec_off,
                                             B.d_unit_step0, tri_ptr, tri_col, (const double *)tri_val,
                                             (const double *)h->d_invd_row, B.d_ovf_ptr,
                                             (unsigned char *)B.d_recs, B.d_ovf_col, (double *)B.d_ovf_val);
    else
        k_rec_fill<float><<<eg, 256, 0, s>>>(n, Wu, nst, unit, unit_rows, step_of, bperm, pos, steps, B.d_rec_off,
                                            B.d_unit_step0, tri_ptr, tri_col, (const float *)tri_val,
                                            (const float *)h->d_invd_row, B.d_ovf_ptr, (unsigned char *)B.d_recs,
                                            B.d_ovf_col, (float *)B.d_ovf_val);
    SPTRSV_CUDA(cudaGetLastError());

    // ---- launch configuration: K co-resident CTAs of kWPC warps
    const size_t smem = fixed + (size_t)kWPC * (Wu + 1) * es + rings;
    void *kn = nullptr;
    for (int tr = 1; tr >= 0; --tr) {
        if (h->dtype == SPTRSV_F64)
            kn = h->diag == SPTRSV_UNIT ? pick_kernel<double, true>(maxw, tr) : pick_kernel<double, false>(maxw, tr);
        else
            kn = h->diag == SPTRSV_UNIT ? pick_kernel<float, true>(maxw, tr) : pick_kernel<float, false>(maxw, tr);
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
    int Wu = B.W, nst = B.nst, rec_max = B.rec_max;
    const unsigned char *recs = (const unsigned char *)B.d_recs;
    void *args[] = {(void *)&Wu, (void *)&nst, (void *)&rec_max, (void *)&B.d_unit_step0, (void *)&B.d_rec_off,
                    (void *)&recs, (void *)&B.d_ovf_ptr, (void *)&B.d_ovf_col, (void *)&B.d_ovf_val, (void *)&b,
                    (void *)&x};
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
