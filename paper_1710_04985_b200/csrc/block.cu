// block.cu -- SPTRSV_ALGO_BLOCK: self-scheduling over warp-owned row tiles with
// register / shared-memory hand-offs (SURVEY.md §7 hard part H1).
//
// Why: the self-scheduled solve's time is its critical path, nlev dependent
// hand-offs (382 on cfg2).  On B200 a cross-SM hand-off costs one
// L2 round trip (~220 ns one way, profiles/microbench_r1.json) while a warp
// shuffle costs ~25 cycles.  So the rows are partitioned over warps such that
// almost every edge of the critical path stays inside one warp:
//
//   * structured grids (detected: every dependency is verified to be a 3x3x3
//     neighbour under the inferred nx, ny): a warp owns a tile of <= 32
//     z-columns (x,y), a CTA a rectangle of warp tiles; lane = column.  Warp
//     step t solves the tile's rows of its t-th level, so the dependencies of
//     a row on (x-1,y,z), (x,y-1,z), (x,y,z-1) (7-point) were solved in the
//     previous step by this warp: they arrive by __shfl_sync from registers.
//   * otherwise contiguous natural-order row blocks (correct for any matrix;
//     SPTRSV_ALGO_AUTO only picks BLOCK when a grid was detected).
//
// A warp walks its steps in level order (every dependency has a
// lower level, so the lowest unfinished step can always proceed; all CTAs are
// co-resident by cooperative launch).  Per dependency, the analysis stores a
// source code:
//   SHFL(l)   solved by this warp in the previous step by lane l: __shfl_sync
//   SMEM(i)   solved by a warp of this CTA: shared slot i, value-as-flag
//             (slots prefilled with a NaN sentinel, polled with volatile LDS)
//   GLOB(g)   solved by another CTA: global mailbox g, value-as-flag polled with
//             relaxed loads issued one step ahead.  Two mailbox arrays swap
//             roles every solve (device epoch): each CTA re-arms its own range
//             of the idle array with the sentinel while it works on the other.
//   NONE      padding
// Non-SHFL terms are accumulated first (they are ready early), SHFL terms last,
// so a step's critical chain is shuffle -> FMAs -> scale.  The order is fixed
// per row, so results are run-to-run bitwise reproducible (reading Q8).
//
// Per (warp, step) the analysis writes one fixed-size record (SoA over lanes)
//   int32 row | oslot | og | ovf | code[W]  ||  T invd | val[W]
// streamed into a per-warp shared-memory ring by TMA (cp.async.bulk +
// mbarrier, nst records in flight); b[row] is gathered PB steps ahead with
// cp.async into a per-warp ring.  Rows with more than W dependencies keep
// their entries in an overflow list (codes SMEM/GLOB only, kNone-terminated).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "internal.h"

namespace sptrsv {
namespace {

constexpr int32_t kNone = (int32_t)(3u << 30);
__host__ __device__ inline int32_t code_smem(int i) { return (int32_t)((1u << 30) | (unsigned)i); }
__host__ __device__ inline int32_t code_glob(int g) { return (int32_t)((2u << 30) | (unsigned)g); }
__host__ __device__ inline unsigned code_kind(int32_t c) { return (unsigned)c >> 30; }
__host__ __device__ inline int code_idx(int32_t c) { return c & 0x3FFFFFFF; }

// Record of one (warp, step), SoA over 32 lanes, every part a multiple of 16 B:
//   compute part: int4 {row, oslot, og, srcs}[32]          (one LDS.128)
//                 T {invd, a_0 .. a_SH-1}: (SH+1) values in 16-byte groups [g][32]
//   helper part:  int ecode[WE][32] | T eval[WE][32]
//   srcs: bits 0-2 = number of SHFL terms, then 5 bits per source lane.
//   ecode[0] = kOvf | i: all EXT terms of the row are in the overflow list at i.
__host__ __device__ constexpr int rec_cv(int) { return 512; }
__host__ __device__ constexpr int rec_ec(int SH, int es) { return 512 + 32 * es * (SH + 1); }
__host__ __device__ constexpr int rec_ev(int SH, int WE, int es) { return rec_ec(SH, es) + 128 * WE; }
__host__ __device__ constexpr int rec_bytes(int SH, int WE, int es) { return rec_ev(SH, WE, es) + 32 * es * WE; }
constexpr int kSH = 3;                       // SHFL terms per row (compute warp)
constexpr int32_t kOvfTag = (int32_t)(3u << 30) | (1 << 29);     // kind NONE + bit 29: overflow index

constexpr int kBuckets = kTprMax + 2;
__device__ __forceinline__ uint32_t bucket_of(int deps) { return deps > kTprMax ? 0u : (uint32_t)(kTprMax + 1 - deps); }

int env_int(const char *name, int dflt) {
    const char *v = getenv(name);
    return (v && *v) ? atoi(v) : dflt;
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

// (x, y) tiles of tw x th columns; CTA = wx x wy tiles; unit = cta * wpc + warp
__global__ void k_part_tiles(int n, int nx, int ny, int tw, int th, int wx, int wy, int cxn, int32_t *unit) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int x = i % nx, y = (i / nx) % ny;
    const int txi = x / tw, tyi = y / th;
    const int cta = (tyi / wy) * cxn + txi / wx;
    unit[i] = cta * (wx * wy) + (tyi % wy) * wx + (txi % wx);
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

// Dependency classes.  Walking a row's dependencies in storage order, the
// first SH that were solved by the same warp in the previous step are SHFL
// (the compute warp's registers); the others are EXT, resolved by the helper
// warp: from a shared slot (producer in the same CTA, bit 0 of need) or from
// a global mailbox (bit 1).  noslot: that CTA's slots overflowed -> GLOB.
// ecnt[pos] = number of EXT dependencies of the row at solve position pos.
__global__ void k_need(int n, int SH, int wpc, const int32_t *__restrict__ tri_ptr,
                       const int32_t *__restrict__ tri_col, const int32_t *__restrict__ unit,
                       const int32_t *__restrict__ pos, const int32_t *__restrict__ step_of,
                       const unsigned char *__restrict__ noslot, int32_t *need, int32_t *ecnt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int a = tri_ptr[i], e = tri_ptr[i + 1];
    const int ui = unit[i], si = step_of[pos[i]];
    const bool ns = noslot[ui / wpc] != 0;
    int nsh = 0, next = 0;
    for (int k = a; k < e; ++k) {
        const int j = tri_col[k];
        const int uj = unit[j], pj = pos[j];
        if (nsh < SH && uj == ui && step_of[pj] == si - 1) {
            ++nsh;
            continue;
        }
        ++next;
        if (uj / wpc == ui / wpc && !ns) atomicOr(&need[pj], 1);
        else atomicOr(&need[pj], 2);
    }
    ecnt[pos[i]] = next;
}

__global__ void k_need_bits(int n, const int32_t *need, int bit, int32_t *out) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) out[p] = (need[p] >> bit) & 1;
    if (p == n) out[p] = 0;
}

__global__ void k_ovf_count(int n, int WE, const int32_t *ecnt, int32_t *cnt) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) cnt[p] = ecnt[p] > WE ? ecnt[p] + 1 : 0;       // + terminator
    if (p == n) cnt[p] = 0;
}

// per CTA: number of shared slots it needs
__global__ void k_cta_slots(int K, const int32_t *cta_p0, const int32_t *slot_scan, int32_t *cnt) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < K) cnt[c] = slot_scan[cta_p0[c + 1]] - slot_scan[cta_p0[c]];
}

// one thread per (step, lane): the record of that lane (padding lanes included)
template <typename T>
__global__ void k_rec_fill(int nsteps, int SH, int WE, int wpc, const int2 *__restrict__ steps,
                           const int32_t *__restrict__ bperm, const int32_t *__restrict__ pos,
                           const int32_t *__restrict__ step_of, const int32_t *__restrict__ unit,
                           const int32_t *__restrict__ tri_ptr, const int32_t *__restrict__ tri_col,
                           const T *__restrict__ tri_val, const T *__restrict__ invd_row, int unit_diag,
                           const unsigned char *__restrict__ noslot, const int32_t *__restrict__ need,
                           const int32_t *__restrict__ ecnt, const int32_t *__restrict__ slot_scan,
                           const int32_t *__restrict__ g_scan, const int32_t *__restrict__ cta_p0,
                           const int32_t *__restrict__ ovf_ptr, unsigned char *__restrict__ recs,
                           int32_t *__restrict__ rows, int32_t *__restrict__ ovf_code, T *__restrict__ ovf_val) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)nsteps * 32) return;
    const int s = (int)(t >> 5), lane = (int)(t & 31);
    const int es = (int)sizeof(T), G16 = 16 / es;
    rows[t] = lane < steps[s].y ? bperm[steps[s].x + lane] : -1;            // values per 16-byte group
    unsigned char *base = recs + (size_t)s * rec_bytes(SH, WE, es);
    int4 *ci = reinterpret_cast<int4 *>(base);
    T *cv = reinterpret_cast<T *>(base + rec_cv(SH));
    int32_t *ec = reinterpret_cast<int32_t *>(base + rec_ec(SH, es));
    T *ev = reinterpret_cast<T *>(base + rec_ev(SH, WE, es));
    auto cvp = [&](int q) -> T & { return cv[((q / G16) * 32 + lane) * G16 + (q % G16)]; };
    const int2 st = steps[s];
    for (int q = 0; q <= SH; ++q) cvp(q) = T(0);
    for (int q = 0; q < WE; ++q) {
        ec[q * 32 + lane] = kNone;
        ev[q * 32 + lane] = T(0);
    }
    if (lane >= st.y) {
        ci[lane] = make_int4(-1, -1, -1, 0);
        return;
    }
    const int p = st.x + lane;
    const int i = bperm[p];
    const int ui = unit[i], cta = ui / wpc;
    const bool ns = noslot[cta] != 0;
    const int nd = need[p];
    const int si = step_of[p];
    const int a = tri_ptr[i], e = tri_ptr[i + 1];
    const bool ovf = ecnt[p] > WE;
    int srcs = 0, nsh = 0, ne = 0;
    int o = ovf ? ovf_ptr[p] : 0;
    if (ovf) ec[lane] = kOvfTag | o;
    for (int k = a; k < e; ++k) {
        const int j = tri_col[k];
        const int uj = unit[j], pj = pos[j];
        if (nsh < SH && uj == ui && step_of[pj] == si - 1) {
            srcs |= (pj - steps[si - 1].x) << (3 + 5 * nsh);
            cvp(1 + nsh) = tri_val[k];
            ++nsh;
            continue;
        }
        const int32_t c = (uj / wpc == cta && !ns) ? code_smem(slot_scan[pj] - slot_scan[cta_p0[cta]])
                                                   : code_glob(g_scan[pj]);
        if (ovf) {
            ovf_code[o] = c;
            ovf_val[o] = tri_val[k];
            ++o;
        } else {
            ec[ne * 32 + lane] = c;
            ev[ne * 32 + lane] = tri_val[k];
            ++ne;
        }
    }
    if (ovf) {
        ovf_code[o] = kNone;
        ovf_val[o] = T(0);
    }
    cvp(0) = unit_diag ? T(1) : invd_row[i];
    ci[lane] = make_int4(i, (nd & 1) ? slot_scan[p] - slot_scan[cta_p0[cta]] : -1, (nd & 2) ? g_scan[p] : -1,
                         srcs | nsh);
}

template <typename T>
__global__ void k_fill_sentinel(T *p, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (; i < n; i += stride) p[i] = Sentinel<T>::value();
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
__device__ __forceinline__ void sts_volatile(double *p, double v) {
    asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"(smem_u32(p)), "d"(v) : "memory");
}
__device__ __forceinline__ void sts_volatile(float *p, float v) {
    asm volatile("st.volatile.shared.f32 [%0], %1;" ::"r"(smem_u32(p)), "f"(v) : "memory");
}
__device__ __forceinline__ void cp_async_val(double *dst, const double *src) { cp_async_8(dst, src); }
__device__ __forceinline__ void cp_async_val(float *dst, const float *src) { cp_async_4(dst, src); }

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
        if (++it > 64) __nanosleep(32);
        v = lds_volatile(p);
        if ((it & 1023u) == 0 && wd_expired(t0)) break;
    }
    return v;
}
template <typename T>
__device__ __noinline__ T poll_global_slow(const T *p) {
    const unsigned long long t0 = wd_now();
    T v = ld_relaxed_val(p);
    unsigned it = 0;
    while (Sentinel<T>::is(v)) {
        if (++it > 16) __nanosleep(64);
        v = ld_relaxed_val(p);
        if ((it & 1023u) == 0 && wd_expired(t0)) break;
    }
    return v;
}

// Debug-only timeline hook (sptrsv_dbg_block_trace): lane 0 of every warp
// records %globaltimer at its first `cap` - 1 steps and at the end.
__device__ unsigned long long *g_trace = nullptr;
__device__ int g_trace_cap = 0;
__device__ unsigned long long *g_phase = nullptr;   // warp 0: 6 clock64 stamps x 128 steps

struct BlockArgs {
    const int32_t *unit_step0;
    const unsigned char *recs;
    const int32_t *rows;          // [nsteps][32] row of every lane (-1: padding)
    const int32_t *cta_g0;
    const int32_t *ovf_code;
    const void *ovf_val;
    void *gmb;
    unsigned *ctr;
    const void *b;
    void *x;
    int G, nslots;
};

// predicated value-as-flag loads (no branch: returns 0 where !pred)
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
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.volatile.shared.b64 %0, [%1];\n\t}"
                 : "+l"(v) : "r"(smem_u32(p)), "r"((unsigned)pred));
    return __longlong_as_double((long long)v);
}
__device__ __forceinline__ float lds_flag_if(const float *p, bool pred) {
    unsigned v = 0;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.volatile.shared.b32 %0, [%1];\n\t}"
                 : "+r"(v) : "r"(smem_u32(p)), "r"((unsigned)pred));
    return __uint_as_float(v);
}
__device__ __forceinline__ void sts_flag(double *p, double v) {
    asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"(smem_u32(p)), "d"(v));
}
__device__ __forceinline__ void sts_flag(float *p, float v) {
    asm volatile("st.volatile.shared.f32 [%0], %1;" ::"r"(smem_u32(p)), "f"(v));
}
// store ordered after every earlier memory access of the thread (compiler side)
__device__ __forceinline__ void sts_flag_last(double *p, double v) {
    asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"(smem_u32(p)), "d"(v) : "memory");
}
__device__ __forceinline__ void sts_flag_last(float *p, float v) {
    asm volatile("st.volatile.shared.f32 [%0], %1;" ::"r"(smem_u32(p)), "f"(v) : "memory");
}
__device__ __forceinline__ void stg_flag(double *p, double v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"((unsigned long long)__double_as_longlong(v)));
}
__device__ __forceinline__ void stg_flag(float *p, float v) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(__float_as_uint(v)));
}
__device__ __forceinline__ void cp_async_wait_n(int n) {      // n <= 7
    switch (n) {
        case 0: cp_async_wait<0>(); break;
        case 1: cp_async_wait<1>(); break;
        case 2: cp_async_wait<2>(); break;
        case 3: cp_async_wait<3>(); break;
        case 4: cp_async_wait<4>(); break;
        case 5: cp_async_wait<5>(); break;
        case 6: cp_async_wait<6>(); break;
        default: cp_async_wait<7>(); break;
    }
}

// the SH + 1 record values {invd, a_0 .. a_SH-1} of one lane (16-byte groups)
template <typename T> struct CV;
template <> struct CV<double> {
    double v[4];
    __device__ __forceinline__ void load(const unsigned char *p, int lane) {
        const double2 g0 = reinterpret_cast<const double2 *>(p)[lane];
        const double2 g1 = reinterpret_cast<const double2 *>(p + 512)[lane];
        v[0] = g0.x; v[1] = g0.y; v[2] = g1.x; v[3] = g1.y;
    }
};
template <> struct CV<float> {
    float v[4];
    __device__ __forceinline__ void load(const unsigned char *p, int lane) {
        const float4 g0 = reinterpret_cast<const float4 *>(p)[lane];
        v[0] = g0.x; v[1] = g0.y; v[2] = g0.z; v[3] = g0.w;
    }
};
static_assert(kSH == 3, "CV<T> holds invd + 3 SHFL coefficients");

// predicated cp.async of one value (no branch; nothing copied where !pred)
__device__ __forceinline__ void cp_async_val_if(double *dst, const double *src, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q cp.async.ca.shared.global [%0], [%1], 8;\n\t}" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"((unsigned)pred)
                 : "memory");
}
__device__ __forceinline__ void cp_async_val_if(float *dst, const float *src, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q cp.async.ca.shared.global [%0], [%1], 4;\n\t}" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"((unsigned)pred)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_wd(uint64_t *bar, uint32_t ph) {
    if (!mbar_try_wait(bar, ph)) {
        const unsigned long long t0 = wd_now();
        while (!mbar_try_wait(bar, ph))
            if (wd_expired(t0)) break;
    }
}

// Warp-specialised tile solve.  A CTA owns ntw tiles; tile w has a COMPUTE
// warp (warp w) and a HELPER warp (warp ntw + w).  The helper works in blocks
// of UB steps:
//   records   block k+DB by one TMA bulk copy (ring of NBB blocks, mbarrier per slot)
//   row ids   block k+R1B by one TMA bulk copy (ring of RRB blocks)
//   b[row]    block k+R2B by cp.async, one group per block
//   EXT terms of the block's UB steps: all their loads issued first (shared
//             slots / global mailboxes, value-as-flag), then per step
//             c = b - sum_EXT a x (storage order) -> the step's c slot
//             (value-as-flag: the NaN sentinel while empty)
// The compute warp, per step: waits for its lane's c, x = (c - sum_SHFL a
// x_prev) * invd with the SHFL sources shuffled from the previous step's
// results, stores x (and the shared slot / mailbox copies other warps need)
// and re-arms the c slot.  Its critical chain between two levels is shuffle
// -> FMA chain -> multiply.  The helper runs at most (NBB - DB) blocks ahead:
// record slot k+DB reuses the slot of block k+DB-NBB, free once the compute
// warp re-armed the c slot of that block's last step.
constexpr int kDB = 3, kNBB = 5, kR2B = 2, kBR = 4, kR1B = 4, kRRB = 4, kPFB = 12;   // kBR: 2 helpers x 2 blocks of b
__host__ __device__ constexpr int ub_of(int WE) { return WE <= 4 ? 4 : 2; }   // steps per helper block
template <typename T, bool UNIT, int WE>
__global__ void __launch_bounds__(384, 1) k_block(const BlockArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ unsigned s_epoch;
    constexpr int SH = kSH, UB = ub_of(WE), DB = kDB, NBB = kNBB, R2B = kR2B, R1B = kR1B, RRB = kRRB;
    constexpr int ES = (int)sizeof(T);
    constexpr int REC = rec_bytes(SH, WE, ES);
    constexpr int CVO = rec_cv(SH), ECO = rec_ec(SH, ES), EVO = rec_ev(SH, WE, ES);
    constexpr int NCS = NBB * UB;                 // c ring (steps)
    constexpr size_t TILE = ((size_t)NBB * UB * REC + (size_t)RRB * UB * 128 + (size_t)NCS * 32 * ES +
                             (size_t)kBR * UB * 32 * ES + 8 * (NBB + RRB) + 127) / 128 * 128;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ntw = blockDim.x / 96;              // tiles per CTA: 1 compute + 2 helper warps each
    const int w = warp % ntw;
    const bool helper = warp >= ntw;
    const int hid = helper ? (warp - ntw) / ntw : 0;   // helper 0 takes even blocks, helper 1 odd
    unsigned char *tb = smem_raw + (size_t)w * TILE;
    unsigned char *ring = tb;                                        // [NBB*UB][REC]
    int32_t *rw = reinterpret_cast<int32_t *>(tb + (size_t)NBB * UB * REC);      // [RRB*UB][32]
    T *cr = reinterpret_cast<T *>(rw + RRB * UB * 32);              // [NCS][32]
    T *br = cr + NCS * 32;                                           // [kBR*UB][32]
    uint64_t *recbar = reinterpret_cast<uint64_t *>(br + kBR * UB * 32);
    uint64_t *rowbar = recbar + NBB;
    T *slots = reinterpret_cast<T *>(smem_raw + (size_t)ntw * TILE);
    const T *b = static_cast<const T *>(a.b);
    T *x = static_cast<T *>(a.x);

    for (int i = threadIdx.x; i < a.nslots; i += blockDim.x) slots[i] = Sentinel<T>::value();
    if (helper && hid == 0) {
        for (int i = lane; i < NCS * 32; i += 32) cr[i] = Sentinel<T>::value();
        if (lane == 0) {
            for (int i = 0; i < NBB + RRB; ++i) mbar_init(&recbar[i], 1);
            fence_mbar_init();
        }
    }
    if (threadIdx.x == 0) s_epoch = (unsigned)ld_relaxed(reinterpret_cast<const int *>(a.ctr));
    __syncthreads();
    const unsigned par = s_epoch & 1u;
    T *gm = static_cast<T *>(a.gmb) + (size_t)par * a.G;
    {   // re-arm this CTA's mailboxes of the idle array (written by the previous solve)
        T *go = static_cast<T *>(a.gmb) + (size_t)(par ^ 1u) * a.G;
        for (int i = a.cta_g0[blockIdx.x] + threadIdx.x; i < a.cta_g0[blockIdx.x + 1]; i += blockDim.x)
            go[i] = Sentinel<T>::value();
    }

    const int u = blockIdx.x * ntw + w;
    const int s0 = a.unit_step0[u], n = a.unit_step0[u + 1] - s0;
    if (n > 0 && helper) {
        const int nblk = (n + UB - 1) / UB;
        const unsigned char *grec = a.recs + (size_t)s0 * REC;
        const int32_t *grow = a.rows + (size_t)s0 * 32;
        const bool trace = g_trace != nullptr && hid == 0;
        T *bh = br + hid * 2 * UB * 32;          // this helper's b ring: its blocks k (slot) and k+2
        auto issue_rec = [&](int kk) {          // lane 0: TMA of record block kk
            const int slot = kk % NBB;
            mbar_arrive_expect_tx(&recbar[slot], UB * REC);
            bulk_g2s(ring + (size_t)slot * UB * REC, grec + (size_t)kk * UB * REC, UB * REC, &recbar[slot]);
        };
        auto issue_rows = [&](int kk) {
            const int slot = kk % RRB;
            mbar_arrive_expect_tx(&rowbar[slot], UB * 128);
            bulk_g2s(rw + slot * UB * 32, grow + (size_t)kk * UB * 32, UB * 128, &rowbar[slot]);
        };
        auto prefetch_l2 = [&](int kk) {
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(grec + (size_t)kk * UB * REC), "r"(UB * REC)
                         : "memory");
        };
        auto rec_wait = [&](int kk) { mbar_wait_wd(&recbar[kk % NBB], (uint32_t)((kk / NBB) & 1)); };
        auto issue_b = [&](int kk, int bslot) {  // b of block kk (row ids landed)
            mbar_wait_wd(&rowbar[kk % RRB], (uint32_t)((kk / RRB) & 1));
            const int32_t *rr = rw + (kk % RRB) * UB * 32 + lane;
            T *bb = bh + bslot * UB * 32 + lane;
#pragma unroll
            for (int j = 0; j < UB; ++j) {
                const int r = rr[j * 32];
                cp_async_val_if(bb + j * 32, b + r, r >= 0);
            }
        };
        int32_t ncode[UB][WE];
        T nv[UB][WE];
        auto ext_loads = [&](int kk) {           // EXT values of block kk (records landed)
            const unsigned char *rb = ring + (size_t)(kk % NBB) * UB * REC;
#pragma unroll
            for (int j = 0; j < UB; ++j) {
                const int32_t *ec = reinterpret_cast<const int32_t *>(rb + j * REC + ECO) + lane;
                const bool vj = kk * UB + j < n;          // the last block may hold the next warp's steps
#pragma unroll
                for (int q = 0; q < WE; ++q) {
                    ncode[j][q] = ec[q * 32];
                    const unsigned kind = code_kind(ncode[j][q]);
                    const T vs_ = lds_flag_if(slots + code_idx(ncode[j][q]), vj && kind == 1u);
                    const T vg_ = ldg_flag_if(gm + code_idx(ncode[j][q]), vj && kind == 2u);
                    nv[j][q] = kind == 1u ? vs_ : vg_;
                }
            }
        };
        if (hid == 0 && lane == 0) {
            for (int kk = 0; kk < min(nblk, kPFB); ++kk) prefetch_l2(kk);
            for (int kk = 0; kk < min(nblk, DB); ++kk) issue_rec(kk);
            for (int kk = 0; kk < min(nblk, R1B); ++kk) issue_rows(kk);
        }
        if (hid < nblk) {
            issue_b(hid, 0);
            cp_async_commit();
            rec_wait(hid);
            __syncwarp();
            ext_loads(hid);
        }
#pragma unroll 1
        for (int k = hid, i = 0; k < nblk; k += 2, ++i) {
            if (trace && lane == 0 && k * UB < g_trace_cap - 1) g_trace[(size_t)u * g_trace_cap + k * UB] = wd_now();
            // (1) refill: records k+DB (the slot of block k+DB-NBB, released by the
            // compute warp), rows k+R1B, L2 prefetch
            if (k + DB < nblk) {
                if (k + DB >= NBB) {
                    const T *f = cr + (((k + DB - NBB) * UB + UB - 1) % NCS) * 32 + lane;
                    if (__any_sync(0xffffffffu, !Sentinel<T>::is(lds_volatile(f)))) {
                        const unsigned long long t0 = wd_now();
                        unsigned it = 0;
                        while (__any_sync(0xffffffffu, !Sentinel<T>::is(lds_volatile(f)))) {
                            __nanosleep(20);
                            if ((++it & 1023u) == 0 && wd_expired(t0)) break;
                        }
                    }
                }
                if (lane == 0) issue_rec(k + DB);
            }
            if (lane == 0) {
                if (k + R1B < nblk) issue_rows(k + R1B);
                if (k + kPFB < nblk) prefetch_l2(k + kPFB);
            }
            // (2) b of this helper's next block k+2
            if (k + 2 < nblk) issue_b(k + 2, (i + 1) & 1);
            cp_async_commit();
            // (3) block k: b (this helper's previous group) and records
            cp_async_wait<1>();
            rec_wait(k);
            __syncwarp();
            const unsigned char *rb = ring + (size_t)(k % NBB) * UB * REC;
            int32_t code[UB][WE];
            T v[UB][WE];
#pragma unroll
            for (int j = 0; j < UB; ++j)
#pragma unroll
                for (int q = 0; q < WE; ++q) {
                    code[j][q] = ncode[j][q];
                    v[j][q] = nv[j][q];
                }
            // (4) EXT loads of this helper's next block k+2 (two blocks of slack)
            if (k + 2 < nblk) {
                rec_wait(k + 2);
                __syncwarp();
                ext_loads(k + 2);
            }
            const int cs = (k * UB) % NCS;
            const int bs = i & 1;
            // (5) block k's c values.  Fast path (every EXT value arrived, no
            // overflow row): straight-line over the UB steps.  Otherwise one step
            // at a time, publishing each c as soon as its values are there (a
            // later step of the block may depend on this warp's own results),
            // re-issuing all pending loads of the block together per round trip.
            bool pend = false, ovf = false;
#pragma unroll
            for (int j = 0; j < UB; ++j) {
#pragma unroll
                for (int q = 0; q < WE; ++q) pend |= Sentinel<T>::is(v[j][q]);
                ovf |= ((unsigned)code[j][0] & 0xE0000000u) == 0xE0000000u && k * UB + j < n;
            }
            const T *evb = reinterpret_cast<const T *>(rb + EVO) + lane;
            if (!__any_sync(0xffffffffu, pend || ovf)) {
#pragma unroll
                for (int j = 0; j < UB; ++j) {
                    T c = bh[(bs * UB + j) * 32 + lane];
#pragma unroll
                    for (int q = 0; q < WE; ++q) c = fnma(evb[j * (REC / ES) + q * 32], v[j][q], c);
                    sts_flag(cr + (cs + j) * 32 + lane, Sentinel<T>::scrub(c));
                }
            } else {
#pragma unroll
                for (int j = 0; j < UB; ++j) {
                    if (k * UB + j >= n) break;
                    bool pj = false;
#pragma unroll
                    for (int q = 0; q < WE; ++q) pj |= Sentinel<T>::is(v[j][q]);
                    if (__any_sync(0xffffffffu, pj)) {
                        const unsigned long long t0 = wd_now();
                        unsigned it = 0;
                        do {
#pragma unroll
                            for (int jj = j; jj < UB; ++jj)
#pragma unroll
                                for (int q = 0; q < WE; ++q) {
                                    const bool p = Sentinel<T>::is(v[jj][q]);
                                    const unsigned kind = code_kind(code[jj][q]);
                                    const T vs_ = lds_flag_if(slots + code_idx(code[jj][q]), p && kind == 1u);
                                    const T vg_ = ldg_flag_if(gm + code_idx(code[jj][q]), p && kind == 2u);
                                    v[jj][q] = p ? (kind == 1u ? vs_ : vg_) : v[jj][q];
                                }
                            pj = false;
#pragma unroll
                            for (int q = 0; q < WE; ++q) pj |= Sentinel<T>::is(v[j][q]);
                            if ((++it & 255u) == 0 && wd_expired(t0)) break;
                        } while (__any_sync(0xffffffffu, pj));
                    }
                    T c = bh[(bs * UB + j) * 32 + lane];
#pragma unroll
                    for (int q = 0; q < WE; ++q) c = fnma(evb[j * (REC / ES) + q * 32], v[j][q], c);
                    if (((unsigned)code[j][0] & 0xE0000000u) == 0xE0000000u) {          // overflow list
                        const T *ov = static_cast<const T *>(a.ovf_val);
                        for (int o = code[j][0] & 0x1FFFFFFF;; ++o) {
                            const int32_t cc = a.ovf_code[o];
                            if (cc == kNone) break;
                            T vv;
                            if (code_kind(cc) == 1u) {
                                vv = lds_volatile(slots + code_idx(cc));
                                if (Sentinel<T>::is(vv)) vv = poll_smem_slow(slots + code_idx(cc));
                            } else {
                                vv = ld_relaxed_val(gm + code_idx(cc));
                                if (Sentinel<T>::is(vv)) vv = poll_global_slow(gm + code_idx(cc));
                            }
                            c = fnma(ov[o], vv, c);
                        }
                    }
                    sts_flag(cr + (cs + j) * 32 + lane, Sentinel<T>::scrub(c));
                }
            }
        }
        cp_async_wait<0>();
        if (trace && lane == 0) g_trace[(size_t)u * g_trace_cap + g_trace_cap - 1] = wd_now();
    } else if (n > 0) {
        // software-pipelined: the next step's c and record fields are loaded
        // before this step's shuffle -> FMA chain; the readiness check of the
        // next c comes after it (warp-uniform; fields reloaded if it was late)
        T xprev = T(0);
        auto wait_c = [&](T *cp) -> T {
            T c = lds_volatile(cp);
            if (__any_sync(0xffffffffu, Sentinel<T>::is(c))) {
                const unsigned long long t0 = wd_now();
                unsigned it = 0;
                do {
                    if (++it > 4) __nanosleep(20);          // leave the issue slots to the helper
                    c = lds_volatile(cp);
                    if ((it & 4095u) == 0 && wd_expired(t0)) break;
                } while (__any_sync(0xffffffffu, Sentinel<T>::is(c)));
            }
            return c;
        };
        T *cp = cr + lane;
        T c = wait_c(cp);
        asm volatile("" ::: "memory");
        const unsigned char *r = ring;
        int4 ci = reinterpret_cast<const int4 *>(r)[lane];
        CV<T> cv;
        cv.load(r + CVO, lane);
        int slot = 0;
#pragma unroll 1
        for (int t = 0; t < n; ++t) {
            const int slot1 = slot + 1 == NCS ? 0 : slot + 1;
            T *cp1 = cr + slot1 * 32 + lane;
            const unsigned char *r1 = ring + (size_t)slot1 * REC;
            T c1 = T(0);
            int4 ci1 = make_int4(-1, -1, -1, 0);
            CV<T> cv1;
            const bool more = t + 1 < n;
            if (more) {
                c1 = lds_volatile(cp1);
                asm volatile("" ::: "memory");
                ci1 = reinterpret_cast<const int4 *>(r1)[lane];
                cv1.load(r1 + CVO, lane);
            }
            const int nsh = ci.w & 7;
            T acc = c;
#pragma unroll
            for (int q = 0; q < SH; ++q) {
                const T vq = __shfl_sync(0xffffffffu, xprev, (ci.w >> (3 + 5 * q)) & 31);
                acc = fnma(cv.v[1 + q], q < nsh ? vq : T(0), acc);
            }
            const T xi = UNIT ? Sentinel<T>::scrub(acc) : acc * cv.v[0];   // (a product is never the sentinel)
            if (ci.x >= 0) __stcg(x + ci.x, xi);
            if (ci.y >= 0) sts_flag(slots + ci.y, xi);
            if (ci.z >= 0) stg_flag(gm + ci.z, xi);
            sts_flag_last(cr + slot * 32 + lane, Sentinel<T>::value());     // step consumed: re-arm the c slot
            xprev = xi;
            if (more && __any_sync(0xffffffffu, Sentinel<T>::is(c1))) {     // the next c was not ready yet
                c1 = wait_c(cp1);
                asm volatile("" ::: "memory");
                ci1 = reinterpret_cast<const int4 *>(r1)[lane];
                cv1.load(r1 + CVO, lane);
            }
            c = c1;
            ci = ci1;
            cv = cv1;
            slot = slot1;
        }
    }

    __syncthreads();
    if (threadIdx.x == 0) {      // the last CTA to finish advances the mailbox epoch
        __threadfence();
        if (atomicAdd(&a.ctr[1], 1u) == gridDim.x - 1) {
            atomicExch(&a.ctr[1], 0u);
            __threadfence();
            atomicAdd(&a.ctr[0], 1u);
        }
    }
}

// ---------------------------------------------------------------- lean BLOCK
// k_block1: the same records, ONE warp per tile doing everything (no helper
// warp, no c hand-off between warps).  Per step t the warp
//   (1) loads step t+1's record fields and its SMEM EXT values (shared slots
//       written by other warps of the CTA, value-as-flag),
//   (2) solves step t: readiness vote, c = b - sum_EXT a x (storage order),
//       the SHFL chain, x * invd, stores,
//   (3) issues step t+2's b[row] and GLOB EXT loads (relaxed) into registers:
//       two steps of cover for an L2 round trip, so a consumer tile needs to
//       lag its producer by only ~2 levels (a whole-block prefetch forced
//       4-7 levels per CTA crossing, tools/wave_trace.py).
// Per block of kLUB steps: record block k+kLDB by TMA (lane 0), L2 prefetch
// of records kLPF blocks ahead and of b[row] of block k+2 (records landed).
// A value still holding the sentinel is re-polled with two loads in flight
// (half the round trip of overshoot instead of a whole one).  Arithmetic
// order equals k_block's (bitwise-equal x).
constexpr int kLUB = 4, kLDB = 3, kLNBB = kLDB + 2, kLPF = 12, kLPB = 4;
__host__ __device__ constexpr size_t lean_tile_bytes_c(int REC, int) {
    return ((size_t)kLNBB * kLUB * REC + 8 * kLNBB + 127) / 128 * 128;
}

template <typename T, int WE>
struct LState {
    int4 ci;
    CV<T> cv;
    int32_t code[WE];
    T ev[WE];
    T v[WE];              // SMEM EXT values (0 for other kinds)
};

// overflow list of one row (rows with more EXT terms than WE): slow path
template <typename T>
__device__ __noinline__ T lean_ovf(T c, int o, const int32_t *__restrict__ ovf_code, const T *__restrict__ ovf_val,
                                   const T *slots, const T *gm) {
    for (;; ++o) {
        const int32_t cc = ovf_code[o];
        if (cc == kNone) break;
        T vv;
        if (code_kind(cc) == 1u) {
            vv = lds_volatile(slots + code_idx(cc));
            if (Sentinel<T>::is(vv)) vv = poll_smem_slow(slots + code_idx(cc));
        } else {
            vv = ld_relaxed_val(gm + code_idx(cc));
            if (Sentinel<T>::is(vv)) vv = poll_global_slow(gm + code_idx(cc));
        }
        c = fnma(ovf_val[o], vv, c);
    }
    return c;
}

__device__ __forceinline__ double ldg_nc_if(const double *p, bool pred) {
    double v = 0.0;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.nc.L1::no_allocate.f64 %0, [%1];\n\t}"
                 : "+d"(v) : "l"(p), "r"((unsigned)pred));
    return v;
}
__device__ __forceinline__ float ldg_nc_if(const float *p, bool pred) {
    float v = 0.f;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.nc.L1::no_allocate.f32 %0, [%1];\n\t}"
                 : "+f"(v) : "l"(p), "r"((unsigned)pred));
    return v;
}
__device__ __forceinline__ void prefetch_l2_if(const void *p, bool pred) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\t@q prefetch.global.L2 [%0];\n\t}" ::"l"(p),
                 "r"((unsigned)pred));
}

template <typename T, bool UNIT, int WE>
__global__ void __launch_bounds__(128, 1) k_block1(const BlockArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ unsigned s_epoch;
    constexpr int SH = kSH, UB = kLUB, DB = kLDB, NBB = kLNBB;
    constexpr int ES = (int)sizeof(T);
    constexpr int REC = rec_bytes(SH, WE, ES);
    constexpr int CVO = rec_cv(SH), ECO = rec_ec(SH, ES), EVO = rec_ev(SH, WE, ES);
    constexpr size_t TILE = lean_tile_bytes_c(REC, ES);
    static_assert(UB % 2 == 0 && UB >= 2, "ping-pong state needs an even block length");
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int ntw = blockDim.x >> 5;
    unsigned char *tb = smem_raw + (size_t)w * TILE;
    unsigned char *ring = tb;                                                       // [NBB][UB][REC]
    uint64_t *recbar = reinterpret_cast<uint64_t *>(tb + (size_t)NBB * UB * REC);
    T *slots = reinterpret_cast<T *>(smem_raw + (size_t)ntw * TILE);
    const T *b = static_cast<const T *>(a.b);
    T *x = static_cast<T *>(a.x);

    for (int i = threadIdx.x; i < a.nslots; i += blockDim.x) slots[i] = Sentinel<T>::value();
    if (lane == 0) {
        for (int i = 0; i < NBB; ++i) mbar_init(&recbar[i], 1);
        fence_mbar_init();
    }
    if (threadIdx.x == 0) s_epoch = (unsigned)ld_relaxed(reinterpret_cast<const int *>(a.ctr));
    __syncthreads();
    const unsigned par = s_epoch & 1u;
    T *gm = static_cast<T *>(a.gmb) + (size_t)par * a.G;
    {   // re-arm this CTA's mailboxes of the idle array (written by the previous solve)
        T *go = static_cast<T *>(a.gmb) + (size_t)(par ^ 1u) * a.G;
        for (int i = a.cta_g0[blockIdx.x] + threadIdx.x; i < a.cta_g0[blockIdx.x + 1]; i += blockDim.x)
            go[i] = Sentinel<T>::value();
    }

    const int u = blockIdx.x * ntw + w;
    const int s0 = a.unit_step0[u], n = a.unit_step0[u + 1] - s0;
    if (n > 0) {
        const int nblk = (n + UB - 1) / UB;
        const unsigned char *grec = a.recs + (size_t)s0 * REC;
        unsigned long long *trc = g_trace != nullptr ? g_trace + (size_t)u * g_trace_cap : nullptr;
        long long dbg[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // debug trace only (g_trace set): cycle counters
        auto issue_rec = [&](int kk) {
            const int slot = kk % NBB;
            mbar_arrive_expect_tx(&recbar[slot], UB * REC);
            bulk_g2s(ring + (size_t)slot * UB * REC, grec + (size_t)kk * UB * REC, UB * REC, &recbar[slot]);
        };
        auto prefetch_rec = [&](int kk) {
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(grec + (size_t)kk * UB * REC), "r"(UB * REC)
                         : "memory");
        };
        auto rec_wait = [&](int kk) { mbar_wait_wd(&recbar[kk % NBB], (uint32_t)((kk / NBB) & 1)); };
        // b[row] is L2-prefetched kLPB-1 blocks ahead from row ids loaded one block earlier
        const int32_t *grow = a.rows + (size_t)s0 * 32 + lane;
        int32_t rowreg[UB];
        auto load_rows = [&](int kk) {
#pragma unroll
            for (int j = 0; j < UB; ++j) rowreg[j] = kk < nblk ? __ldg(grow + ((size_t)kk * UB + j) * 32) : -1;
        };
        auto prefetch_b = [&]() {
#pragma unroll
            for (int j = 0; j < UB; ++j) prefetch_l2_if(b + rowreg[j], rowreg[j] >= 0);
        };
        // start of block kb: refill the record ring, b prefetch
        auto block_work = [&](int kb) {
            const long long c0 = trc != nullptr ? clock64() : 0;
            __syncwarp();
            if (lane == 0) {
                if (kb + DB < nblk) issue_rec(kb + DB);
                if (kb + kLPF < nblk) prefetch_rec(kb + kLPF);
            }
            prefetch_b();                        // b of block kb + kLPB - 1
            load_rows(kb + kLPB);
            if (kb + 1 < nblk) rec_wait(kb + 1);
            if (trc != nullptr) dbg[4] += clock64() - c0;
        };
        auto load_state = [&](LState<T, WE> &S, const unsigned char *r) {
            S.ci = reinterpret_cast<const int4 *>(r)[lane];
            S.cv.load(r + CVO, lane);
#pragma unroll
            for (int q = 0; q < WE; ++q) {
                S.code[q] = reinterpret_cast<const int32_t *>(r + ECO)[q * 32 + lane];
                S.ev[q] = reinterpret_cast<const T *>(r + EVO)[q * 32 + lane];
                S.v[q] = lds_flag_if(slots + code_idx(S.code[q]), code_kind(S.code[q]) == 1u);
            }
        };
        // b and GLOB EXT values of a step, loads in flight until first use
        T Bv[2], Gv[2][WE];
        auto issue_far = [&](int par2, const unsigned char *r, bool valid) {
            const int row = reinterpret_cast<const int4 *>(r)[lane].x;
            Bv[par2] = ldg_nc_if(b + row, valid && row >= 0);
#pragma unroll
            for (int q = 0; q < WE; ++q) {
                const int32_t cd = reinterpret_cast<const int32_t *>(r + ECO)[q * 32 + lane];
                Gv[par2][q] = ldg_flag_if(gm + code_idx(cd), valid && code_kind(cd) == 2u);
            }
        };

        if (lane == 0) {
            for (int kk = 0; kk < min(nblk, kLPF); ++kk) prefetch_rec(kk);
            for (int kk = 0; kk < min(nblk, DB); ++kk) issue_rec(kk);
        }
        for (int kk = 0; kk < kLPB - 1; ++kk) {
            load_rows(kk);
            prefetch_b();
        }
        load_rows(kLPB - 1);
        rec_wait(0);
        issue_far(0, ring, true);
        issue_far(1, ring + REC, n > 1);
        block_work(0);

        LState<T, WE> st[2];
        load_state(st[0], ring);
        T xprev = T(0);
        int rslot = 0;
        // one block of UB steps; false when the warp's steps are done
        auto do_block = [&](int k) -> bool {
            if (trc != nullptr && lane == 0 && k * UB < g_trace_cap - 16) trc[k * UB] = wd_now();
            const unsigned char *rbk = ring + (size_t)rslot * UB * REC;
            const int rslot1 = rslot + 1 == NBB ? 0 : rslot + 1;
            const unsigned char *rbk1 = ring + (size_t)rslot1 * UB * REC;
#pragma unroll
            for (int j = 0; j < UB; ++j) {
                const int t = k * UB + j;
                if (t >= n) return false;
                LState<T, WE> &S = st[j & 1];
                LState<T, WE> &N = st[(j + 1) & 1];
                const bool more = t + 1 < n;
                if (more) {
                    if (j == UB - 1) {
                        block_work(k + 1);
                        load_state(N, rbk1);
                    } else {
                        load_state(N, rbk + (size_t)(j + 1) * REC);
                    }
                }
                // EXT readiness (value-as-flag); slow path re-polls with two loads in flight
                T v[WE];
                bool pend = false;
#pragma unroll
                for (int q = 0; q < WE; ++q) {
                    const unsigned kind = code_kind(S.code[q]);
                    v[q] = kind == 2u ? Gv[j & 1][q] : S.v[q];
                    pend |= (kind == 1u || kind == 2u) && Sentinel<T>::is(v[q]);
                }
                if (__any_sync(0xffffffffu, pend)) {
                    const unsigned long long t0 = wd_now();
                    const long long c0 = trc != nullptr ? clock64() : 0;
                    unsigned it = 0;
                    T inf[WE];
                    auto issue_polls = [&](T (&dst)[WE]) {
#pragma unroll
                        for (int q = 0; q < WE; ++q) {
                            const unsigned kind = code_kind(S.code[q]);
                            const bool p = (kind == 1u || kind == 2u) && Sentinel<T>::is(v[q]);
                            const T vs_ = lds_flag_if(slots + code_idx(S.code[q]), p && kind == 1u);
                            const T vg_ = ldg_flag_if(gm + code_idx(S.code[q]), p && kind == 2u);
                            dst[q] = kind == 1u ? vs_ : vg_;
                        }
                    };
                    issue_polls(inf);
                    do {
                        T nx[WE];
                        __nanosleep(32);
                        issue_polls(nx);
                        pend = false;
#pragma unroll
                        for (int q = 0; q < WE; ++q) {
                            const unsigned kind = code_kind(S.code[q]);
                            const bool p = (kind == 1u || kind == 2u) && Sentinel<T>::is(v[q]);
                            v[q] = (p && !Sentinel<T>::is(inf[q])) ? inf[q] : v[q];
                            pend |= (kind == 1u || kind == 2u) && Sentinel<T>::is(v[q]);
                            inf[q] = nx[q];
                        }
                        if ((++it & 255u) == 0 && wd_expired(t0)) break;
                    } while (__any_sync(0xffffffffu, pend));
                    if (trc != nullptr) {
                        bool gl = false;
#pragma unroll
                        for (int q = 0; q < WE; ++q) gl |= code_kind(S.code[q]) == 2u;
                        gl = __any_sync(0xffffffffu, gl);
                        if (t == 0) dbg[0] += clock64() - c0;
                        else if (gl) { dbg[1] += clock64() - c0; ++dbg[2]; }
                        else { dbg[3] += clock64() - c0; ++dbg[7]; }
                    }
                }
                T c = Bv[j & 1];
#pragma unroll
                for (int q = 0; q < WE; ++q) c = fnma(S.ev[q], v[q], c);
                if (((unsigned)S.code[0] & 0xE0000000u) == 0xE0000000u && S.ci.x >= 0)
                    c = lean_ovf<T>(c, S.code[0] & 0x1FFFFFFF, a.ovf_code, static_cast<const T *>(a.ovf_val), slots,
                                    gm);
                const int nsh = S.ci.w & 7;
                T acc = Sentinel<T>::scrub(c);
#pragma unroll
                for (int q = 0; q < SH; ++q) {
                    const T vq = __shfl_sync(0xffffffffu, xprev, (S.ci.w >> (3 + 5 * q)) & 31);
                    acc = fnma(S.cv.v[1 + q], q < nsh ? vq : T(0), acc);
                }
                const T xi = UNIT ? Sentinel<T>::scrub(acc) : acc * S.cv.v[0];
                if (S.ci.x >= 0) __stcg(x + S.ci.x, xi);
                if (S.ci.y >= 0) sts_flag(slots + S.ci.y, xi);
                if (S.ci.z >= 0) stg_flag(gm + S.ci.z, xi);
                xprev = xi;
                // (3) step t+2's b and GLOB loads (its records have landed)
                if (j + 2 < UB) issue_far(j & 1, rbk + (size_t)(j + 2) * REC, t + 2 < n);
                else issue_far(j & 1, rbk1 + (size_t)(j + 2 - UB) * REC, t + 2 < n);
            }
            rslot = rslot1;
            return true;
        };
#pragma unroll 1
        for (int k = 0; k < nblk; ++k)
            if (!do_block(k)) break;
        if (trc != nullptr && lane == 0) {
            trc[g_trace_cap - 1] = wd_now();
            for (int i = 0; i < 8; ++i) trc[g_trace_cap - 16 + i] = (unsigned long long)dbg[i];
        }
    }

    __syncthreads();
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
void *pick_kernel_lean(int W, int &we) {
    if (W <= 3) { we = 2; return (void *)k_block1<T, UNIT, 2>; }
    we = 4;
    return (void *)k_block1<T, UNIT, 4>;
}

// per-tile shared memory of k_block (must match TILE there)
size_t block_tile_bytes(int REC, int es, int ub) {
    return ((size_t)kNBB * ub * REC + (size_t)kRRB * ub * 128 + (size_t)kNBB * ub * 32 * es +
            (size_t)kBR * ub * 32 * es + 8 * (kNBB + kRRB) + 127) / 128 * 128;
}

// EXT entries per record row: enough for the detected-grid plans (7-point:
// <= 2 EXT terms; 27-point: <= 13); more -> the overflow list
template <typename T, bool UNIT>
void *pick_kernel(int W, int &we) {
    if (W <= 3) { we = 2; return (void *)k_block<T, UNIT, 2>; }
    if (W <= 4) { we = 4; return (void *)k_block<T, UNIT, 4>; }
    if (W <= 8) { we = 8; return (void *)k_block<T, UNIT, 8>; }
    we = 13;
    return (void *)k_block<T, UNIT, 13>;
}
bool g_host_trace = false;

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
    for (int64_t a : offs)
        for (int da = -1; da <= 1; ++da) {
            const int64_t nx = a + da;
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

int i32_at(const int32_t *d, int64_t i, cudaStream_t s, sptrsv_status_t &st) {
    int32_t v = 0;
    cudaError_t e = cudaMemcpyAsync(&v, d + i, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) st = cuda_fail(e, "i32_at");
    return v;
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
    sptrsv_status_t st = SPTRSV_SUCCESS;
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

    // kernel instance (EXT entries per record row) and shared-memory budget
    int WE = 0;
    const int W = std::max(1, h->info.max_row_deps);
    void *kn = nullptr;
    if (h->dtype == SPTRSV_F64)
        kn = h->diag == SPTRSV_UNIT ? pick_kernel<double, true>(W, WE) : pick_kernel<double, false>(W, WE);
    else
        kn = h->diag == SPTRSV_UNIT ? pick_kernel<float, true>(W, WE) : pick_kernel<float, false>(W, WE);
    // lean kernel (one warp per tile, k_block1) when SPTRSV_BLOCK_LEAN=1 (opt-in:
    // cfg2 0.327 ms vs 0.271 ms for the helper design, profiles/lean_block_r1f.md);
    // rows with more than 4 EXT terms use the overflow lists
    const bool lean = env_int("SPTRSV_BLOCK_LEAN", 0) != 0;
    if (lean) {
        if (h->dtype == SPTRSV_F64)
            kn = h->diag == SPTRSV_UNIT ? pick_kernel_lean<double, true>(W, WE) : pick_kernel_lean<double, false>(W, WE);
        else
            kn = h->diag == SPTRSV_UNIT ? pick_kernel_lean<float, true>(W, WE) : pick_kernel_lean<float, false>(W, WE);
    }
    const int REC = rec_bytes(kSH, WE, (int)es);
    const size_t budget = (size_t)max_smem - 1024;          // static smem + slack
    // per CTA (nt tiles): the tiles' rings; the rest holds shared slots
    auto ring_bytes = [&](int nt) {
        return (size_t)nt * (lean ? lean_tile_bytes_c(REC, (int)es) : block_tile_bytes(REC, (int)es, ub_of(WE)));
    };

    // ---- 2. partition rows over U = K x wpc warps of K co-resident CTAs
    int32_t *unit = nullptr;
    if ((st = h->arena.alloc_n(&unit, n)) != SPTRSV_SUCCESS) return st;
    B.d_unit = unit;
    int gnx = 0, gny = 0;
    if (n >= 64 && !env_int("SPTRSV_BLOCK_NO_GRID", 0)) {
        if ((st = detect_grid(h, tri_ptr, tri_col, tmp, s, gnx, gny)) != SPTRSV_SUCCESS) return st;
    }
    int K = 1, wpc = 4;
    B.grid_nx = B.grid_ny = B.tile_w = B.tile_h = 0;
    if (gnx > 0) {
        // warp tile tw x th columns (<= 32: one step per level), CTA = wx x wy
        // tiles; the fewest warps per CTA that fit all CTAs on the SMs
        int tw = std::min(env_int("SPTRSV_BLOCK_TW", gny == 1 ? 32 : 8), gnx);
        int th = std::max(1, std::min(32 / std::max(tw, 1), gny));
        const int ewx = env_int("SPTRSV_BLOCK_WX", 0), ewy = env_int("SPTRSV_BLOCK_WY", 0);
        static const int shapes[][2] = {{1, 1}, {2, 1}, {1, 2}, {2, 2}};
        int wx = 0, wy = 0;
        for (int grow = 0; grow < 8 && wx == 0; ++grow) {
            const int ntx = (gnx + tw - 1) / tw, nty = (gny + th - 1) / th;
            if (ewx > 0 && ewy > 0) {
                wx = ewx;
                wy = ewy;
                break;
            }
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
            k_part_tiles<<<eg, 256, 0, s>>>(n, gnx, gny, tw, th, wx, wy, cxn, unit);
            B.grid_nx = gnx;
            B.grid_ny = gny;
            B.tile_w = tw;
            B.tile_h = th;
        } else {
            gnx = 0;
        }
    }
    if (gnx == 0) {
        int Kn = env_int("SPTRSV_BLOCK_K", 0);
        if (Kn <= 0) Kn = (int)std::max<int64_t>(1, std::min<int64_t>(h->num_sms, n / 8192));
        K = std::min(Kn, h->num_sms);
        wpc = 4;
        while (wpc > 1 && ring_bytes(wpc) + 2048 * es > budget) wpc /= 2;
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
    if ((st = h->arena.alloc_n(&B.d_unit_step0, (size_t)U + 1)) != SPTRSV_SUCCESS) return st;
    k_steps<<<gg, 256, 0, s>>>(gp0, sub0, ngroups, bperm, unit, steps, step_unit);
    k_unit_step0<<<(nsteps + 255) / 256, 256, 0, s>>>(step_unit, nsteps, U, B.d_unit_step0);
    k_pos_step<<<eg, 256, 0, s>>>(head, gid, gp0, sub0, n, step_of);
    k_cta_p0<<<(K + 1 + 255) / 256, 256, 0, s>>>(K, wpc, nsteps, n, B.d_unit_step0, steps, cta_p0);
    SPTRSV_CUDA(cudaGetLastError());

    // ---- 4. shared-memory budget, dependency classes
    auto fixed_bytes = [&]() { return ring_bytes(wpc); };
    if (fixed_bytes() > budget) return SPTRSV_ERR_NOT_SUPPORTED;
    const int cap = (int)((budget - fixed_bytes()) / es);

    unsigned char *noslot = nullptr;
    int32_t *need = nullptr, *bits = nullptr, *slot_scan = nullptr, *g_scan = nullptr, *ccnt = nullptr;
    int32_t *ecnt = nullptr;
    if ((st = tmp.alloc_n(&ecnt, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&noslot, (size_t)K)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&need, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&bits, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&slot_scan, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&g_scan, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&ccnt, (size_t)K)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemsetAsync(noslot, 0, (size_t)K, s));
    std::vector<int32_t> hcnt(K);
    std::vector<unsigned char> hns(K, 0);
    int max_slots = 0;
    for (int pass = 0; pass < 2; ++pass) {
        SPTRSV_CUDA(cudaMemsetAsync(need, 0, sizeof(int32_t) * ((size_t)n + 1), s));
        k_need<<<eg, 256, 0, s>>>(n, kSH, wpc, tri_ptr, tri_col, unit, pos, step_of, noslot, need, ecnt);
        k_need_bits<<<(n + 1 + 255) / 256, 256, 0, s>>>(n, need, 0, bits);
        if ((st = exclusive_scan_i32(bits, slot_scan, (int64_t)n + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
        k_cta_slots<<<(K + 255) / 256, 256, 0, s>>>(K, cta_p0, slot_scan, ccnt);
        SPTRSV_CUDA(cudaGetLastError());
        SPTRSV_CUDA(cudaMemcpyAsync(hcnt.data(), ccnt, sizeof(int32_t) * K, cudaMemcpyDeviceToHost, s));
        SPTRSV_CUDA(cudaStreamSynchronize(s));
        bool over = false;
        max_slots = 0;
        for (int c = 0; c < K; ++c) {
            if (hcnt[c] > cap) {
                hns[c] = 1;
                over = true;
            } else {
                max_slots = std::max(max_slots, hcnt[c]);
            }
        }
        if (!over) break;
        if (pass == 1) return SPTRSV_ERR_NOT_SUPPORTED;
        SPTRSV_CUDA(cudaMemcpyAsync(noslot, hns.data(), (size_t)K, cudaMemcpyHostToDevice, s));
    }
    k_need_bits<<<(n + 1 + 255) / 256, 256, 0, s>>>(n, need, 1, bits);
    if ((st = exclusive_scan_i32(bits, g_scan, (int64_t)n + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    const int32_t G = i32_at(g_scan, n, s, st);
    if (st != SPTRSV_SUCCESS) return st;
    B.G = G;
    B.nslots = max_slots;
    // per-CTA mailbox ranges: [g_scan[cta_p0[c]], g_scan[cta_p0[c+1]])
    if ((st = h->arena.alloc_n(&B.d_cta_g0, (size_t)K + 1)) != SPTRSV_SUCCESS) return st;
    {
        std::vector<int32_t> hp0(K + 1), hg0(K + 1);
        SPTRSV_CUDA(cudaMemcpyAsync(hp0.data(), cta_p0, sizeof(int32_t) * (K + 1), cudaMemcpyDeviceToHost, s));
        SPTRSV_CUDA(cudaStreamSynchronize(s));
        for (int c = 0; c <= K; ++c) {
            hg0[c] = i32_at(g_scan, hp0[c], s, st);
            if (st != SPTRSV_SUCCESS) return st;
        }
        SPTRSV_CUDA(cudaMemcpyAsync(B.d_cta_g0, hg0.data(), sizeof(int32_t) * (K + 1), cudaMemcpyHostToDevice, s));
    }

    // ---- 5. overflow lists and records
    int32_t *ocnt = nullptr, *ovf_ptr = nullptr;
    if ((st = tmp.alloc_n(&ocnt, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&ovf_ptr, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    k_ovf_count<<<(n + 1 + 255) / 256, 256, 0, s>>>(n, WE, ecnt, ocnt);
    if ((st = exclusive_scan_i32(ocnt, ovf_ptr, (int64_t)n + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    const int32_t novf = i32_at(ovf_ptr, n, s, st);
    if (st != SPTRSV_SUCCESS) return st;
    B.novf = novf;
    // + 4 padding steps: a warp's last block of records / row ids is copied whole
    if ((st = h->arena.alloc(&B.d_recs, (size_t)((int64_t)nsteps + 4) * REC)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&B.d_rows, (size_t)((int64_t)nsteps + 4) * 32)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemsetAsync((unsigned char *)B.d_recs + (size_t)nsteps * REC, 0xFF, (size_t)4 * REC, s));
    SPTRSV_CUDA(cudaMemsetAsync(B.d_rows + (size_t)nsteps * 32, 0xFF, (size_t)4 * 128, s));
    if ((st = h->arena.alloc_n(&B.d_ovf_code, (size_t)std::max(novf, 1))) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc(&B.d_ovf_val, (size_t)std::max(novf, 1) * es)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc(&B.d_gmb, (size_t)2 * std::max(G, 1) * es)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&B.d_ctr, 2)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemsetAsync(B.d_ctr, 0, 2 * sizeof(unsigned), s));
    const int pg = (int)std::max<int64_t>(1, ((int64_t)nsteps * 32 + 255) / 256);
    const int fg = std::max(1, std::min((int)((2 * (int64_t)std::max(G, 1) + 255) / 256), h->num_sms * 8));
    if (h->dtype == SPTRSV_F64) {
        k_rec_fill<double><<<pg, 256, 0, s>>>(nsteps, kSH, WE, wpc, steps, bperm, pos, step_of, unit, tri_ptr,
                                              tri_col, (const double *)tri_val, (const double *)h->d_invd_row,
                                              h->diag == SPTRSV_UNIT, noslot, need, ecnt, slot_scan, g_scan, cta_p0, ovf_ptr, (unsigned char *)B.d_recs,
                                              B.d_rows, B.d_ovf_code, (double *)B.d_ovf_val);
        k_fill_sentinel<double><<<fg, 256, 0, s>>>((double *)B.d_gmb, 2 * (int64_t)std::max(G, 1));
    } else {
        k_rec_fill<float><<<pg, 256, 0, s>>>(nsteps, kSH, WE, wpc, steps, bperm, pos, step_of, unit, tri_ptr,
                                             tri_col, (const float *)tri_val, (const float *)h->d_invd_row,
                                             h->diag == SPTRSV_UNIT, noslot, need, ecnt, slot_scan, g_scan, cta_p0, ovf_ptr, (unsigned char *)B.d_recs,
                                             B.d_rows, B.d_ovf_code, (float *)B.d_ovf_val);
        k_fill_sentinel<float><<<fg, 256, 0, s>>>((float *)B.d_gmb, 2 * (int64_t)std::max(G, 1));
    }
    SPTRSV_CUDA(cudaGetLastError());

    // ---- launch configuration: K co-resident CTAs of wpc tiles (2 warps each)
    const size_t smem = fixed_bytes() + (size_t)max_slots * es;
    SPTRSV_CUDA(cudaFuncSetAttribute(kn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    const int tpw = lean ? 32 : 96;          // threads per tile
    SPTRSV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kn, tpw * wpc, smem));
    if (per_sm * h->num_sms < K) return SPTRSV_ERR_NOT_SUPPORTED;
    B.kernel = kn;
    B.smem = smem;
    B.threads = tpw * wpc;
    B.lean = lean;
    B.nst = lean ? kLNBB * kLUB : kNBB * ub_of(WE);
    B.bb = lean ? 2 : kR2B * ub_of(WE);
    B.d = lean ? kLDB * kLUB : kDB * ub_of(WE);
    B.W = WE;
    B.rec_bytes = REC;
    B.nent = (int64_t)nsteps * REC;
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    B.built = true;
    return SPTRSV_SUCCESS;
}

// ---------------------------------------------------------------- CTA-tile multi-RHS plan
// Positions sorted by (CTA, level, row) with the BLOCK partition's CTAs; a
// per-position CSR (same shape as the level-ordered multi-RHS CSR, so the
// row kernels are shared); per (CTA, level) position ranges; per CTA the list
// of CTAs that produce its dependencies.  k_tile_mrhs (solve.cu) walks each
// CTA's levels with __syncthreads between them and waits only for its
// producer CTAs' level counters: no grid-wide barrier.
__global__ void k_tm_keys(int n, int nlev, int wpc, const int32_t *unit, const int32_t *lev, uint32_t *keys,
                          int32_t *cnt) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t k = (uint32_t)(unit[i] / wpc) * (uint32_t)nlev + (uint32_t)lev[i];
    keys[i] = k;
    atomicAdd(&cnt[k], 1);
}

template <typename T>
__global__ void k_tm_rows(int n, const int32_t *perm, const int32_t *dp, const T *invd_row, int unit_diag,
                          T *invd, int32_t *deg) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) {
        const int i = perm[p];
        invd[p] = unit_diag ? T(1) : invd_row[i];
        deg[p] = dp[i];
    }
    if (p == n) deg[p] = 0;
}

template <typename T>
__global__ void k_tm_fill(int n, int K, int wpc, const int32_t *perm, const int32_t *tri_ptr, const int32_t *tri_col,
                          const T *tri_val, const int32_t *unit, const int32_t *ptr, int32_t *col, T *val,
                          unsigned char *depm) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int i = perm[p];
    const int ci = unit[i] / wpc;
    int o = ptr[p];
    for (int k = tri_ptr[i]; k < tri_ptr[i + 1]; ++k, ++o) {
        const int j = tri_col[k];
        col[o] = j;
        val[o] = tri_val[k];
        const int cj = unit[j] / wpc;
        if (cj != ci) depm[(size_t)ci * K + cj] = 1;
    }
}

sptrsv_status_t tile_mrhs_build(sptrsv_handle_t h, cudaStream_t s) {
    BlockPlan &B = h->block;
    if (!B.built || B.grid_nx == 0) return SPTRSV_ERR_NOT_SUPPORTED;
    const int n = h->n, nlev = h->info.nlev, K = B.nblocks, wpc = B.wpc;
    const size_t es = h->esize;
    if ((uint64_t)K * (uint64_t)nlev >= (1ull << 31)) return SPTRSV_ERR_NOT_SUPPORTED;
    DevArena tmp;
    struct Guard {
        DevArena &a;
        ~Guard() { a.release_all(); }
    } guard{tmp};
    sptrsv_status_t st;
    const int eg = (n + 256) / 256;
    // natural-order CSR of the triangle (as in block_build)
    int32_t *tri_ptr = nullptr, *tri_col = nullptr, *dpx = nullptr;
    void *tri_val = nullptr;
    const int64_t nnz = std::max<int64_t>(h->info.nnz_used, 1);
    if ((st = tmp.alloc_n(&tri_ptr, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&tri_col, (size_t)nnz)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc(&tri_val, (size_t)nnz * es)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&dpx, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemcpyAsync(dpx, h->d_dp, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
    SPTRSV_CUDA(cudaMemsetAsync(dpx + n, 0, sizeof(int32_t), s));
    if ((st = exclusive_scan_i32(dpx, tri_ptr, (int64_t)n + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    const int cgrid = std::max(1, std::min((h->nchunks * 32 + 255) / 256, h->num_sms * 16));
    if (h->dtype == SPTRSV_F64)
        k_tri_fill<double><<<cgrid, 256, 0, s>>>(h->nchunks, h->d_chunks, h->d_perm, h->d_ecol,
                                                 (const double *)h->d_eval, tri_ptr, tri_col, (double *)tri_val);
    else
        k_tri_fill<float><<<cgrid, 256, 0, s>>>(h->nchunks, h->d_chunks, h->d_perm, h->d_ecol,
                                                (const float *)h->d_eval, tri_ptr, tri_col, (float *)tri_val);
    // order by (CTA, level, row); (CTA, level) offsets
    const int64_t KL = (int64_t)K * nlev;
    uint32_t *keys = nullptr, *skeys = nullptr;
    int32_t *cnt = nullptr, *deg = nullptr;
    unsigned char *depm = nullptr;
    if ((st = tmp.alloc_n(&keys, n)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&skeys, n)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&cnt, (size_t)KL + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&deg, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&depm, (size_t)K * K)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&B.d_tm_perm, n)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc(&B.d_tm_invd, (size_t)n * es)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&B.d_tm_ptr, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&B.d_tm_col, (size_t)nnz)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc(&B.d_tm_val, (size_t)nnz * es)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&B.d_tm_off, (size_t)KL + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&B.d_tm_done, (size_t)K)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * ((size_t)KL + 1), s));
    SPTRSV_CUDA(cudaMemsetAsync(depm, 0, (size_t)K * K, s));
    SPTRSV_CUDA(cudaMemsetAsync(B.d_tm_done, 0, sizeof(unsigned long long) * K, s));
    k_tm_keys<<<eg, 256, 0, s>>>(n, nlev, wpc, B.d_unit, h->d_lev, keys, cnt);
    if ((st = radix_sort_pairs(keys, nullptr, skeys, B.d_tm_perm, n, (uint32_t)(KL - 1), tmp, s)) != SPTRSV_SUCCESS)
        return st;
    if ((st = exclusive_scan_i32(cnt, B.d_tm_off, (int64_t)KL + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    if (h->dtype == SPTRSV_F64)
        k_tm_rows<double><<<eg, 256, 0, s>>>(n, B.d_tm_perm, h->d_dp, (const double *)h->d_invd_row,
                                             h->diag == SPTRSV_UNIT, (double *)B.d_tm_invd, deg);
    else
        k_tm_rows<float><<<eg, 256, 0, s>>>(n, B.d_tm_perm, h->d_dp, (const float *)h->d_invd_row,
                                            h->diag == SPTRSV_UNIT, (float *)B.d_tm_invd, deg);
    if ((st = exclusive_scan_i32(deg, B.d_tm_ptr, (int64_t)n + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    if (h->dtype == SPTRSV_F64)
        k_tm_fill<double><<<eg, 256, 0, s>>>(n, K, wpc, B.d_tm_perm, tri_ptr, tri_col, (const double *)tri_val,
                                             B.d_unit, B.d_tm_ptr, B.d_tm_col, (double *)B.d_tm_val, depm);
    else
        k_tm_fill<float><<<eg, 256, 0, s>>>(n, K, wpc, B.d_tm_perm, tri_ptr, tri_col, (const float *)tri_val,
                                            B.d_unit, B.d_tm_ptr, B.d_tm_col, (float *)B.d_tm_val, depm);
    SPTRSV_CUDA(cudaGetLastError());
    // producer lists
    std::vector<unsigned char> hdep((size_t)K * K);
    SPTRSV_CUDA(cudaMemcpyAsync(hdep.data(), depm, (size_t)K * K, cudaMemcpyDeviceToHost, s));
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    std::vector<int32_t> dptr(K + 1, 0), dl;
    for (int c = 0; c < K; ++c) {
        for (int p = 0; p < K; ++p)
            if (hdep[(size_t)c * K + p]) dl.push_back(p);
        dptr[c + 1] = (int32_t)dl.size();
    }
    if (dl.empty()) dl.push_back(0);
    if ((st = h->arena.alloc_n(&B.d_tm_dptr, (size_t)K + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&B.d_tm_dl, dl.size())) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemcpyAsync(B.d_tm_dptr, dptr.data(), sizeof(int32_t) * (K + 1), cudaMemcpyHostToDevice, s));
    SPTRSV_CUDA(cudaMemcpyAsync(B.d_tm_dl, dl.data(), sizeof(int32_t) * dl.size(), cudaMemcpyHostToDevice, s));
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    B.tm_K = K;
    B.tm_base = 0;
    B.tm_built = true;
    h->info.device_bytes = h->arena.bytes;
    return SPTRSV_SUCCESS;
}

sptrsv_status_t block_solve(sptrsv_handle_t h, const void *b, void *x, cudaStream_t s) {
    BlockPlan &B = h->block;
    if (!B.built) return SPTRSV_ERR_NOT_SUPPORTED;
    BlockArgs a;
    a.unit_step0 = B.d_unit_step0;
    a.recs = (const unsigned char *)B.d_recs;
    a.rows = B.d_rows;
    a.cta_g0 = B.d_cta_g0;
    a.ovf_code = B.d_ovf_code;
    a.ovf_val = B.d_ovf_val;
    a.gmb = B.d_gmb;
    a.ctr = B.d_ctr;
    a.b = b;
    a.x = x;
    a.G = B.G;
    a.nslots = B.nslots;
    void *args[] = {(void *)&a};
    SPTRSV_CUDA(cudaLaunchCooperativeKernel(B.kernel, B.nblocks, B.threads, args, B.smem, s));
    return SPTRSV_SUCCESS;
}

}  // namespace sptrsv

// Debug hook (not part of include/sptrsv.h): install a device trace buffer of
// (#warps) x cap uint64 timestamps for SPTRSV_ALGO_BLOCK solves (NULL disables).
extern "C" int sptrsv_dbg_block_trace(void *dev_buf, int cap) {
    unsigned long long *p = (unsigned long long *)dev_buf;
    if (cudaMemcpyToSymbol(sptrsv::g_trace, &p, sizeof(p)) != cudaSuccess) return 5;
    if (cudaMemcpyToSymbol(sptrsv::g_trace_cap, &cap, sizeof(int)) != cudaSuccess) return 5;
    sptrsv::g_host_trace = (dev_buf != nullptr);
    return 0;
}

extern "C" int sptrsv_dbg_block_phase(void *dev_buf) {
    unsigned long long *p = (unsigned long long *)dev_buf;
    return cudaMemcpyToSymbol(sptrsv::g_phase, &p, sizeof(p)) == cudaSuccess ? 0 : 5;
}

// Debug hook: returns and clears the spin-watchdog flag (1 = a wait gave up).
extern "C" int sptrsv_dbg_watchdog(void) {
    unsigned v = 0, z = 0;
    cudaMemcpyFromSymbol(&v, sptrsv::g_watchdog, sizeof(v));
    cudaMemcpyToSymbol(sptrsv::g_watchdog, &z, sizeof(z));
    return (int)v;
}
