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

// record geometry (W entries per row; SoA over 32 lanes; both parts 16 B multiples)
__host__ __device__ constexpr int rec_ibytes(int W) { return 32 * 4 * (4 + W); }
__host__ __device__ constexpr int rec_bytes(int W, int es) { return rec_ibytes(W) + 32 * es * (1 + W); }

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

// Dependency classes -> which producers need a shared slot (bit 0) or a global
// mailbox (bit 1).  A row with more than W dependencies (or in a CTA whose
// slots overflowed: noslot) takes no SHFL / SMEM codes respectively.
__global__ void k_need(int n, int W, int wpc, const int32_t *__restrict__ tri_ptr, const int32_t *__restrict__ tri_col,
                       const int32_t *__restrict__ unit, const int32_t *__restrict__ pos,
                       const int32_t *__restrict__ step_of, const unsigned char *__restrict__ noslot,
                       int32_t *need) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int a = tri_ptr[i], e = tri_ptr[i + 1];
    const bool ovf = e - a > W;
    const int ui = unit[i], si = step_of[pos[i]];
    const bool ns = noslot[ui / wpc] != 0;
    for (int k = a; k < e; ++k) {
        const int j = tri_col[k];
        const int uj = unit[j], pj = pos[j];
        if (!ovf && uj == ui && step_of[pj] == si - 1) continue;        // SHFL
        if (uj / wpc == ui / wpc && !ns) atomicOr(&need[pj], 1);
        else atomicOr(&need[pj], 2);
    }
}

__global__ void k_need_bits(int n, const int32_t *need, int bit, int32_t *out) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) out[p] = (need[p] >> bit) & 1;
    if (p == n) out[p] = 0;
}

__global__ void k_ovf_count(int n, int W, const int32_t *bperm, const int32_t *tri_ptr, int32_t *cnt) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) {
        const int i = bperm[p];
        const int d = tri_ptr[i + 1] - tri_ptr[i];
        cnt[p] = d > W ? d + 1 : 0;          // + terminator
    }
    if (p == n) cnt[p] = 0;
}

// per CTA: number of shared slots it needs
__global__ void k_cta_slots(int K, const int32_t *cta_p0, const int32_t *slot_scan, int32_t *cnt) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < K) cnt[c] = slot_scan[cta_p0[c + 1]] - slot_scan[cta_p0[c]];
}

// one thread per (step, lane): the record of that lane (padding lanes included)
template <typename T>
__global__ void k_rec_fill(int nsteps, int W, int wpc, const int2 *__restrict__ steps,
                           const int32_t *__restrict__ step_unit, const int32_t *__restrict__ bperm,
                           const int32_t *__restrict__ pos, const int32_t *__restrict__ step_of,
                           const int32_t *__restrict__ unit, const int32_t *__restrict__ tri_ptr,
                           const int32_t *__restrict__ tri_col, const T *__restrict__ tri_val,
                           const T *__restrict__ invd_row, const unsigned char *__restrict__ noslot,
                           const int32_t *__restrict__ need, const int32_t *__restrict__ slot_scan,
                           const int32_t *__restrict__ g_scan, const int32_t *__restrict__ cta_p0,
                           const int32_t *__restrict__ ovf_ptr, unsigned char *__restrict__ recs,
                           int32_t *__restrict__ ovf_code, T *__restrict__ ovf_val) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long long)nsteps * 32) return;
    const int s = (int)(t >> 5), lane = (int)(t & 31);
    const int REC = rec_bytes(W, sizeof(T));
    unsigned char *base = recs + (size_t)s * REC;
    int32_t *ip = reinterpret_cast<int32_t *>(base);
    T *vp = reinterpret_cast<T *>(base + rec_ibytes(W));
    const int2 st = steps[s];
    if (lane >= st.y) {
        ip[lane] = -1;
        ip[32 + lane] = -1;
        ip[64 + lane] = -1;
        ip[96 + lane] = -1;
        for (int k = 0; k < W; ++k) {
            ip[(4 + k) * 32 + lane] = kNone;
            vp[(1 + k) * 32 + lane] = T(0);
        }
        vp[lane] = T(0);
        return;
    }
    const int p = st.x + lane;
    const int i = bperm[p];
    const int ui = unit[i], ci = ui / wpc;
    const bool ns = noslot[ci] != 0;
    const int nd = need[p];
    ip[lane] = i;
    ip[32 + lane] = (nd & 1) ? slot_scan[p] - slot_scan[cta_p0[ci]] : -1;
    ip[64 + lane] = (nd & 2) ? g_scan[p] : -1;
    vp[lane] = invd_row[i];
    const int a = tri_ptr[i], e = tri_ptr[i + 1];
    const bool ovf = e - a > W;
    auto code_of = [&](int j, bool allow_shfl, bool &is_shfl) -> int32_t {
        const int uj = unit[j], pj = pos[j];
        is_shfl = false;
        if (allow_shfl && uj == ui && step_of[pj] == s - 1) {
            is_shfl = true;
            return pj - steps[s - 1].x;                       // lane of j in the previous step
        }
        if (uj / wpc == ci && !ns) return code_smem(slot_scan[pj] - slot_scan[cta_p0[ci]]);
        return code_glob(g_scan[pj]);
    };
    if (ovf) {
        ip[96 + lane] = ovf_ptr[p];
        int o = ovf_ptr[p];
        bool sh;
        for (int k = a; k < e; ++k, ++o) {
            ovf_code[o] = code_of(tri_col[k], false, sh);
            ovf_val[o] = tri_val[k];
        }
        ovf_code[o] = kNone;
        ovf_val[o] = T(0);
        for (int k = 0; k < W; ++k) {
            ip[(4 + k) * 32 + lane] = kNone;
            vp[(1 + k) * 32 + lane] = T(0);
        }
        return;
    }
    ip[96 + lane] = -1;
    // non-SHFL terms first, then SHFL terms, each in storage order
    int w = 0;
    for (int pass = 0; pass < 2; ++pass)
        for (int k = a; k < e; ++k) {
            bool sh;
            const int32_t c = code_of(tri_col[k], true, sh);
            if (sh != (pass == 1)) continue;
            ip[(4 + w) * 32 + lane] = c;
            vp[(1 + w) * 32 + lane] = tri_val[k];
            ++w;
        }
    for (; w < W; ++w) {
        ip[(4 + w) * 32 + lane] = kNone;
        vp[(1 + w) * 32 + lane] = T(0);
    }
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
    const int32_t *cta_g0;
    const int32_t *ovf_code;
    const void *ovf_val;
    void *gmb;
    unsigned *ctr;
    const void *b;
    void *x;
    int G, nst, nslots, bb;
};

template <typename T, int W>
struct Fields {
    int row, oslot, og, ovf;
    int32_t code[W];
    T invd;
    T val[W];
    T g[W];
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
__device__ __forceinline__ void stg_flag(double *p, double v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"((unsigned long long)__double_as_longlong(v)));
}
__device__ __forceinline__ void stg_flag(float *p, float v) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(__float_as_uint(v)));
}

// Pipeline per warp, in blocks of UB steps (no mbarrier on the step path;
// cp.async groups are per thread, one group per block):
//   group G(k), issued at the end of block k = { records of block k + NB
//   (every lane copies 16-byte pieces), b[row] of block k + BB (own lane) },
//   ring = NB blocks of records, BB blocks of b, NB >= 2 BB.
//   Start of block k: cp.async.wait_group(BB - 1) + __syncwarp -> every group
//   <= G(k - BB) landed in every lane: b of block k, the records of block k
//   and of block k + BB (whose rows the b gather of G(k) needs).
//   Then the UB records and b values go to registers (LDS), and the UB steps
//   run back to back: only shuffles, FMAs and stores between two levels.
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

template <typename T, bool UNIT, int W, int UB>
__global__ void __launch_bounds__(256, 1) k_block(const BlockArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ unsigned s_epoch;
    constexpr int REC = rec_bytes(W, sizeof(T));
    constexpr int IB = rec_ibytes(W);
    constexpr int NPIECE = REC * UB / 16;         // 16-byte pieces of one block of records
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wpc = blockDim.x >> 5;
    const int nst = a.nst;                        // ring length in steps (NB * UB)
    const int NB = nst / UB, BB = a.bb;
    unsigned char *rings = smem_raw;
    T *bring = reinterpret_cast<T *>(smem_raw + (size_t)wpc * nst * REC);
    T *slots = bring + wpc * BB * UB * 32;
    const T *b = static_cast<const T *>(a.b);
    T *x = static_cast<T *>(a.x);

    for (int i = threadIdx.x; i < a.nslots; i += blockDim.x) slots[i] = Sentinel<T>::value();
    if (threadIdx.x == 0) s_epoch = (unsigned)ld_relaxed(reinterpret_cast<const int *>(a.ctr));
    __syncthreads();
    const unsigned par = s_epoch & 1u;
    T *gm = static_cast<T *>(a.gmb) + (size_t)par * a.G;
    {   // re-arm this CTA's mailboxes of the idle array (written by the previous solve)
        T *go = static_cast<T *>(a.gmb) + (size_t)(par ^ 1u) * a.G;
        for (int i = a.cta_g0[blockIdx.x] + threadIdx.x; i < a.cta_g0[blockIdx.x + 1]; i += blockDim.x)
            go[i] = Sentinel<T>::value();
    }

    const int u = blockIdx.x * wpc + warp;
    const int s0 = a.unit_step0[u], s1 = a.unit_step0[u + 1];
    if (s0 < s1) {
        unsigned char *ring = rings + (size_t)warp * nst * REC;
        T *br = bring + warp * BB * UB * 32;
        const int nblk = (s1 - s0 + UB - 1) / UB;
        // a warp's last block may read past its steps (the next warp's records,
        // or the analysis' padding steps): they are never solved
        auto blk_of = [&](int k) { return ring + (size_t)(k % NB) * (UB * REC); };
        auto issue_rec = [&](int k) {            // block k of this warp
            const unsigned char *src = a.recs + (size_t)(s0 + k * UB) * REC;
            unsigned char *dst = blk_of(k);
#pragma unroll
            for (int q = lane; q < NPIECE; q += 32) cp_async_16(dst + 16 * q, src + 16 * q);
        };
        auto issue_b = [&](int k) {
#pragma unroll
            for (int j = 0; j < UB; ++j) {
                const int r = reinterpret_cast<const int32_t *>(blk_of(k) + j * REC)[lane];
                if (r >= 0) cp_async_val(&br[(((k % BB) * UB) + j) * 32 + lane], b + r);
            }
        };
        // SMEM values: loaded one step ahead (shared-memory latency);
        // GLOB values (another SM, an L2 round trip): one whole block ahead
        auto prefetch_smem = [&](Fields<T, W> &F) {
#pragma unroll
            for (int q = 0; q < W; ++q)
                if (code_kind(F.code[q]) != 2u)
                    F.g[q] = lds_flag_if(slots + code_idx(F.code[q]), code_kind(F.code[q]) == 1u);
        };
        auto prefetch_glob = [&](T (&g)[UB][W], int k) {
#pragma unroll
            for (int j = 0; j < UB; ++j) {
                const int32_t *ip = reinterpret_cast<const int32_t *>(blk_of(k) + j * REC);
#pragma unroll
                for (int q = 0; q < W; ++q) {
                    const int32_t c = ip[(4 + q) * 32 + lane];
                    g[j][q] = ldg_flag_if(gm + code_idx(c), code_kind(c) == 2u);
                }
            }
        };

#pragma unroll 1
        for (int k = 0; k < min(nblk, NB); ++k) issue_rec(k);
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
#pragma unroll 1
        for (int k = 0; k < BB; ++k) {
            if (k < nblk) issue_b(k);
            cp_async_commit();
        }
        T gnx[UB][W];
        prefetch_glob(gnx, 0);
        T xprev = T(0);
        const bool trace = g_trace != nullptr;
#pragma unroll 1
        for (int k = 0; k < nblk; ++k) {
            if (trace && lane == 0 && k * UB < g_trace_cap - 1) g_trace[(size_t)u * g_trace_cap + k * UB] = wd_now();
            cp_async_wait_n(BB - 1);
            __syncwarp();
            Fields<T, W> F[UB];
            T bv[UB];
#pragma unroll
            for (int j = 0; j < UB; ++j) {
                const unsigned char *r = blk_of(k) + j * REC;
                const int32_t *ip = reinterpret_cast<const int32_t *>(r);
                const T *vp = reinterpret_cast<const T *>(r + IB);
                F[j].row = ip[lane];
                F[j].oslot = ip[32 + lane];
                F[j].og = ip[64 + lane];
                F[j].ovf = ip[96 + lane];
#pragma unroll
                for (int q = 0; q < W; ++q) F[j].code[q] = ip[(4 + q) * 32 + lane];
                F[j].invd = vp[lane];
#pragma unroll
                for (int q = 0; q < W; ++q) F[j].val[q] = vp[(1 + q) * 32 + lane];
                bv[j] = br[(((k % BB) * UB) + j) * 32 + lane];
#pragma unroll
                for (int q = 0; q < W; ++q) F[j].g[q] = gnx[j][q];
            }
            if (k + 1 < nblk) prefetch_glob(gnx, k + 1);
            prefetch_smem(F[0]);
#pragma unroll
            for (int j = 0; j < UB; ++j) {
                if (UB > 1 && k * UB + j >= s1 - s0) break;          // warp-uniform tail
                // SHFL sources from the previous step's registers; SMEM / GLOB
                // values were prefetched (re-polled only if still the sentinel)
                T vs[W];
#pragma unroll
                for (int q = 0; q < W; ++q) vs[q] = __shfl_sync(0xffffffffu, xprev, F[j].code[q] & 31);
                bool pend = false;
#pragma unroll
                for (int q = 0; q < W; ++q) pend |= Sentinel<T>::is(F[j].g[q]);
                if (pend) {
#pragma unroll
                    for (int q = 0; q < W; ++q)
                        if (Sentinel<T>::is(F[j].g[q]))
                            F[j].g[q] = code_kind(F[j].code[q]) == 1u ? poll_smem_slow(slots + code_idx(F[j].code[q]))
                                                                     : poll_global_slow(gm + code_idx(F[j].code[q]));
                }
                T acc = bv[j];
#pragma unroll
                for (int q = 0; q < W; ++q)
                    acc = fnma(F[j].val[q], code_kind(F[j].code[q]) == 0u ? vs[q] : F[j].g[q], acc);
                if (F[j].ovf >= 0) {
                    const T *ov = static_cast<const T *>(a.ovf_val);
                    for (int o = F[j].ovf;; ++o) {
                        const int32_t c = a.ovf_code[o];
                        if (c == kNone) break;
                        T v;
                        if (code_kind(c) == 1u) {
                            v = lds_volatile(slots + code_idx(c));
                            if (Sentinel<T>::is(v)) v = poll_smem_slow(slots + code_idx(c));
                        } else {
                            v = ld_relaxed_val(gm + code_idx(c));
                            if (Sentinel<T>::is(v)) v = poll_global_slow(gm + code_idx(c));
                        }
                        acc = fnma(ov[o], v, acc);
                    }
                }
                const T xi = Sentinel<T>::scrub(UNIT ? acc : acc * F[j].invd);
                if (F[j].oslot >= 0) sts_flag(slots + F[j].oslot, xi);
                if (F[j].og >= 0) stg_flag(gm + F[j].og, xi);
                if (F[j].row >= 0) __stcg(x + F[j].row, xi);
                xprev = xi;
                if (j + 1 < UB) prefetch_smem(F[j + 1]);
            }
            __syncwarp();                       // every lane is done with block k: its ring slots are free
            if (k + NB < nblk) issue_rec(k + NB);
            if (k + BB < nblk) issue_b(k + BB);
            cp_async_commit();
        }
        cp_async_wait<0>();
        if (trace && lane == 0) g_trace[(size_t)u * g_trace_cap + min(s1 - s0, g_trace_cap - 1)] = wd_now();
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

// record width W (>= max dependencies, else overflow lists), UB steps per
// block (registers: UB records live at once), BB blocks of b lookahead
// record width W (>= max dependencies, else overflow lists), ub steps per
// block (registers: ub records live at once)
template <typename T, bool UNIT>
void *pick_kernel(int W, int &Wk, int &ub) {
    if (W <= 3) { Wk = 3; ub = 4; return (void *)k_block<T, UNIT, 3, 4>; }
    if (W <= 4) { Wk = 4; ub = 4; return (void *)k_block<T, UNIT, 4, 4>; }
    if (W <= 8) { Wk = 8; ub = 2; return (void *)k_block<T, UNIT, 8, 2>; }
    if (W <= 13) { Wk = 13; ub = 1; return (void *)k_block<T, UNIT, 13, 1>; }
    Wk = 16; ub = 1;
    return (void *)k_block<T, UNIT, 16, 1>;
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

    // kernel instance (record width W) and shared-memory budget
    int Wk = 0, ub = 1;
    const int W = std::max(1, std::min(h->info.max_row_deps, 16));
    void *kn = nullptr;
    if (h->dtype == SPTRSV_F64)
        kn = h->diag == SPTRSV_UNIT ? pick_kernel<double, true>(W, Wk, ub) : pick_kernel<double, false>(W, Wk, ub);
    else
        kn = h->diag == SPTRSV_UNIT ? pick_kernel<float, true>(W, Wk, ub) : pick_kernel<float, false>(W, Wk, ub);
    // lookahead in blocks of ub steps: b gathered bb blocks ahead, records
    // nb >= 2 bb blocks ahead (bb <= 8: cp.async.wait_group immediate)
    const int bb = std::max(1, std::min(env_int("SPTRSV_BLOCK_BB", std::max(1, 8 / ub)), 8));
    const int pb = bb * ub;          // steps of b ring per warp
    const int REC = rec_bytes(Wk, (int)es);
    const size_t budget = (size_t)max_smem - 1024;          // static smem + slack
    // per CTA: record rings (nst per warp) + b rings; the rest holds shared slots
    auto ring_bytes = [&](int nw, int ns) { return (size_t)nw * ns * REC + (size_t)nw * pb * 32 * es; };

    // ---- 2. partition rows over U = K x wpc warps of K co-resident CTAs
    int32_t *unit = nullptr;
    if ((st = tmp.alloc_n(&unit, n)) != SPTRSV_SUCCESS) return st;
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
        static const int shapes[][2] = {{1, 1}, {2, 1}, {1, 2}, {2, 2}, {4, 2}, {2, 4}};
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
        while (wpc > 1 && ring_bytes(wpc, 2 * pb) + 2048 * es > budget) wpc /= 2;
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
    int nst = std::max(env_int("SPTRSV_BLOCK_NST", 2 * pb), 2 * pb);
    nst = (nst + ub - 1) / ub * ub;
    auto fixed_bytes = [&](int ns) { return ring_bytes(wpc, ns); };
    if (nst < 2 * pb || fixed_bytes(nst) > budget) return SPTRSV_ERR_NOT_SUPPORTED;
    const int cap = (int)((budget - fixed_bytes(nst)) / es);

    unsigned char *noslot = nullptr;
    int32_t *need = nullptr, *bits = nullptr, *slot_scan = nullptr, *g_scan = nullptr, *ccnt = nullptr;
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
        k_need<<<eg, 256, 0, s>>>(n, Wk, wpc, tri_ptr, tri_col, unit, pos, step_of, noslot, need);
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
    k_ovf_count<<<(n + 1 + 255) / 256, 256, 0, s>>>(n, Wk, bperm, tri_ptr, ocnt);
    if ((st = exclusive_scan_i32(ocnt, ovf_ptr, (int64_t)n + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    const int32_t novf = i32_at(ovf_ptr, n, s, st);
    if (st != SPTRSV_SUCCESS) return st;
    B.novf = novf;
    // + 16 padding steps (0xFF: row -1, codes NONE) so a warp's last block of ub
    // records can be read whole
    if ((st = h->arena.alloc(&B.d_recs, (size_t)((int64_t)nsteps + 16) * REC)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemsetAsync((unsigned char *)B.d_recs + (size_t)nsteps * REC, 0xFF, (size_t)16 * REC, s));
    if ((st = h->arena.alloc_n(&B.d_ovf_code, (size_t)std::max(novf, 1))) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc(&B.d_ovf_val, (size_t)std::max(novf, 1) * es)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc(&B.d_gmb, (size_t)2 * std::max(G, 1) * es)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&B.d_ctr, 2)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemsetAsync(B.d_ctr, 0, 2 * sizeof(unsigned), s));
    const int pg = (int)std::max<int64_t>(1, ((int64_t)nsteps * 32 + 255) / 256);
    const int fg = std::max(1, std::min((int)((2 * (int64_t)std::max(G, 1) + 255) / 256), h->num_sms * 8));
    if (h->dtype == SPTRSV_F64) {
        k_rec_fill<double><<<pg, 256, 0, s>>>(nsteps, Wk, wpc, steps, step_unit, bperm, pos, step_of, unit, tri_ptr,
                                              tri_col, (const double *)tri_val, (const double *)h->d_invd_row, noslot,
                                              need, slot_scan, g_scan, cta_p0, ovf_ptr, (unsigned char *)B.d_recs,
                                              B.d_ovf_code, (double *)B.d_ovf_val);
        k_fill_sentinel<double><<<fg, 256, 0, s>>>((double *)B.d_gmb, 2 * (int64_t)std::max(G, 1));
    } else {
        k_rec_fill<float><<<pg, 256, 0, s>>>(nsteps, Wk, wpc, steps, step_unit, bperm, pos, step_of, unit, tri_ptr,
                                             tri_col, (const float *)tri_val, (const float *)h->d_invd_row, noslot,
                                             need, slot_scan, g_scan, cta_p0, ovf_ptr, (unsigned char *)B.d_recs,
                                             B.d_ovf_code, (float *)B.d_ovf_val);
        k_fill_sentinel<float><<<fg, 256, 0, s>>>((float *)B.d_gmb, 2 * (int64_t)std::max(G, 1));
    }
    SPTRSV_CUDA(cudaGetLastError());

    // ---- launch configuration: K co-resident CTAs of wpc warps
    const size_t smem = fixed_bytes(nst) + (size_t)max_slots * es;
    SPTRSV_CUDA(cudaFuncSetAttribute(kn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    SPTRSV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kn, 32 * wpc, smem));
    if (per_sm * h->num_sms < K) return SPTRSV_ERR_NOT_SUPPORTED;
    B.kernel = kn;
    B.smem = smem;
    B.threads = 32 * wpc;
    B.nst = nst;
    B.bb = bb;
    B.W = Wk;
    B.rec_bytes = REC;
    B.nent = (int64_t)nsteps * REC;
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    B.built = true;
    return SPTRSV_SUCCESS;
}

sptrsv_status_t block_solve(sptrsv_handle_t h, const void *b, void *x, cudaStream_t s) {
    BlockPlan &B = h->block;
    if (!B.built) return SPTRSV_ERR_NOT_SUPPORTED;
    BlockArgs a;
    a.unit_step0 = B.d_unit_step0;
    a.recs = (const unsigned char *)B.d_recs;
    a.cta_g0 = B.d_cta_g0;
    a.ovf_code = B.d_ovf_code;
    a.ovf_val = B.d_ovf_val;
    a.gmb = B.d_gmb;
    a.ctr = B.d_ctr;
    a.b = b;
    a.x = x;
    a.G = B.G;
    a.nst = B.nst;
    a.nslots = B.nslots;
    a.bb = B.bb;
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
