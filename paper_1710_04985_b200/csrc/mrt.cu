// mrt.cu -- multi-RHS tile solve (a8; many right-hand
// sides amortise the matrix stream): the paper's row update applied to nrhs
// columns at once, self-scheduled between CTAs, level-synchronous inside one.
//
// Layout.  Rows are partitioned over K co-resident CTAs (the BLOCK tile
// partition when the analysis detected a structured grid -- a CTA owns a
// rectangle of z-columns -- else contiguous natural-order row blocks).  A
// CTA's rows are sorted by (level, row) and cut into GROUPS of <= kGmax rows
// of one level; a CTA solves its groups in order, one column block of <= 64
// right-hand sides per launch.  Every dependency value a group reads is in
// shared memory:
//   * rows of the CTA's previous group: its output buffer (kept per group);
//   * every other row (another CTA's, or an older group of this CTA): the
//     group's HALO buffer, filled by TMA bulk copies of those x rows before
//     the group starts (<= kHmax distinct rows per group; any further ones --
//     never on the 5-/7-point factors -- are loaded from global memory).
// Per solve position a record {row, #deps, dep slot[4] (storage order), a[4],
// 1/d}: slot < kGmax is a previous-group row, slot >= kGmax halo row
// slot - kGmax, slot < 0 global row -(slot + 1).  Rows with more than 4
// dependencies use the other multi-RHS kernels.
//
// Synchronisation.  One CTA barrier per group; between CTAs a progress
// counter per CTA, prog[c] = (epoch << 32) | groups done, published with
// st.release after the barrier that ends a group.  A loader warp per CTA
// streams the records by TMA (3-deep ring), polls its producers' counters
// for the NEXT group (relaxed loads, one fence.acquire), then copies that
// group's halo rows by TMA -- all while the compute warps solve the current
// group.  Every dependency points to a lower level and all CTAs are
// co-resident (cooperative launch), so the lowest unfinished group can always
// proceed.  A per-launch watchdog turns a hung wait into SPTRSV_ERR_TIMEOUT
// (sptrsv_get_solve_status).
//
// Arithmetic per (row, column) = the sweep of P:176-187 in storage order:
// s = b(i); s = fma(-a_k, x(j_k), s); x(i) = s * (1/d(i)) (UNIT: s) -- the
// same sequence as every other multi-RHS kernel and SELF's thread-per-row
// rows, so a column's result is bitwise independent of nrhs and of the
// column block it is solved in (SURVEY §8e partition invariant).
#include <algorithm>
#include <vector>

#include <cuda.h>

#include "internal.h"

namespace sptrsv {
namespace {

constexpr int kGmax = 128;                         // rows per group
constexpr int kHmax = 32;                          // halo rows per group
constexpr int kCw = 16;                            // compute warps per CTA
// a release warp publishes the CTA's progress after each group barrier (the
// st.release waits ~1 us for the group's x stores to drain) while the loader
// warp already waits for the next group's producers and copies its halo
#ifndef SPTRSV_MRT_RELW
#define SPTRSV_MRT_RELW 1
#endif
constexpr int kRelw = SPTRSV_MRT_RELW;
// the b row loads (cache policy)
#ifndef SPTRSV_MRT_BLOAD
#define SPTRSV_MRT_BLOAD __ldcg      // measured: 1.656 ms vs 1.722 with __ldcs (evict-first)
#endif

// BSTAGE: the b rows of a group's first kBs positions come into shared memory
// by TMA tile::gather4 copies issued by the loader a group ahead (the compute
// warps copy them out at the group's start and free the buffer), the rest by
// loads one group ahead -- fewer rows through the per-SM load path
#ifndef SPTRSV_MRT_BSTAGE
#define SPTRSV_MRT_BSTAGE 3
#endif
constexpr int kBs = SPTRSV_MRT_BSTAGE ? 64 : 0;             // staged rows per group (per wave)
static_assert(kBs % 16 == 0 && kBs <= 128, "staged rows: whole rows of every compute warp");
// BSTAGE == 2: every b row staged, in two waves per group (positions 0..63,
// 64..127) through the one 64-row buffer, by a stager warp of its own: wave
// B of group k is issued when wave A was copied out, wave A of k + 1 when B was
constexpr bool kBw2 = SPTRSV_MRT_BSTAGE >= 2;
// XTMA (needs the release warp): a group's x rows leave shared memory by TMA
// tile::scatter4 stores issued by the release warp after the group barrier
// (instead of the compute warps' global stores); the progress release
// follows their completion
#ifndef SPTRSV_MRT_XTMA
#define SPTRSV_MRT_XTMA 1
#endif
constexpr bool kXtma = SPTRSV_MRT_XTMA && SPTRSV_MRT_RELW;
// HALO_G4 (with XTMA's x tensor map): halo rows by tile::gather4, 4 per op
#ifndef SPTRSV_MRT_HALO_G4
#define SPTRSV_MRT_HALO_G4 1
#endif
// BSTAGE == 3: waves of 32 rows through two 32-row halves of the buffer (two
// waves in flight: wave v + 2 is issued when wave v was copied out)
constexpr int kNbuf = SPTRSV_MRT_BSTAGE == 3 ? 2 : 1;      // buffer parts
constexpr int kWrows = kBs / kNbuf;                          // rows per wave
constexpr int kWr = kWrows / kCw;                            // rows per compute warp per wave
constexpr int kWaves = kGmax / kWrows;                       // waves per group (BSTAGE >= 2)
constexpr int kThreadsBar = (kCw + 1 + kRelw) * 32;         // the group barrier: compute, loader (, release) warps
constexpr int kThreadsMrt = kThreadsBar + (kBw2 ? 32 : 0);  // (+ the stager warp)
constexpr int kRpw = kGmax / kCw;                  // rows per compute warp per group
constexpr int kMaxDeps = 4;
constexpr int kCols = 64;                          // columns per launch (column blocks of <= 64)
template <typename T> __host__ __device__ constexpr int rec_bytes() { return sizeof(T) == 8 ? 80 : 64; }
// record: int32 row, nd, slot[4], pad[2] | T a[4], 1/d (| pad)

// shared memory: [out_0 | halo_1 | out_1 | halo_0] (rows of NC values), so
// that group k's previous outputs (out_{k+1 & 1}) and its halo (halo_{k & 1})
// are one contiguous region: slot s of group k is at region + s rows.
template <typename T, int CPL>
__host__ __device__ constexpr size_t mrt_smem() {
    return (size_t)2 * (kGmax + kHmax) * 32 * CPL * sizeof(T) + (size_t)3 * kGmax * rec_bytes<T>() + 9 * 8 + 16 +
           128 + (size_t)kBs * 32 * CPL * sizeof(T);
}

struct alignas(64) MrtArgs {
    CUtensorMap bmap;             // BSTAGE: b of this column block as a 2-D tensor {ncols (OOB: 0), n rows}
    CUtensorMap xmap;             // XTMA: x of this column block, the same shape (OOB columns not written)
    const int32_t *gc0;           // [K+1] first group of every CTA
    const int32_t *gstart;        // [ngroups+1] first solve position of every group
    const int32_t *wptr;          // [ngroups+1] wait list of every group
    const int2 *waits;            // {producer CTA, groups it must have done}
    const int32_t *hptr;          // [ngroups+1] halo list of every group
    const int32_t *hrow;          // halo rows
    const unsigned char *rec;     // records by solve position
    unsigned long long *prog;     // [K] (epoch << 32) | groups done
    unsigned *status;             // [0] epoch of the last launch whose wait timed out
    const void *b;
    void *x;
    int64_t ld;                   // row stride of b and x (elements)
    int ncols;                    // columns of this launch (<= 32 * CPL)
    unsigned epoch;
    unsigned long long timeout_ns;
    unsigned long long *trace;    // debug: per CTA [cap][2] %globaltimer {barrier k, group k+1 prepared}
    int trace_cap;
};

// The loader warp and the compute warps reach the group barrier at different
// instructions: the non-.aligned barrier.sync (bar.sync is .aligned, which
// requires every thread of the CTA at the same instruction -- synccheck);
// lanes reconverge first (the loader's lane-strided loops diverge)
__device__ __forceinline__ void bar_all() {
    __syncwarp();
    asm volatile("barrier.sync 1, %0;" ::"n"(kThreadsBar) : "memory");
}
__device__ __forceinline__ void bulk_g2s_u32(uint32_t dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void l2_prefetch_bulk(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <typename T, bool UNIT, int CPL>
__global__ void __launch_bounds__(kThreadsMrt, 1) k_mrt(const __grid_constant__ MrtArgs a) {
    extern __shared__ __align__(128) unsigned char sm[];
    constexpr int RB = rec_bytes<T>();
    constexpr int NC = 32 * CPL;
    constexpr uint32_t RS = NC * sizeof(T);                 // bytes per buffered row
    constexpr uint32_t OUT = kGmax * RS, HALO = kHmax * RS;
    // group k: region (= its previous outputs, then its halo), its output buffer, its halo buffer
    auto region = [&](int k) -> T * { return reinterpret_cast<T *>(sm + ((k & 1) ? 0u : OUT + HALO)); };
    auto out_of = [&](int k) -> T * { return reinterpret_cast<T *>(sm + ((k & 1) ? OUT + HALO : 0u)); };
    auto halo_of = [&](int k) -> uint32_t { return smem_u32(sm) + ((k & 1) ? OUT : 2 * OUT + HALO); };
    unsigned char *meta = sm + 2 * (OUT + HALO);                                   // [3][kGmax * RB]
    uint64_t *mbar = reinterpret_cast<uint64_t *>(meta + (size_t)3 * kGmax * RB);  // [3] records, [2] halos, bfull[2], bfree[2]
    int *nrow = reinterpret_cast<int *>(mbar + 9);                                  // [3] rows of the groups in the ring
    T *bst = reinterpret_cast<T *>(sm + ((2 * (OUT + HALO) + (size_t)3 * kGmax * RB + 9 * 8 + 16 + 127) & ~(size_t)127));
    uint64_t *bfull = &mbar[5], *bfree = &mbar[7];           // [kNbuf] each
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int c = blockIdx.x;
    const int g0 = a.gc0[c], ng = a.gc0[c + 1] - g0;
    const unsigned long long ep = (unsigned long long)a.epoch << 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 7; ++i) mbar_init(&mbar[i], 1);
        mbar_init(&mbar[7], kCw);
        mbar_init(&mbar[8], kCw);
        fence_mbar_init();
    }
    __syncthreads();
    const T *b = static_cast<const T *>(a.b);
    T *x = static_cast<T *>(a.x);
    const uint32_t rowbytes = (uint32_t)a.ncols * (uint32_t)sizeof(T);

    if (kBw2 && w == kCw + 1 + kRelw) {
        // ---- stager warp (BSTAGE >= 2): wave v = kWaves k + q holds positions kWrows q ..
        // kWrows (q + 1) - 1 of group k, in buffer part v % kNbuf
        auto stage = [&](int v) {
            const int k = v / kWaves, lo = (v % kWaves) * kWrows, slot = k % 3, pb = v % kNbuf;
            mbar_wait(&mbar[slot], (uint32_t)((k / 3) & 1));
            const int cnt = max(0, min(nrow[slot] - lo, kWrows)), nq = (cnt + 3) >> 2;
            const unsigned char *mt = meta + (size_t)slot * kGmax * RB;
            if (lane == 0) mbar_arrive_expect_tx(&bfull[pb], (uint32_t)nq * 4u * RS);
            __syncwarp();
            if (lane < nq) {
                int r[4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    r[i] = reinterpret_cast<const int32_t *>(mt + (size_t)(lo + min(4 * lane + i, cnt - 1)) * RB)[0];
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(bst) + (uint32_t)(pb * kWrows + 4 * lane) * RS),
                    "l"(reinterpret_cast<uint64_t>(&a.bmap)), "r"(smem_u32(&bfull[pb])), "r"(0), "r"(r[0]), "r"(r[1]),
                    "r"(r[2]), "r"(r[3])
                    : "memory");
            }
        };
        const int nw = kWaves * ng;
        for (int v = 0; v < min(kNbuf, nw); ++v) stage(v);
        for (int v = 0; v + kNbuf < nw; ++v) {
            mbar_wait(&bfree[v % kNbuf], (uint32_t)((v / kNbuf) & 1));   // wave v copied out by every compute warp
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            stage(v + kNbuf);
        }
        return;
    }
    if (kRelw && w == kCw + 1) {
        // ---- release warp: progress counter after every group barrier (XTMA: after the
        // group's x rows went out by scatter4 TMA stores from its output buffer)
        int rq[4] = {0, 0, 0, 0}, nr = 0;                  // XTMA: global rows of the group's positions 4 lane ..
        auto rows_of = [&](int k) {
            const int slot = k % 3;
            mbar_wait(&mbar[slot], (uint32_t)((k / 3) & 1));
            nr = nrow[slot];
            const unsigned char *mt = meta + (size_t)slot * kGmax * RB;
#pragma unroll
            for (int i = 0; i < 4; ++i)
                rq[i] = reinterpret_cast<const int32_t *>(mt + (size_t)min(4 * lane + i, max(nr - 1, 0)) * RB)[0];
        };
        for (int k = 0; k <= ng; ++k) {
            bar_all();
            if (kXtma && k > 0) {
                const int nfull = nr >> 2;                 // full quadruples by TMA; the tail by this warp
                const uint32_t src = smem_u32(out_of(k - 1)) + (uint32_t)(4 * lane) * RS;
                if (lane < nfull)
                    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile::scatter4.bulk_group"
                                 " [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(reinterpret_cast<uint64_t>(&a.xmap)),
                                 "r"(src), "r"(0), "r"(rq[0]), "r"(rq[1]), "r"(rq[2]), "r"(rq[3])
                                 : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                for (int p = 4 * nfull; p < nr; ++p) {     // <= 3 tail rows
                    const int row = __shfl_sync(0xffffffffu, rq[p & 3], nfull);
                    const T *sr = out_of(k - 1) + (size_t)p * NC;
                    T *xr = x + (int64_t)row * a.ld;
                    for (int j = lane; j < a.ncols; j += 32) xr[j] = sr[j];
                }
                asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
                asm volatile("fence.proxy.async.global;" ::: "memory");
            }
            // rows of the group now running, for its stores after the next barrier (its
            // record slot is reused once that barrier passes)
            if (kXtma && k < ng) rows_of(k);
            if (lane == 0 && k > 0) st_release_u64(a.prog + c, ep | (unsigned)k);
        }
        return;
    }
    if (w == kCw) {
        // ---- loader warp: records, producer waits, halo copies, progress releases
        auto issue_meta = [&](int k) {
            if (k < ng) {
                const int p0 = a.gstart[g0 + k], p1 = a.gstart[g0 + k + 1];
                const uint32_t bytes = (uint32_t)(p1 - p0) * RB;
                nrow[k % 3] = p1 - p0;                  // published by the arrive (release)
                mbar_arrive_expect_tx(&mbar[k % 3], bytes);
                bulk_g2s(meta + (size_t)(k % 3) * kGmax * RB, a.rec + (size_t)p0 * RB, bytes, &mbar[k % 3]);
            }
        };
        bool gave_up = false;
        unsigned long long *tr = a.trace != nullptr ? a.trace + (size_t)c * a.trace_cap * 2 : nullptr;
        // waits for group k's producers, then copies its halo rows by TMA (mbar[3 + (k & 1)])
        // a group's wait and halo lists, loaded one group ahead (lane e holds wait
        // entry e < 32 and halo row e < kHmax): their global-load latency stays
        // off the loader's chain
        struct Meta {
            int w0, w1, h0, nh, hr;
            int2 wt;
        };
        auto load_meta = [&](int k) -> Meta {
            Meta m{0, 0, 0, 0, 0, make_int2(0, 0)};
            if (k >= ng) return m;
            const int g = g0 + k;
            m.w0 = a.wptr[g];
            m.w1 = a.wptr[g + 1];
            m.h0 = a.hptr[g];
            m.nh = a.hptr[g + 1] - m.h0;
            if (m.w0 + lane < m.w1) m.wt = a.waits[m.w0 + lane];
            if (lane < m.nh) m.hr = a.hrow[m.h0 + lane];
            return m;
        };
        // waits for group k's producers, then copies its halo rows by TMA (mbar[3 + (k & 1)])
        auto prepare = [&](int k, const Meta &m) {
            if (k >= ng) return;
            if (!gave_up) {
                for (int e = m.w0 + lane; e < m.w1; e += 32) {
                    const int2 wt = e - m.w0 < 32 ? m.wt : a.waits[e];
                    const unsigned long long target = ep | (unsigned)wt.y;
                    unsigned it = 0;
                    unsigned long long t0 = 0;
                    while (ld_relaxed_u64(a.prog + wt.x) < target) {
                        if ((++it & 15u) == 0) {
                            if (it == 16u) t0 = gtime();
                            else if (gtime() - t0 > a.timeout_ns) {
                                st_relaxed(reinterpret_cast<int *>(a.status), (int)a.epoch);
                                gave_up = true;
                                break;
                            }
                        }
                    }
                    if (gave_up) break;
                }
                gave_up = __any_sync(0xffffffffu, gave_up);
            }
            // acquire: the producers' x rows are visible, then also to the async proxy
            // (the proxy fence only where TMA reads follow)
            const int nh = m.nh;
            if (nh > 0) asm volatile("fence.acquire.gpu;\n\tfence.proxy.async.global;" ::: "memory");
            else asm volatile("fence.acquire.gpu;" ::: "memory");
            uint64_t *hb = &mbar[3 + (k & 1)];
            const uint32_t hd = halo_of(k);
            if (SPTRSV_MRT_HALO_G4 && kXtma) {
                // 4 halo rows per tile::gather4 op on the x tensor map (the last quadruple
                // padded with its last row into unused slots; kHmax is a multiple of 4)
                const int nq = (nh + 3) >> 2;
                int r[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) r[i] = __shfl_sync(0xffffffffu, m.hr, max(0, min(4 * lane + i, nh - 1)) & 31);
                if (lane == 0) mbar_arrive_expect_tx(hb, (uint32_t)nq * 4u * RS);
                __syncwarp();
                if (lane < nq)
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(hd + (uint32_t)(4 * lane) * RS),
                        "l"(reinterpret_cast<uint64_t>(&a.xmap)), "r"(smem_u32(hb)), "r"(0), "r"(r[0]), "r"(r[1]),
                        "r"(r[2]), "r"(r[3])
                        : "memory");
            } else {
                if (lane == 0) mbar_arrive_expect_tx(hb, (uint32_t)nh * rowbytes);
                __syncwarp();
                if (lane < nh) bulk_g2s_u32(hd + (uint32_t)lane * RS, x + (int64_t)m.hr * a.ld, rowbytes, hb);
            }
        };
        // b rows of group k's first kBs positions into the staging buffer (4 rows per op)
        auto stage_b = [&](int k) {
            if (!kBs || k >= ng) return;
            const int slot = k % 3;
            mbar_wait(&mbar[slot], (uint32_t)((k / 3) & 1));
            const int nr = min(nrow[slot], kBs), nq = (nr + 3) >> 2;
            const unsigned char *mt = meta + (size_t)slot * kGmax * RB;
            if (lane == 0) mbar_arrive_expect_tx(bfull, (uint32_t)nq * 4u * RS);
            __syncwarp();
            if (lane < nq) {
                int r[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) r[i] = reinterpret_cast<const int32_t *>(mt + (size_t)min(4 * lane + i, nr - 1) * RB)[0];
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(bst) + (uint32_t)(4 * lane) * RS),
                    "l"(reinterpret_cast<uint64_t>(&a.bmap)), "r"(smem_u32(bfull)), "r"(0), "r"(r[0]), "r"(r[1]),
                    "r"(r[2]), "r"(r[3])
                    : "memory");
            }
        };
        if (lane == 0) {
            issue_meta(0);
            issue_meta(1);
        }
        if (!kBw2) stage_b(0);
        Meta mn = load_meta(1);
        prepare(0, load_meta(0));
        for (int k = 0; k <= ng; ++k) {
            bar_all();                          // barrier k: group k-1 done, group k's halo issued
            if (tr != nullptr && lane == 0 && k < a.trace_cap) tr[2 * k] = gtime();
            if (lane == 0) {
                if (!kRelw && k > 0) st_release_u64(a.prog + c, ep | (unsigned)k);
                issue_meta(k + 2);              // its ring slot held group k-1's records
            }
            if (kBs && !kBw2 && k + 1 < ng) {   // the compute warps copied group k's staged b out: stage k + 1
                mbar_wait(bfree, (uint32_t)(k & 1));
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // their reads before the TMA writes
                stage_b(k + 1);
            }
            prepare(k + 1, mn);                 // overlaps group k
            mn = load_meta(k + 2);
            if (tr != nullptr && lane == 0 && k < a.trace_cap) tr[2 * k + 1] = gtime();
        }
        return;
    }

    // ---- compute warps: rows w, w + kCw, ... of every group; lane = columns lane + 32 j
    T bcur[kRpw][CPL], bnxt[kRpw][CPL];
    auto load_b = [&](int k, T (&bb)[kRpw][CPL]) {
        const int slot = k % 3;
        mbar_wait(&mbar[slot], (uint32_t)((k / 3) & 1));
        const int nrows = nrow[slot];
        const unsigned char *mt = meta + (size_t)slot * kGmax * RB;
#pragma unroll
        for (int r = kBs / kCw; r < kRpw; ++r) {
            const int rr = w + r * kCw;
            const int row = rr < nrows ? reinterpret_cast<const int32_t *>(mt + (size_t)rr * RB)[0] : 0;
            const T *br = b + (int64_t)row * a.ld + lane;
#pragma unroll
            for (int j = 0; j < CPL; ++j)
                bb[r][j] = (rr < nrows && lane + 32 * j < a.ncols) ? SPTRSV_MRT_BLOAD(br + 32 * j) : T(0);
        }
    };
    // one group; bc holds its b rows, bn receives the next group's (the two
    // register sets alternate by group parity)
    auto group = [&](int k, T (&bc)[kRpw][CPL], T (&bn)[kRpw][CPL]) {
        bar_all();                                          // barrier k
        // staged b rows of wave v (rows r0 .. r0 + kBs / kCw - 1 of this warp), then free the buffer
        auto take_wave = [&](int v, int r0) {
            const int pb = kBw2 ? v % kNbuf : 0;
            const int ph = kBw2 ? (v / kNbuf) & 1 : v & 1;
            constexpr int WR = kBw2 ? kWr : kBs / kCw;
            mbar_wait(&bfull[pb], (uint32_t)ph);
#pragma unroll
            for (int r = 0; r < WR; ++r) {
                const T *sb = bst + (size_t)(pb * kWrows + w + r * kCw) * NC + lane;
#pragma unroll
                for (int j = 0; j < CPL; ++j) bc[r0 + r][j] = sb[32 * j];
            }
            __syncwarp();
            if (lane == 0)
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(kBw2 ? &bfree[pb] : bfree)) : "memory");
        };
        if (kBs) take_wave(kBw2 ? kWaves * k : k, 0);
        if (!kBw2 && k + 1 < ng) load_b(k + 1, bn);         // next group's b in flight during this one
        mbar_wait(&mbar[3 + (k & 1)], (uint32_t)((k >> 1) & 1));   // group k's halo rows
        const int nrows = nrow[k % 3];
        const unsigned char *mt = meta + (size_t)(k % 3) * kGmax * RB;
        const T *reg = region(k) + lane;
        T *outk = out_of(k) + lane;
#pragma unroll
        for (int r = 0; r < kRpw; ++r) {
            const int rr = w + r * kCw;
            if (kBw2 && r > 0 && r % kWr == 0) take_wave(kWaves * k + r / kWr, r);   // the group's next wave
            if (rr < nrows) {
                const unsigned char *rc = mt + (size_t)rr * RB;
                const int4 h0 = *reinterpret_cast<const int4 *>(rc);
                const int2 h1 = *reinterpret_cast<const int2 *>(rc + 16);
                const T *av = reinterpret_cast<const T *>(rc + 32);
                const int slot[kMaxDeps] = {h0.z, h0.w, h1.x, h1.y};
                T acc[CPL];
#pragma unroll
                for (int j = 0; j < CPL; ++j) acc[j] = bc[r][j];
#pragma unroll
                for (int d = 0; d < kMaxDeps; ++d)
                    if (d < h0.y) {
                        const T ad = av[d];
                        if (slot[d] >= 0) {
                            const T *p = reg + slot[d] * NC;
#pragma unroll
                            for (int j = 0; j < CPL; ++j) acc[j] = fnma(ad, p[32 * j], acc[j]);
                        } else {                    // beyond the halo capacity: global memory
                            const T *xr = x + (int64_t)(-slot[d] - 1) * a.ld + lane;
#pragma unroll
                            for (int j = 0; j < CPL; ++j)
                                acc[j] = fnma(ad, lane + 32 * j < a.ncols ? ld_cg(xr + 32 * j) : T(0), acc[j]);
                        }
                    }
                const T di = av[kMaxDeps];
                T *xo = x + (int64_t)h0.x * a.ld + lane;
                T *po = outk + rr * NC;
#pragma unroll
                for (int j = 0; j < CPL; ++j) {
                    const T xi = UNIT ? acc[j] : acc[j] * di;
                    po[32 * j] = xi;
                    if (!kXtma && lane + 32 * j < a.ncols) xo[32 * j] = xi;
                }
            }
        }
        // XTMA: this warp's output rows, written by the generic proxy, are read by the
        // release warp's TMA stores after the barrier
        if (kXtma) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    };
    if (ng > 0 && !kBw2) load_b(0, bcur);
    for (int k = 0; k < ng; k += 2) {
        group(k, bcur, bnxt);
        if (k + 1 < ng) group(k + 1, bnxt, bcur);
    }
    bar_all();                                              // barrier ng
}

// ---------------------------------------------------------------- build
__global__ void k_mrt_cta_grid(int n, int wpc, const int32_t *unit, int32_t *cta) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) cta[i] = unit[i] / wpc;
}
__global__ void k_mrt_cta_natural(int n, int K, int uplo, int32_t *cta) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int t = uplo == SPTRSV_LOWER ? i : n - 1 - i;
    cta[i] = (int)((int64_t)t * K / n);
}
__global__ void k_mrt_keys(int n, int nlev, const int32_t *cta, const int32_t *lev, uint32_t *keys) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) keys[i] = (uint32_t)cta[i] * (uint32_t)nlev + (uint32_t)lev[i];
}
// run heads (new (CTA, level)) and the inverse permutation
__global__ void k_mrt_heads(int n, const uint32_t *skeys, const int32_t *perm, int32_t *head, int32_t *pos) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p == n) head[p] = 0;
    if (p >= n) return;
    head[p] = (p == 0 || skeys[p - 1] != skeys[p]) ? 1 : 0;
    pos[perm[p]] = p;
}
__global__ void k_mrt_runstart(int n, const int32_t *head, const int32_t *rid, int32_t *rstart) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n && head[p]) rstart[rid[p]] = p;
}
// group heads: every kGmax-th position of a run
__global__ void k_mrt_gheads(int n, const int32_t *head, const int32_t *rid, const int32_t *rstart, int32_t *gh) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p == n) gh[p] = 0;
    if (p >= n) return;
    const int r = rid[p] + head[p] - 1;
    gh[p] = ((p - rstart[r]) % kGmax) == 0 ? 1 : 0;
}
__global__ void k_mrt_groups(int n, const int32_t *gh, const int32_t *gex, const int32_t *perm, const int32_t *cta,
                             int ng, int32_t *gstart, int32_t *gcta, int32_t *gid) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p == 0) gstart[ng] = n;
    if (p >= n) return;
    const int g = gex[p] + gh[p] - 1;
    gid[p] = g;
    if (gh[p]) {
        gstart[g] = p;
        gcta[g] = cta[perm[p]];
    }
}
// first item of every segment of a sorted segment-id list: ptr[s] for s in [0, ns]
__global__ void k_seg_ptr(int m, int ns, const int32_t *seg, int32_t *ptr) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o > m) return;
    const int s1 = o < m ? seg[o] : ns;
    const int s0 = o > 0 ? seg[o - 1] : -1;
    for (int q = s0 + 1; q <= s1; ++q) ptr[q] = o;
}
// records (previous-group slots; global dependencies marked -(row+1)) and,
// per position, the number of global dependencies and of cross-CTA ones
template <typename T>
__global__ void k_mrt_rec(int n, const int32_t *perm, const int32_t *pos, const int32_t *cta, const int32_t *gid,
                          const int32_t *gstart, const int32_t *tri_ptr, const int32_t *tri_col,
                          const T *tri_val, const T *invd_row, int unit_diag, unsigned char *rec, int32_t *gcnt,
                          int32_t *xcnt) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p == n) gcnt[p] = xcnt[p] = 0;
    if (p >= n) return;
    const int i = perm[p], ci = cta[i], gi = gid[p];
    int32_t hd[8] = {i, 0, 0, 0, 0, 0, 0, 0};
    T av[kMaxDeps + 1] = {T(0), T(0), T(0), T(0), unit_diag ? T(1) : invd_row[i]};
    int ng = 0, nx = 0, d = 0;
    for (int k = tri_ptr[i]; k < tri_ptr[i + 1] && d < kMaxDeps; ++k, ++d) {
        const int j = tri_col[k];
        const int pj = pos[j];
        int slot;
        if (cta[j] == ci && gid[pj] == gi - 1) {
            slot = pj - gstart[gi - 1];
        } else {
            slot = -(j + 1);
            ++ng;
            if (cta[j] != ci || kXtma) ++nx;      // XTMA: own older groups' rows land late too
        }
        hd[2 + d] = slot;
        av[d] = tri_val[k];
    }
    hd[1] = d;
    unsigned char *r = rec + (size_t)p * rec_bytes<T>();
    reinterpret_cast<int4 *>(r)[0] = make_int4(hd[0], hd[1], hd[2], hd[3]);
    reinterpret_cast<int4 *>(r)[1] = make_int4(hd[4], hd[5], 0, 0);
    T *ar = reinterpret_cast<T *>(r + 32);
    for (int q = 0; q <= kMaxDeps; ++q) ar[q] = av[q];
    gcnt[p] = ng;
    xcnt[p] = nx;
}
// global dependencies as (position, dep index) items keyed by their row, and
// cross-CTA ones as (group * K + producer CTA, groups needed)
__global__ void k_mrt_items(int n, int K, const int32_t *perm, const int32_t *pos, const int32_t *cta,
                            const int32_t *gid, const int32_t *gc0, const unsigned char *rec, int rb,
                            const int32_t *goff, const int32_t *xoff, uint32_t *hkey, int32_t *hitem,
                            uint32_t *wkey, int32_t *wneed) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int ci = cta[perm[p]];
    const int4 h0 = reinterpret_cast<const int4 *>(rec + (size_t)p * rb)[0];
    const int4 h1 = reinterpret_cast<const int4 *>(rec + (size_t)p * rb)[1];
    const int slot[kMaxDeps] = {h0.z, h0.w, h1.x, h1.y};
    int o = goff[p], q = xoff[p];
    for (int d = 0; d < h0.y; ++d) {
        if (slot[d] >= 0) continue;
        const int j = -slot[d] - 1, cj = cta[j];
        hkey[o] = (uint32_t)j;
        hitem[o] = p * kMaxDeps + d;
        ++o;
        if (cj != ci || kXtma) {         // XTMA: also wait for this CTA's own stores of older groups
            wkey[q] = (uint32_t)gid[p] * (uint32_t)K + (uint32_t)cj;
            wneed[q] = gid[pos[j]] - gc0[cj] + 1;
            ++q;
        }
    }
}
// stable second pass of the (group, row) sort: key = group of the item
__global__ void k_mrt_item_gkey(int m, const int32_t *hitem_sorted, const int32_t *gid, uint32_t *gkey) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o < m) gkey[o] = (uint32_t)gid[hitem_sorted[o] / kMaxDeps];
}
__global__ void k_gather_i32(int m, const int32_t *perm, const int32_t *in, int32_t *out) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o < m) out[o] = in[perm[o]];
}
__global__ void k_gather_u32(int m, const int32_t *perm, const uint32_t *in, uint32_t *out) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o < m) out[o] = in[perm[o]];
}
// unique (group, row) heads
__global__ void k_mrt_hheads(int m, const uint32_t *g, const uint32_t *j, int32_t *uh) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o == m) uh[o] = 0;
    if (o >= m) return;
    uh[o] = (o == 0 || g[o - 1] != g[o] || j[o - 1] != j[o]) ? 1 : 0;
}
// first unique item of every group (over the unique list)
__global__ void k_mrt_ufirst(int m, const uint32_t *g, const int32_t *uh, const int32_t *uex, int32_t *first) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= m || !uh[o]) return;
    if (o == 0 || g[o - 1] != g[o]) first[g[o]] = uex[o];
}
// halo rows and their groups; the record slot of every item within the capacity
__global__ void k_mrt_hfill(int m, const uint32_t *g, const uint32_t *j, const int32_t *items, const int32_t *uh,
                            const int32_t *uex, const int32_t *first, unsigned char *rec, int rb, int32_t *hrow,
                            int32_t *hgrp) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= m) return;
    const int u = uex[o] + uh[o] - 1;
    const int gg = (int)g[o];
    if (uh[o]) {
        hrow[u] = (int)j[o];
        hgrp[u] = gg;
    }
    const int rank = u - first[gg];          // halo slot within the group
    if (rank < kHmax) {
        const int p = items[o] / kMaxDeps, d = items[o] % kMaxDeps;
        reinterpret_cast<int32_t *>(rec + (size_t)p * rb)[2 + d] = kGmax + rank;
    }
}
// keep at most kHmax halo rows per group: compacted list
__global__ void k_mrt_hkeep(int nu, const int32_t *hgrp, const int32_t *first, int32_t *keep) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u == nu) keep[u] = 0;
    if (u < nu) keep[u] = (u - first[hgrp[u]]) < kHmax ? 1 : 0;
}
__global__ void k_mrt_hcompact(int nu, const int32_t *keep, const int32_t *kex, const int32_t *hrow, const int32_t *hgrp,
                               int32_t *hrow_out, int32_t *hgrp_out) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u < nu && keep[u]) {
        hrow_out[kex[u]] = hrow[u];
        hgrp_out[kex[u]] = hgrp[u];
    }
}
// unique (group, producer) with the maximum need (waits zero-filled before)
__global__ void k_mrt_wheads(int m, const uint32_t *skey, int32_t *uh) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o == m) uh[o] = 0;
    if (o < m) uh[o] = (o == 0 || skey[o - 1] != skey[o]) ? 1 : 0;
}
__global__ void k_mrt_wfill(int m, int K, const uint32_t *skey, const int32_t *sperm, const int32_t *wneed,
                            const int32_t *uh, const int32_t *uex, int2 *waits, int32_t *wgrp) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= m) return;
    const int u = uex[o] + uh[o] - 1;
    if (uh[o]) {
        waits[u].x = (int)(skey[o] % (uint32_t)K);
        wgrp[u] = (int)(skey[o] / (uint32_t)K);
    }
    atomicMax(&waits[u].y, wneed[sperm[o]]);
}

// new values into the records (NEXT-2 value update): slots kept, a[d] and 1/d re-read
template <typename T>
__global__ void k_mrt_refill(int n, unsigned char *rec, const int32_t *__restrict__ tri_ptr,
                             const T *__restrict__ tri_val, const T *__restrict__ invd_row, int unit_diag) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    unsigned char *r = rec + (size_t)p * rec_bytes<T>();
    const int4 h0 = reinterpret_cast<const int4 *>(r)[0];
    T *ar = reinterpret_cast<T *>(r + 32);
    for (int d = 0; d < h0.y; ++d) ar[d] = tri_val[tri_ptr[h0.x] + d];
    ar[kMaxDeps] = unit_diag ? T(1) : invd_row[h0.x];
}

int i32_read(const int32_t *d, int64_t i, cudaStream_t s, sptrsv_status_t &st) {
    int32_t v = 0;
    cudaError_t e = cudaMemcpyAsync(&v, d + i, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) st = cuda_fail(e, "mrt i32_read");
    return v;
}

template <typename T, bool UNIT, int CPL>
void *mrt_kernel() { return (void *)k_mrt<T, UNIT, CPL>; }

void *pick(int dtype, int diag, int cpl) {
    if (dtype == SPTRSV_F64)
        return diag == SPTRSV_UNIT ? (cpl == 1 ? mrt_kernel<double, true, 1>() : mrt_kernel<double, true, 2>())
                                   : (cpl == 1 ? mrt_kernel<double, false, 1>() : mrt_kernel<double, false, 2>());
    return diag == SPTRSV_UNIT ? (cpl == 1 ? mrt_kernel<float, true, 1>() : mrt_kernel<float, true, 2>())
                               : (cpl == 1 ? mrt_kernel<float, false, 1>() : mrt_kernel<float, false, 2>());
}
size_t smem_of(int dtype, int cpl) {
    if (dtype == SPTRSV_F64) return cpl == 1 ? mrt_smem<double, 1>() : mrt_smem<double, 2>();
    return cpl == 1 ? mrt_smem<float, 1>() : mrt_smem<float, 2>();
}

sptrsv_status_t mrt_build(sptrsv_handle_t h, cudaStream_t s) {
    ArenaStream as_{h->arena, s};     // the handle's allocations in this call: stream-ordered on s
    MrtPlan &M = h->mrt;
    const int n = h->n, nlev = h->info.nlev;
    DevArena tmp(s);
    struct Guard {
        DevArena &a;
        ~Guard() { a.release_all(); }
    } guard{tmp};
    sptrsv_status_t st;
    const int eg = (n + 1 + 255) / 256;
    auto grid_of = [](int64_t m) { return (int)((m + 1 + 255) / 256); };
    for (int cpl = 1; cpl <= 2; ++cpl)
        for (int diag = 0; diag <= 1; ++diag)
            SPTRSV_CUDA(cudaFuncSetAttribute(pick(h->dtype, diag, cpl), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem_of(h->dtype, cpl)));
    int per_sm = 0;
    SPTRSV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pick(h->dtype, h->diag, 2), kThreadsMrt,
                                                              smem_of(h->dtype, 2)));
    if (per_sm < 1) return SPTRSV_ERR_NOT_SUPPORTED;
    // 1. partition: the BLOCK tile partition on detected grids, else natural blocks
    int32_t *cta = nullptr;
    if ((st = tmp.alloc_n(&cta, (size_t)n)) != SPTRSV_SUCCESS) return st;
    int K;
    if (h->block.built && h->block.grid_nx > 0 && h->block.nblocks <= per_sm * h->num_sms) {
        K = h->block.nblocks;
        k_mrt_cta_grid<<<eg, 256, 0, s>>>(n, h->block.wpc, h->block.d_unit, cta);
    } else {
        K = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)h->num_sms * per_sm, (n + 4095) / 4096));
        k_mrt_cta_natural<<<eg, 256, 0, s>>>(n, K, h->uplo, cta);
    }
    SPTRSV_CUDA(cudaGetLastError());
    if ((uint64_t)K * (uint64_t)std::max(nlev, 1) >= (1ull << 32)) return SPTRSV_ERR_NOT_SUPPORTED;
    // 2. order by (CTA, level, row); runs of (CTA, level) cut into groups of <= kGmax
    int32_t *tri_ptr = nullptr, *tri_col = nullptr;
    void *tri_val = nullptr;
    if ((st = build_tri_csr(h, tmp, s, &tri_ptr, &tri_col, &tri_val)) != SPTRSV_SUCCESS) return st;
    uint32_t *keys = nullptr, *skeys = nullptr;
    int32_t *perm = nullptr, *pos = nullptr, *head = nullptr, *rid = nullptr, *rstart = nullptr, *gh = nullptr,
            *gex = nullptr, *gid = nullptr;
    if ((st = tmp.alloc_n(&keys, (size_t)n)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&skeys, (size_t)n)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&perm, (size_t)n)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&pos, (size_t)n)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&head, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&rid, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&rstart, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&gh, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&gex, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&gid, (size_t)n)) != SPTRSV_SUCCESS) return st;
    k_mrt_keys<<<eg, 256, 0, s>>>(n, nlev, cta, h->d_lev, keys);
    if ((st = radix_sort_pairs(keys, nullptr, skeys, perm, n, (uint32_t)((uint64_t)K * nlev - 1), tmp, s)) !=
        SPTRSV_SUCCESS)
        return st;
    k_mrt_heads<<<eg, 256, 0, s>>>(n, skeys, perm, head, pos);
    if ((st = exclusive_scan_i32(head, rid, (int64_t)n + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    k_mrt_runstart<<<eg, 256, 0, s>>>(n, head, rid, rstart);
    k_mrt_gheads<<<eg, 256, 0, s>>>(n, head, rid, rstart, gh);
    if ((st = exclusive_scan_i32(gh, gex, (int64_t)n + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    const int ng = i32_read(gex, n, s, st);
    if (st != SPTRSV_SUCCESS) return st;
    if ((uint64_t)ng * (uint64_t)K >= (1ull << 32)) return SPTRSV_ERR_NOT_SUPPORTED;
    int32_t *gcta = nullptr;
    if ((st = tmp.alloc_n(&gcta, (size_t)ng + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&M.d_gstart, (size_t)ng + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&M.d_gc0, (size_t)K + 1)) != SPTRSV_SUCCESS) return st;
    k_mrt_groups<<<eg, 256, 0, s>>>(n, gh, gex, perm, cta, ng, M.d_gstart, gcta, gid);
    k_seg_ptr<<<grid_of(ng), 256, 0, s>>>(ng, K, gcta, M.d_gc0);
    // 3. records; counts of global and cross-CTA dependencies per position
    const int RB = h->dtype == SPTRSV_F64 ? rec_bytes<double>() : rec_bytes<float>();
    int32_t *gcnt = nullptr, *goff = nullptr, *xcnt = nullptr, *xoff = nullptr;
    if ((st = tmp.alloc_n(&gcnt, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&goff, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&xcnt, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&xoff, (size_t)n + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc(reinterpret_cast<void **>(&M.d_rec), (size_t)n * RB)) != SPTRSV_SUCCESS) return st;
    if (h->dtype == SPTRSV_F64)
        k_mrt_rec<double><<<eg, 256, 0, s>>>(n, perm, pos, cta, gid, M.d_gstart, tri_ptr, tri_col,
                                             (const double *)tri_val, (const double *)h->d_invd_row,
                                             h->diag == SPTRSV_UNIT, M.d_rec, gcnt, xcnt);
    else
        k_mrt_rec<float><<<eg, 256, 0, s>>>(n, perm, pos, cta, gid, M.d_gstart, tri_ptr, tri_col,
                                            (const float *)tri_val, (const float *)h->d_invd_row,
                                            h->diag == SPTRSV_UNIT, M.d_rec, gcnt, xcnt);
    SPTRSV_CUDA(cudaGetLastError());
    if ((st = exclusive_scan_i32(gcnt, goff, (int64_t)n + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    if ((st = exclusive_scan_i32(xcnt, xoff, (int64_t)n + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
    const int mh = i32_read(goff, n, s, st);
    if (st != SPTRSV_SUCCESS) return st;
    const int mx = i32_read(xoff, n, s, st);
    if (st != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&M.d_hptr, (size_t)ng + 1)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&M.d_wptr, (size_t)ng + 1)) != SPTRSV_SUCCESS) return st;
    // 4. global dependencies: items sorted by (group, row), unique halo rows per group
    uint32_t *hkey = nullptr, *wkey = nullptr;
    int32_t *hitem = nullptr, *wneed = nullptr;
    if ((st = tmp.alloc_n(&hkey, (size_t)std::max(mh, 1))) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&hitem, (size_t)std::max(mh, 1))) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&wkey, (size_t)std::max(mx, 1))) != SPTRSV_SUCCESS) return st;
    if ((st = tmp.alloc_n(&wneed, (size_t)std::max(mx, 1))) != SPTRSV_SUCCESS) return st;
    k_mrt_items<<<eg, 256, 0, s>>>(n, K, perm, pos, cta, gid, M.d_gc0, M.d_rec, RB, goff, xoff, hkey, hitem, wkey,
                                   wneed);
    SPTRSV_CUDA(cudaGetLastError());
    int nh = 0;
    if (mh > 0) {
        uint32_t *sj = nullptr, *gk = nullptr, *sg = nullptr, *sj2 = nullptr;
        int32_t *p1 = nullptr, *it1 = nullptr, *p2 = nullptr, *it2 = nullptr, *uh = nullptr, *uex = nullptr,
                *first = nullptr, *hrow = nullptr, *hgrp = nullptr, *keep = nullptr, *kex = nullptr;
        const size_t mm = (size_t)mh + 1;
        for (int32_t **pp : {&p1, &it1, &p2, &it2, &uh, &uex, &hrow, &hgrp, &keep, &kex})
            if ((st = tmp.alloc_n(pp, mm)) != SPTRSV_SUCCESS) return st;
        for (uint32_t **pp : {&sj, &gk, &sg, &sj2})
            if ((st = tmp.alloc_n(pp, mm)) != SPTRSV_SUCCESS) return st;
        if ((st = tmp.alloc_n(&first, (size_t)ng + 1)) != SPTRSV_SUCCESS) return st;
        // LSD: by row, then (stable) by group
        if ((st = radix_sort_pairs(hkey, nullptr, sj, p1, mh, (uint32_t)(n - 1), tmp, s)) != SPTRSV_SUCCESS) return st;
        k_gather_i32<<<grid_of(mh), 256, 0, s>>>(mh, p1, hitem, it1);
        k_mrt_item_gkey<<<grid_of(mh), 256, 0, s>>>(mh, it1, gid, gk);
        if ((st = radix_sort_pairs(gk, nullptr, sg, p2, mh, (uint32_t)std::max(ng - 1, 0), tmp, s)) != SPTRSV_SUCCESS)
            return st;
        k_gather_i32<<<grid_of(mh), 256, 0, s>>>(mh, p2, it1, it2);
        k_gather_u32<<<grid_of(mh), 256, 0, s>>>(mh, p2, sj, sj2);
        k_mrt_hheads<<<grid_of(mh), 256, 0, s>>>(mh, sg, sj2, uh);
        if ((st = exclusive_scan_i32(uh, uex, (int64_t)mh + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
        const int nu = i32_read(uex, mh, s, st);
        if (st != SPTRSV_SUCCESS) return st;
        k_mrt_ufirst<<<grid_of(mh), 256, 0, s>>>(mh, sg, uh, uex, first);
        k_mrt_hfill<<<grid_of(mh), 256, 0, s>>>(mh, sg, sj2, it2, uh, uex, first, M.d_rec, RB, hrow, hgrp);
        k_mrt_hkeep<<<grid_of(nu), 256, 0, s>>>(nu, hgrp, first, keep);
        if ((st = exclusive_scan_i32(keep, kex, (int64_t)nu + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
        nh = i32_read(kex, nu, s, st);
        if (st != SPTRSV_SUCCESS) return st;
        int32_t *hg2 = nullptr;
        if ((st = tmp.alloc_n(&hg2, (size_t)std::max(nh, 1))) != SPTRSV_SUCCESS) return st;
        if ((st = h->arena.alloc_n(&M.d_hrow, (size_t)std::max(nh, 1))) != SPTRSV_SUCCESS) return st;
        k_mrt_hcompact<<<grid_of(nu), 256, 0, s>>>(nu, keep, kex, hrow, hgrp, M.d_hrow, hg2);
        k_seg_ptr<<<grid_of(nh), 256, 0, s>>>(nh, ng, hg2, M.d_hptr);
    } else {
        if ((st = h->arena.alloc_n(&M.d_hrow, 1)) != SPTRSV_SUCCESS) return st;
        SPTRSV_CUDA(cudaMemsetAsync(M.d_hptr, 0, sizeof(int32_t) * ((size_t)ng + 1), s));
    }
    // 5. wait lists: max groups needed per (group, producer CTA)
    int nu = 0;
    if (mx > 0) {
        uint32_t *skey = nullptr;
        int32_t *sperm = nullptr, *uh = nullptr, *uex = nullptr, *wgrp = nullptr;
        if ((st = tmp.alloc_n(&skey, (size_t)mx)) != SPTRSV_SUCCESS) return st;
        if ((st = tmp.alloc_n(&sperm, (size_t)mx)) != SPTRSV_SUCCESS) return st;
        if ((st = tmp.alloc_n(&uh, (size_t)mx + 1)) != SPTRSV_SUCCESS) return st;
        if ((st = tmp.alloc_n(&uex, (size_t)mx + 1)) != SPTRSV_SUCCESS) return st;
        if ((st = tmp.alloc_n(&wgrp, (size_t)mx + 1)) != SPTRSV_SUCCESS) return st;
        if ((st = radix_sort_pairs(wkey, nullptr, skey, sperm, mx, (uint32_t)((uint64_t)ng * K - 1), tmp, s)) !=
            SPTRSV_SUCCESS)
            return st;
        k_mrt_wheads<<<grid_of(mx), 256, 0, s>>>(mx, skey, uh);
        if ((st = exclusive_scan_i32(uh, uex, (int64_t)mx + 1, tmp, s)) != SPTRSV_SUCCESS) return st;
        nu = i32_read(uex, mx, s, st);
        if (st != SPTRSV_SUCCESS) return st;
        if ((st = h->arena.alloc_n(&M.d_waits, (size_t)nu)) != SPTRSV_SUCCESS) return st;
        SPTRSV_CUDA(cudaMemsetAsync(M.d_waits, 0, sizeof(int2) * (size_t)nu, s));
        k_mrt_wfill<<<grid_of(mx), 256, 0, s>>>(mx, K, skey, sperm, wneed, uh, uex, M.d_waits, wgrp);
        k_seg_ptr<<<grid_of(nu), 256, 0, s>>>(nu, ng, wgrp, M.d_wptr);
    } else {
        if ((st = h->arena.alloc_n(&M.d_waits, 1)) != SPTRSV_SUCCESS) return st;
        SPTRSV_CUDA(cudaMemsetAsync(M.d_wptr, 0, sizeof(int32_t) * ((size_t)ng + 1), s));
    }
    if ((st = h->arena.alloc_n(&M.d_prog, (size_t)K)) != SPTRSV_SUCCESS) return st;
    if ((st = h->arena.alloc_n(&M.d_status, 4)) != SPTRSV_SUCCESS) return st;
    SPTRSV_CUDA(cudaMemsetAsync(M.d_prog, 0, sizeof(unsigned long long) * (size_t)K, s));
    SPTRSV_CUDA(cudaMemsetAsync(M.d_status, 0, 4 * sizeof(unsigned), s));
    SPTRSV_CUDA(cudaGetLastError());
    SPTRSV_CUDA(cudaStreamSynchronize(s));
    M.K = K;
    M.ngroups = ng;
    M.nwaits = nu;
    M.nhalo = nh;
    M.built = true;
    h->info.device_bytes = h->arena.bytes + (int64_t)h->stage_bytes;
    return SPTRSV_SUCCESS;
}

}  // namespace

// Eligible: every row has <= 4 referenced dependencies (5-/7-point factors;
// the others use the level-scheduled or value-as-flag multi-RHS kernels),
// and b, x and the row stride are 16-byte aligned (the halo rows are TMA bulk
// copies of x row segments; column blocks start at multiples of 64 values).
bool mrt_eligible(sptrsv_handle_t h, const void *b, const void *x, int32_t nrhs) {
    auto al = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
    return h->n > 0 && !h->mrt.failed && h->info.max_row_deps <= kMaxDeps && al(b) && al(x) &&
           ((size_t)nrhs * h->esize) % 16 == 0;
}

// b of one column block as a 2-D tensor map for the staged rows: {nc columns,
// n rows}, row stride ld elements, box {32 cpl columns, 1 row} (columns past
// nc read as zero)
using EncodeTiled = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                 const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
sptrsv_status_t encode_bmap(CUtensorMap *m, const void *bp, int n, int nc, int cpl, int64_t ld, size_t es) {
    static EncodeTiled fn = nullptr;
    if (fn == nullptr) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || p == nullptr)
            return SPTRSV_ERR_CUDA;
        fn = reinterpret_cast<EncodeTiled>(p);
    }
    const cuuint64_t dims[2] = {(cuuint64_t)nc, (cuuint64_t)n};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * es};
    const cuuint32_t box[2] = {(cuuint32_t)(32 * cpl), 1u};
    const cuuint32_t estr[2] = {1u, 1u};
    const CUresult r = fn(m, es == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                          const_cast<void *>(bp), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? SPTRSV_SUCCESS : SPTRSV_ERR_CUDA;
}

sptrsv_status_t mrt_solve(sptrsv_handle_t h, const void *b, void *x, int32_t nrhs, cudaStream_t s) {
    MrtPlan &M = h->mrt;
    if (!M.built) {
        sptrsv_status_t st = mrt_build(h, s);
        if (st != SPTRSV_SUCCESS) {
            M.failed = true;
            return st;
        }
    }
    const size_t es = h->esize;
    M.solve_first = M.epoch + 1;
    for (int c0 = 0; c0 < nrhs; c0 += kCols) {
        const int nc = std::min(kCols, nrhs - c0);
        const int cpl = nc <= 32 ? 1 : 2;
        MrtArgs a;
        a.gc0 = M.d_gc0;
        a.gstart = M.d_gstart;
        a.wptr = M.d_wptr;
        a.waits = M.d_waits;
        a.hptr = M.d_hptr;
        a.hrow = M.d_hrow;
        a.rec = M.d_rec;
        a.prog = M.d_prog;
        a.status = M.d_status;
        a.b = static_cast<const char *>(b) + (size_t)c0 * es;
        a.x = static_cast<char *>(x) + (size_t)c0 * es;
        a.ld = nrhs;
        a.ncols = nc;
        if (kBs) {
            sptrsv_status_t st = encode_bmap(&a.bmap, a.b, h->n, nc, cpl, nrhs, es);
            if (st != SPTRSV_SUCCESS) return st;
        }
        if (kXtma) {
            sptrsv_status_t st = encode_bmap(&a.xmap, a.x, h->n, nc, cpl, nrhs, es);
            if (st != SPTRSV_SUCCESS) return st;
        }
        a.epoch = ++M.epoch;
        a.timeout_ns = h->timeout_ns;
        a.trace = static_cast<unsigned long long *>(M.trace);
        a.trace_cap = M.trace_cap;
        void *args[] = {(void *)&a};
        SPTRSV_CUDA(cudaLaunchCooperativeKernel(pick(h->dtype, h->diag, cpl), M.K, kThreadsMrt, args,
                                                smem_of(h->dtype, cpl), s));
    }
    h->last_solve = 2;
    return SPTRSV_SUCCESS;
}

sptrsv_status_t mrt_refresh_values(sptrsv_handle_t h, const int32_t *tri_ptr, const void *tri_val, cudaStream_t s) {
    const MrtPlan &M = h->mrt;
    const int g = (h->n + 255) / 256;
    if (h->dtype == SPTRSV_F64)
        k_mrt_refill<double><<<g, 256, 0, s>>>(h->n, M.d_rec, tri_ptr, (const double *)tri_val,
                                               (const double *)h->d_invd_row, h->diag == SPTRSV_UNIT);
    else
        k_mrt_refill<float><<<g, 256, 0, s>>>(h->n, M.d_rec, tri_ptr, (const float *)tri_val,
                                              (const float *)h->d_invd_row, h->diag == SPTRSV_UNIT);
    SPTRSV_CUDA(cudaGetLastError());
    return SPTRSV_SUCCESS;
}

// TIMEOUT iff a wait of the last multi-RHS tile solve gave up (the status word
// holds the epoch of the last launch that did; a solve's launches have epochs
// solve_first .. epoch).
sptrsv_status_t mrt_solve_status(sptrsv_handle_t h) {
    const MrtPlan &M = h->mrt;
    if (!M.built) return SPTRSV_SUCCESS;
    unsigned v = 0;
    SPTRSV_CUDA(cudaMemcpy(&v, M.d_status, sizeof(unsigned), cudaMemcpyDeviceToHost));
    return (v != 0 && v >= M.solve_first) ? SPTRSV_ERR_TIMEOUT : SPTRSV_SUCCESS;
}

}  // namespace sptrsv
