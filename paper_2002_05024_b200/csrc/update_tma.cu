// update_tma.cu -- the off-diagonal window updates (window_tasks.cpp:12-30,
// 72-86) with bulk-copy (TMA engine) fed panels and register-resident Q_w
// fragments.
//
// Same contract as update_dmma.cu (one launch = one wavefront, tiles located
// through the WinDesc prefix sums, in-place output tiles) and the same
// per-element arithmetic (k ascending in m8n8k4 groups of four, so the two
// paths agree bit for bit), different data movement:
//  * Q_w never goes through shared memory: each warp holds its 16-row (left:
//    Q_w^T) or 16-column (right: Q_w) slice for the whole K = 128 extent as
//    m8n8k4 fragments in registers (64 doubles per lane), reloaded only when
//    the CTA's tile range crosses into the next window;
//  * the panel streams through a 3-stage shared-memory ring.  Every panel
//    column segment is one cp.async.bulk (SASS UBLKCP: the TMA engine's 1-D
//    copy) completing on the stage's mbarrier; right after the block barrier
//    that ends a sub-tile, one thread per panel column (32 left, 128 right)
//    refills the freed stage with the sub-tile a ring depth ahead (one arrival
//    per producing warp carrying its bytes), so the copies of the next
//    sub-tiles overlap the DMMAs of the current one (a single producer lane
//    or warp measured 5-40 % slower: its copies serialise);
//  * persistent grid (one CTA per SM, grid_for): each CTA walks one
//    contiguous range of planner tiles
//    (one or two windows as a rule), so the fragment loads and the pipeline
//    fill are amortised and there is no partial last wave.
// Shared-memory column strides are 4 (left, B fragments) and 8 (right, A
// fragments) mod 16 doubles: both fragment loads take the minimum two
// wavefronts.  Bulk copies need 16-byte aligned sources: a column segment
// starts one row early when its first element is odd (the fragment index
// carries the shift; with an even leading dimension it is the same for all
// columns of a sub-tile); a segment whose rounded end would pass the end of
// the matrix allocation stops one pair short and the issuing lane stores its
// last element itself before the stage's arrive.
//
// (2-D tensor-map TMA, cp.async.bulk.tensor, was the first choice: on this
// pool's B200 nodes every tensor-map load -- CUTLASS's own SM90_TMA_LOAD_2D on
// a cuTensorMapEncodeTiled descriptor included -- faults with an illegal
// instruction while 1-D bulk copies work; tools/microbench/tma_min.cu.)
//
// Used for windows of order <= 128 on a matrix whose leading dimension is
// even and whose base is 16-byte aligned (other calls take update_dmma.cu),
// in two instantiations: order 65..128 (one CTA of 8 warps per SM, 255
// registers: 64 Q_w fragments per lane) and order <= 64 (the generalized
// reorder's windows, C5: half the fragments and rows, two CTAs per SM so one
// CTA's barriers and refills overlap the other's DMMAs; TEIG_NO_BULK64=1
// sends these windows to the cp.async kernels).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "device_types.h"
#include "launch.h"

namespace teig {

// DMMA instructions issued by the bulk update kernels (zero fragments skipped
// are not counted; every warp adds once, at its end)
__device__ unsigned long long g_dmma_bulk = 0;

namespace {

constexpr int kWarps = 8;
constexpr int kBulkThreads = kWarps * 32;  // 2 warps per SMSP: up to 255 registers each
constexpr int kMinTilesPerCta = 4;  // below this the launch gets more, shorter CTAs
#ifndef TEIG_LSUB
#define TEIG_LSUB 64
#endif
constexpr int kLSub = TEIG_LSUB;                // left: columns per sub-tile
constexpr int kRSub = 64;        // right: rows per sub-tile (the whole planner tile)
constexpr int kLdA = 72;         // right: doubles per panel column in smem (<= kRSub+1 rows used, = 8 mod 16)

// Window-order class DW = 128 (windows of order 65..128; the order <= 64
// class has its own kernels below).  Left: warps tile the DW output rows in
// 16-row slices (DW / 16 of them) and split the sub-tile's columns among the
// rest; right: DW / 16 slices of 16 output columns, the sub-tile's rows split
// among the rest.  Q_w fragments in registers: 2 x DW / 4 per lane.
template <int DW>
struct LeftCfg {
    static constexpr int kLd = DW == 128 ? 132 : 68;  // doubles per panel column in smem (<= DW+1 used, = 4 mod 16)
    static constexpr int kStages = kLSub == 64 ? 3 : 4;
    static constexpr int kStage = kLSub * kLd * 8;    // bytes: kLSub columns x DW(+1) rows
    static constexpr int kMGroups = DW / 16;          // warps along the rows
    static constexpr int kNSplit = kWarps / kMGroups; // warps along the sub-tile's columns
    static constexpr int kNT = kLSub / 8 / kNSplit;   // 8-column tiles per warp
    static constexpr int kKS = DW / 4;                // k-steps of 4
    static constexpr size_t kSmem = (size_t)kStages * kStage;
};
template <int DW>
struct RightCfg {
    static constexpr int kStages = 3;
    static constexpr int kStage = DW * kLdA * 8;      // bytes: DW columns x kRSub(+1) rows
    static constexpr int kNGroups = DW / 16;          // warps along the output columns
    static constexpr int kMSplit = kWarps / kNGroups; // warps along the sub-tile's rows
    static constexpr int kMT = kRSub / 8 / kMSplit;   // 8-row tiles per warp
    static constexpr int kKS = DW / 4;
    static constexpr size_t kSmem = (size_t)kStages * kStage;
};

// The order <= 64 kernels (the generalized reorder's windows, C5): each warp
// owns ONE 8-row (left) / 8-column (right) fragment tile over the whole
// sub-tile, so the 16 Q_w fragments per lane and the accumulators fit 128
// registers without spills at two CTAs per SM (the order-128 kernels'
// 16-row slices on half the warps spilled there: C5 1.47 -> 1.23 s).  Kept
// apart from the order-128 kernels, whose register allocation is tuned.
struct Left64Cfg {
    static constexpr int kLd = 68;                    // doubles per panel column in smem (<= 65 used, = 4 mod 16)
    static constexpr int kStages = kLSub == 64 ? 3 : 4;
    static constexpr int kStage = kLSub * kLd * 8;
    static constexpr int kFT = 1;
    static constexpr int kMGroups = 8;                // warps along the rows (8 rows each)
    static constexpr int kNSplit = 1;
    static constexpr int kNT = kLSub / 8;
    static constexpr int kKS = 16;
    static constexpr size_t kSmem = (size_t)kStages * kStage;
};
struct Right64Cfg {
    static constexpr int kStages = 3;
    static constexpr int kStage = 64 * kLdA * 8;
    static constexpr int kFT = 1;
    static constexpr int kNGroups = 8;                // warps along the columns (8 columns each)
    static constexpr int kMSplit = 1;
    static constexpr int kMT = kRSub / 8;
    static constexpr int kKS = 16;
    static constexpr size_t kSmem = (size_t)kStages * kStage;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1-D bulk copy global -> shared (16-byte aligned, multiple of 16 bytes)
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// 1-D bulk copy shared -> global (bulk-group completion)
__device__ __forceinline__ void bulk_store(void* gdst, const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(
                     reinterpret_cast<uint64_t>(gdst)),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

// one output column segment: global g[0..len) <- sm[0..len) (sm = the stage
// column + the segment's shift).  The 16-byte aligned interior goes as one
// bulk store; an odd first / last element is stored by the thread itself (a
// padded bulk store would overwrite a neighbour's element).
__device__ __forceinline__ void store_column(double* g, const double* sm, int shift, int len) {
    int j0 = 0;
    if (shift && len > 0) {
        g[0] = sm[0];
        j0 = 1;
    }
    const int cnt = len - j0, nb = cnt & ~1;
    if (nb > 0) bulk_store(g + j0, sm + j0, (unsigned)nb * 8u);
    if (cnt & 1) g[len - 1] = sm[len - 1];
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

template <int Field>
__device__ __forceinline__ int pref_of(const WinDesc& w) {
    return Field == 0 ? w.tl_pref : (Field == 1 ? w.tr_pref : w.tq_pref);
}
// largest k with pref[k] <= t (serial binary search, once per CTA)
template <int Field>
__device__ __forceinline__ int window_of(const WinDesc* wins, int nwin, int t) {
    int lo = 0, hi = nwin - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (pref_of<Field>(wins[mid]) <= t) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// the fields of the window owning the current tile, held in registers; the
// next window's prefix decides when to move on (one global round trip per
// window instead of several per tile)
struct TileWin {
    int wi, a, d, pref, r0, r1, next_pref;
    long long qw_off;
};
template <int Field>
__device__ __forceinline__ void load_win(TileWin& tw, const WinDesc* wins, int nwin, int wi) {
    const WinDesc& w = wins[wi];
    tw.wi = wi;
    tw.a = w.a;
    tw.d = w.d;
    tw.pref = pref_of<Field>(w);
    tw.r0 = Field == 0 ? w.lc0 : (Field == 1 ? w.rr0 : w.qr0);
    tw.r1 = Field == 0 ? w.lc1 : (Field == 1 ? w.rr1 : w.qr1);
    tw.qw_off = w.qw_off;
    tw.next_pref = (wi + 1 < nwin) ? pref_of<Field>(wins[wi + 1]) : 0x7fffffff;
}
template <int Field>
__device__ __forceinline__ void seek_win(TileWin& tw, const WinDesc* wins, int nwin, int t) {
    while (t >= tw.next_pref) load_win<Field>(tw, wins, nwin, tw.wi + 1);
}

// one arrival per producing warp carrying the warp's bytes (after the lanes'
// edge stores; 128 single-thread arrivals on one mbarrier serialise)
__device__ __forceinline__ void warp_arrive(uint64_t* bar, unsigned my_bytes) {
    const unsigned total = __reduce_add_sync(0xffffffffu, my_bytes);
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_expect_tx(bar, total);
}

// the copy of one column segment: `len` elements from element offset `off`
// of `base` into dst, as a 16-byte aligned bulk copy starting at off - shift.
// Returns the bulk doubles to copy (the edge element, if any, is stored here).
__device__ __forceinline__ int plan_segment(double* dst, const double* base, long long off, int len,
                                            long long alloc, long long& start) {
    const int shift = (int)(off & 1);
    start = off - shift;
    int n = (len + shift + 1) & ~1;
    if (start + n > alloc) {  // only the allocation's last column can get here
        n -= 2;
        const int tail = len + shift - 1;
        if (tail >= n) dst[tail] = base[start + tail];
    }
    return n > 0 ? n : 0;
}

// barriers + a zeroed ring (stale stage contents are then always finite
// matrix values, so rows/columns beyond a window's order only ever meet zero
// fragments)
__device__ __forceinline__ void init_ring(uint64_t* full, int nstages, double* ring, int bytes, unsigned full_count) {
    for (int i = threadIdx.x; i < bytes / 8; i += kBulkThreads) ring[i] = 0.0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nstages; ++s) mbar_init(&full[s], full_count);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // the zeroes before any bulk write
    __syncthreads();
}

}  // namespace

// ---------------------------------------------------------------------------
// LEFT: S[a:a+d, c:c+64] <- Q_w^T S[a:a+d, c:c+64], in kLSub-column
// sub-tiles; warp w owns output rows [16 wm, 16 wm + 16) (wm = w mod DW/16)
// of the sub-tile's column slice w / (DW/16).
template <int DW>
__global__ void __launch_bounds__(kBulkThreads, DW == 64 ? 2 : 1)
update_left_bulk_kernel(const WinDesc* __restrict__ wins, int nwin, int ntiles, const double* __restrict__ qw_pool,
                        double* __restrict__ S, long long lds, long long alloc) {
    using C = LeftCfg<DW>;
    constexpr int kLdB = C::kLd, kLeftStage = C::kStage, kLStages = C::kStages, kNT = C::kNT, kKS = C::kKS;
    extern __shared__ __align__(128) double ring[];
    __shared__ __align__(8) uint64_t full[kLStages];
    init_ring(full, kLStages, ring, kLStages * kLeftStage, kLSub / 32);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm = warp % C::kMGroups, wn = warp / C::kMGroups;
    const int t0 = (int)((long long)ntiles * blockIdx.x / gridDim.x);
    const int t1 = (int)((long long)ntiles * (blockIdx.x + 1) / gridDim.x);

    // every thread walks the (tile, sub-tile) sequence a ring depth ahead of the
    // one it computes; thread j < kLSub copies panel column j of each refilled
    // stage and arrives on its full barrier with its own byte count
    int pt = t0, psub = 0;
    TileWin pw;
    const int jj = threadIdx.x;
    auto produce = [&](int slot) {  // block-uniform
        while (pt < t1) {
            seek_win<0>(pw, wins, nwin, pt);
            const int c = pw.r0 + (pt - pw.pref) * kLeftBN;
            const int ncols = min(kLeftBN, pw.r1 - c);
            if (psub * kLSub >= ncols) {
                ++pt;
                psub = 0;
                continue;
            }
            if (jj < kLSub) {
                double* dst = ring + slot * (kLeftStage / 8) + jj * kLdB;
                long long start = 0;
                int n = 0;
                if (kLSub * psub + jj < ncols)
                    n = plan_segment(dst, S, (long long)pw.a + (long long)(c + kLSub * psub + jj) * lds, pw.d, alloc,
                                     start);
                warp_arrive(&full[slot], (unsigned)n * 8u);
                if (n > 0) bulk_copy(dst, S + start, (unsigned)n * 8u, &full[slot]);
            }
            ++psub;
            return;
        }
    };
    const int wi0 = window_of<0>(wins, nwin, t0);
    load_win<0>(pw, wins, nwin, wi0);
    for (int sl = 0; sl < kLStages; ++sl) produce(sl);

    const int gid = lane >> 2, tig = lane & 3;
    double af[2][kKS];
    unsigned nz0 = 0, nz1 = 0;  // bit ks: fragment af[mt][ks] is nonzero in some lane (warp-uniform)
    unsigned long long ndmma = 0;
    TileWin wd;
    load_win<0>(wd, wins, nwin, wi0);
    int cur = -1, stage = 0, prev = -1;
    unsigned phase = 0;
    for (int t = t0; t < t1; ++t) {
        seek_win<0>(wd, wins, nwin, t);
        const int d = wd.d;
        if (wd.wi != cur) {  // A = Q_w^T: af[mt][ks] = Q_w(k = 4ks + tig, m = 16 wm + 8 mt + gid)
            const double* Qw = qw_pool + wd.qw_off;
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                const int m = 16 * wm + 8 * mt + gid;
#pragma unroll
                for (int ks = 0; ks < kKS; ++ks) {
                    const int k = 4 * ks + tig;
                    af[mt][ks] = (m < d && k < d) ? __ldg(Qw + k + (long long)m * d) : 0.0;
                }
            }
            nz0 = nz1 = 0;
#pragma unroll
            for (int ks = 0; ks < kKS; ++ks) {
                nz0 |= (__any_sync(0xffffffffu, af[0][ks] != 0.0) ? 1u : 0u) << ks;
                nz1 |= (__any_sync(0xffffffffu, af[1][ks] != 0.0) ? 1u : 0u) << ks;
            }
            cur = wd.wi;
        }
        const int c = wd.r0 + (t - wd.pref) * kLeftBN;
        const int ncols = min(kLeftBN, wd.r1 - c);
        double* P = S + (long long)wd.a + (long long)c * lds;
        for (int sub = 0; kLSub * sub < ncols; ++sub) {
            double acc[2][kNT][2];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < kNT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
            // column 8 (wn kNT + nt) + gid, row k = 4 ks + tig (+ the sub-tile's shift)
            const int shift = (int)(((long long)wd.a + (long long)(c + kLSub * sub) * lds) & 1);
            const double* sb = ring + stage * (kLeftStage / 8) + (8 * kNT * wn + gid) * kLdB + tig + shift;
            mbar_wait(&full[stage], phase);
            ndmma += (unsigned long long)(__popc(nz0) + __popc(nz1)) * kNT;
            // Q_w's zero 8x4 fragments (about 45 % of them: a window only mixes
            // the blocks it moves past each other) are skipped -- their products
            // are exact zeros and the sums start at +0, so the bits do not change
#pragma unroll
            for (int ks = 0; ks < kKS; ++ks) {
                const bool u0 = (nz0 >> ks) & 1u, u1 = (nz1 >> ks) & 1u;
                if (!(u0 | u1)) continue;
                double bf[kNT];
#pragma unroll
                for (int nt = 0; nt < kNT; ++nt) bf[nt] = sb[nt * 8 * kLdB + 4 * ks];
                if (u0)
#pragma unroll
                    for (int nt = 0; nt < kNT; ++nt) dmma(acc[0][nt][0], acc[0][nt][1], af[0][ks], bf[nt]);
                if (u1)
#pragma unroll
                    for (int nt = 0; nt < kNT; ++nt) dmma(acc[1][nt][0], acc[1][nt][1], af[1][ks], bf[nt]);
            }
            // epilogue through the consumed stage: accumulators to smem at the
            // inputs' positions, then one bulk store per column (async: the
            // warps go on to the next sub-tile while the TMA engine writes)
            __syncthreads();  // every warp is done reading the stage
            double* so = ring + stage * (kLeftStage / 8) + shift;
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                const int r = 16 * wm + 8 * mt + gid;
#pragma unroll
                for (int nt = 0; nt < kNT; ++nt) {
                    const int cc = 8 * (kNT * wn + nt) + 2 * tig;
                    so[cc * kLdB + r] = acc[mt][nt][0];
                    so[(cc + 1) * kLdB + r] = acc[mt][nt][1];
                }
            }
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncthreads();
            if (jj < kLSub && kLSub * sub + jj < ncols)
                store_column(P + (long long)(kLSub * sub + jj) * lds, so + jj * kLdB, shift, d);
            bulk_commit();
            // refill the stage of the previous sub-tile (its stores went out
            // one sub-tile ago) with the sub-tile a ring depth after it
            if (prev >= 0) {
                bulk_wait_read<1>();
                produce(prev);
            }
            prev = stage;
            if (++stage == kLStages) {
                stage = 0;
                phase ^= 1u;
            }
        }
    }
    if (lane == 0 && ndmma) atomicAdd(&g_dmma_bulk, ndmma);
    bulk_wait_all();  // the last stores land before the CTA retires
}

// ---------------------------------------------------------------------------
// RIGHT: M[r0:r0+64, a:a+d] <- M[r0:r0+64, a:a+d] Q_w, in kRSub-row
// sub-tiles; warp w owns output columns [16 wn, 16 wn + 16) (wn = w mod DW/16)
// of the sub-tile's row slice w / (DW/16).  (64-row sub-tiles:
// the 128 column copies of a stage are 512 bytes each -- 32-row stages of
// 256-byte copies left the ring starved, the TMA engine's per-copy cost.)
template <int DW, int Field>
__global__ void __launch_bounds__(kBulkThreads, DW == 64 ? 2 : 1)
update_right_bulk_kernel(const WinDesc* __restrict__ wins, int nwin, int ntiles, const double* __restrict__ qw_pool,
                         double* __restrict__ M, long long ldm, long long alloc) {
    using C = RightCfg<DW>;
    constexpr int kRightStage = C::kStage, kRStages = C::kStages, kMT = C::kMT, kKS = C::kKS;
    extern __shared__ __align__(128) double ring[];
    __shared__ __align__(8) uint64_t full[kRStages];
    init_ring(full, kRStages, ring, kRStages * kRightStage, DW / 32);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wn = warp % C::kNGroups, wm = warp / C::kNGroups;
    const int t0 = (int)((long long)ntiles * blockIdx.x / gridDim.x);
    const int t1 = (int)((long long)ntiles * (blockIdx.x + 1) / gridDim.x);
    auto tile_rows = [&](const TileWin& w, int t, int& r0, int& nrows) {
        r0 = w.r0 + (t - w.pref) * kRightBM;
        nrows = min(kRightBM, w.r1 - r0);
    };

    // every thread walks the (tile, sub-tile) sequence a ring depth ahead of the
    // one it computes; thread j < DW copies panel column j of each refilled
    // stage and arrives on its full barrier with its own byte count
    int pt = t0, psub = 0;
    TileWin pw;
    const int kk = threadIdx.x;
    auto produce = [&](int slot) {  // block-uniform
        while (pt < t1) {
            seek_win<Field>(pw, wins, nwin, pt);
            int r0, nrows;
            tile_rows(pw, pt, r0, nrows);
            if (psub * kRSub >= nrows) {
                ++pt;
                psub = 0;
                continue;
            }
            if (kk < DW) {
                const int rs = r0 + kRSub * psub, len = min(kRSub, nrows - kRSub * psub);
                double* dst = ring + slot * (kRightStage / 8) + kk * kLdA;
                long long st = 0;
                int n = 0;
                if (kk < pw.d)
                    n = plan_segment(dst, M, (long long)rs + (long long)(pw.a + kk) * ldm, len, alloc, st);
                warp_arrive(&full[slot], (unsigned)n * 8u);
                if (n > 0) bulk_copy(dst, M + st, (unsigned)n * 8u, &full[slot]);
            }
            ++psub;
            return;
        }
    };
    const int wi0 = window_of<Field>(wins, nwin, t0);
    load_win<Field>(pw, wins, nwin, wi0);
    for (int sl = 0; sl < kRStages; ++sl) produce(sl);

    const int gid = lane >> 2, tig = lane & 3;
    double bf[2][kKS];
    unsigned nz0 = 0, nz1 = 0;  // bit ks: fragment bf[nt][ks] is nonzero in some lane (warp-uniform)
    unsigned long long ndmma = 0;
    TileWin wd;
    load_win<Field>(wd, wins, nwin, wi0);
    int cur = -1, stage = 0;
    unsigned phase = 0;
    for (int t = t0; t < t1; ++t) {
        seek_win<Field>(wd, wins, nwin, t);
        const int d = wd.d;
        if (wd.wi != cur) {  // B = Q_w: bf[nt][ks] = Q_w(k = 4ks + tig, n = 16 wn + 8 nt + gid)
            const double* Qw = qw_pool + wd.qw_off;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                const int nn = 16 * wn + 8 * nt + gid;
#pragma unroll
                for (int ks = 0; ks < kKS; ++ks) {
                    const int k = 4 * ks + tig;
                    bf[nt][ks] = (nn < d && k < d) ? __ldg(Qw + k + (long long)nn * d) : 0.0;
                }
            }
            nz0 = nz1 = 0;
#pragma unroll
            for (int ks = 0; ks < kKS; ++ks) {
                nz0 |= (__any_sync(0xffffffffu, bf[0][ks] != 0.0) ? 1u : 0u) << ks;
                nz1 |= (__any_sync(0xffffffffu, bf[1][ks] != 0.0) ? 1u : 0u) << ks;
            }
            cur = wd.wi;
        }
        int r0, nrows;
        tile_rows(wd, t, r0, nrows);
        double* P = M + (long long)r0 + (long long)wd.a * ldm;
        for (int sub = 0; kRSub * sub < nrows; ++sub) {
            double acc[kMT][2][2];
#pragma unroll
            for (int i = 0; i < kMT; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
            // row 8 mt + gid, column k = 4 ks + tig (+ the sub-tile's shift)
            const int shift = (int)(((long long)r0 + kRSub * sub + (long long)wd.a * ldm) & 1);
            const double* sa = ring + stage * (kRightStage / 8) + tig * kLdA + 8 * kMT * wm + gid + shift;
            mbar_wait(&full[stage], phase);
            ndmma += (unsigned long long)(__popc(nz0) + __popc(nz1)) * kMT;
            // zero fragments of Q_w skipped (exact: see the left kernel)
#pragma unroll
            for (int ks = 0; ks < kKS; ++ks) {
                const bool u0 = (nz0 >> ks) & 1u, u1 = (nz1 >> ks) & 1u;
                if (!(u0 | u1)) continue;
                double a[kMT];
#pragma unroll
                for (int mt = 0; mt < kMT; ++mt) a[mt] = sa[4 * ks * kLdA + 8 * mt];
                if (u0)
#pragma unroll
                    for (int mt = 0; mt < kMT; ++mt) dmma(acc[mt][0][0], acc[mt][0][1], a[mt], bf[0][ks]);
                if (u1)
#pragma unroll
                    for (int mt = 0; mt < kMT; ++mt) dmma(acc[mt][1][0], acc[mt][1][1], a[mt], bf[1][ks]);
            }
            // direct stores: with a 3-deep ring of 64-row stages the staged
            // (bulk-store) epilogue of the left kernel delays the refill by one
            // sub-tile and measured 2-3 % slower here
            __syncthreads();  // the stage is free
            produce(stage);
            if (++stage == kRStages) {
                stage = 0;
                phase ^= 1u;
            }
#pragma unroll
            for (int mt = 0; mt < kMT; ++mt) {
                const int r = kRSub * sub + 8 * (kMT * wm + mt) + gid;
                if (r >= nrows) continue;
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) {
                    const int cc = 16 * wn + 8 * nt + 2 * tig;
                    if (cc < d) P[r + (long long)cc * ldm] = acc[mt][nt][0];
                    if (cc + 1 < d) P[r + (long long)(cc + 1) * ldm] = acc[mt][nt][1];
                }
            }
        }
    }
    if (lane == 0 && ndmma) atomicAdd(&g_dmma_bulk, ndmma);
}

// ---------------------------------------------------------------------------
// LEFT, windows of order <= 64: S[a:a+d, c:c+64] <- Q_w^T S[a:a+d, c:c+64], in kLSub-column
// sub-tiles; warp w owns output rows [16 wm, 16 wm + 16) (wm = w mod DW/16)
// of the sub-tile's column slice w / (DW/16).
__global__ void __launch_bounds__(kBulkThreads, 2)
update_left_bulk64_kernel(const WinDesc* __restrict__ wins, int nwin, int ntiles, const double* __restrict__ qw_pool,
                        double* __restrict__ S, long long lds, long long alloc) {
    constexpr int DW = 64;
    using C = Left64Cfg;
    constexpr int kLdB = C::kLd, kLeftStage = C::kStage, kLStages = C::kStages, kNT = C::kNT, kKS = C::kKS;
    constexpr int FT = C::kFT;
    extern __shared__ __align__(128) double ring[];
    __shared__ __align__(8) uint64_t full[kLStages];
    init_ring(full, kLStages, ring, kLStages * kLeftStage, kLSub / 32);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm = warp % C::kMGroups, wn = warp / C::kMGroups;
    const int t0 = (int)((long long)ntiles * blockIdx.x / gridDim.x);
    const int t1 = (int)((long long)ntiles * (blockIdx.x + 1) / gridDim.x);

    // every thread walks the (tile, sub-tile) sequence a ring depth ahead of the
    // one it computes; thread j < kLSub copies panel column j of each refilled
    // stage and arrives on its full barrier with its own byte count
    int pt = t0, psub = 0;
    TileWin pw;
    const int jj = threadIdx.x;
    auto produce = [&](int slot) {  // block-uniform
        while (pt < t1) {
            seek_win<0>(pw, wins, nwin, pt);
            const int c = pw.r0 + (pt - pw.pref) * kLeftBN;
            const int ncols = min(kLeftBN, pw.r1 - c);
            if (psub * kLSub >= ncols) {
                ++pt;
                psub = 0;
                continue;
            }
            if (jj < kLSub) {
                double* dst = ring + slot * (kLeftStage / 8) + jj * kLdB;
                long long start = 0;
                int n = 0;
                if (kLSub * psub + jj < ncols)
                    n = plan_segment(dst, S, (long long)pw.a + (long long)(c + kLSub * psub + jj) * lds, pw.d, alloc,
                                     start);
                warp_arrive(&full[slot], (unsigned)n * 8u);
                if (n > 0) bulk_copy(dst, S + start, (unsigned)n * 8u, &full[slot]);
            }
            ++psub;
            return;
        }
    };
    const int wi0 = window_of<0>(wins, nwin, t0);
    load_win<0>(pw, wins, nwin, wi0);
    for (int sl = 0; sl < kLStages; ++sl) produce(sl);

    const int gid = lane >> 2, tig = lane & 3;
    double af[FT][kKS];
    unsigned nz[FT];  // bit ks: fragment af[mt][ks] is nonzero in some lane (warp-uniform)
#pragma unroll
    for (int f = 0; f < FT; ++f) nz[f] = 0;
    unsigned long long ndmma = 0;
    TileWin wd;
    load_win<0>(wd, wins, nwin, wi0);
    int cur = -1, stage = 0, prev = -1;
    unsigned phase = 0;
    for (int t = t0; t < t1; ++t) {
        seek_win<0>(wd, wins, nwin, t);
        const int d = wd.d;
        if (wd.wi != cur) {  // A = Q_w^T: af[mt][ks] = Q_w(k = 4ks + tig, m = 8 (FT wm + mt) + gid)
            const double* Qw = qw_pool + wd.qw_off;
#pragma unroll
            for (int mt = 0; mt < FT; ++mt) {
                const int m = 8 * (FT * wm + mt) + gid;
#pragma unroll
                for (int ks = 0; ks < kKS; ++ks) {
                    const int k = 4 * ks + tig;
                    af[mt][ks] = (m < d && k < d) ? __ldg(Qw + k + (long long)m * d) : 0.0;
                }
            }
#pragma unroll
            for (int mt = 0; mt < FT; ++mt) nz[mt] = 0;
#pragma unroll
            for (int ks = 0; ks < kKS; ++ks)
#pragma unroll
                for (int mt = 0; mt < FT; ++mt) nz[mt] |= (__any_sync(0xffffffffu, af[mt][ks] != 0.0) ? 1u : 0u) << ks;
            cur = wd.wi;
        }
        const int c = wd.r0 + (t - wd.pref) * kLeftBN;
        const int ncols = min(kLeftBN, wd.r1 - c);
        double* P = S + (long long)wd.a + (long long)c * lds;
        for (int sub = 0; kLSub * sub < ncols; ++sub) {
            double acc[FT][kNT][2];
#pragma unroll
            for (int i = 0; i < FT; ++i)
#pragma unroll
                for (int j = 0; j < kNT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
            // column 8 (wn kNT + nt) + gid, row k = 4 ks + tig (+ the sub-tile's shift)
            const int shift = (int)(((long long)wd.a + (long long)(c + kLSub * sub) * lds) & 1);
            const double* sb = ring + stage * (kLeftStage / 8) + (8 * kNT * wn + gid) * kLdB + tig + shift;
            mbar_wait(&full[stage], phase);
#pragma unroll
            for (int mt = 0; mt < FT; ++mt) ndmma += (unsigned long long)__popc(nz[mt]) * kNT;
            // Q_w's zero 8x4 fragments (about 45 % of them: a window only mixes
            // the blocks it moves past each other) are skipped -- their products
            // are exact zeros and the sums start at +0, so the bits do not change
#pragma unroll
            for (int ks = 0; ks < kKS; ++ks) {
                bool u[FT], any = false;
#pragma unroll
                for (int mt = 0; mt < FT; ++mt) {
                    u[mt] = (nz[mt] >> ks) & 1u;
                    any |= u[mt];
                }
                if (!any) continue;
                double bf[kNT];
#pragma unroll
                for (int nt = 0; nt < kNT; ++nt) bf[nt] = sb[nt * 8 * kLdB + 4 * ks];
#pragma unroll
                for (int mt = 0; mt < FT; ++mt)
                    if (u[mt])
#pragma unroll
                        for (int nt = 0; nt < kNT; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt][ks], bf[nt]);
            }
            // epilogue through the consumed stage: accumulators to smem at the
            // inputs' positions, then one bulk store per column (async: the
            // warps go on to the next sub-tile while the TMA engine writes)
            __syncthreads();  // every warp is done reading the stage
            double* so = ring + stage * (kLeftStage / 8) + shift;
#pragma unroll
            for (int mt = 0; mt < FT; ++mt) {
                const int r = 8 * (FT * wm + mt) + gid;
#pragma unroll
                for (int nt = 0; nt < kNT; ++nt) {
                    const int cc = 8 * (kNT * wn + nt) + 2 * tig;
                    so[cc * kLdB + r] = acc[mt][nt][0];
                    so[(cc + 1) * kLdB + r] = acc[mt][nt][1];
                }
            }
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncthreads();
            if (jj < kLSub && kLSub * sub + jj < ncols)
                store_column(P + (long long)(kLSub * sub + jj) * lds, so + jj * kLdB, shift, d);
            bulk_commit();
            // refill the stage of the previous sub-tile (its stores went out
            // one sub-tile ago) with the sub-tile a ring depth after it
            if (prev >= 0) {
                bulk_wait_read<1>();
                produce(prev);
            }
            prev = stage;
            if (++stage == kLStages) {
                stage = 0;
                phase ^= 1u;
            }
        }
    }
    if (lane == 0 && ndmma) atomicAdd(&g_dmma_bulk, ndmma);
    bulk_wait_all();  // the last stores land before the CTA retires
}

// ---------------------------------------------------------------------------
// RIGHT, windows of order <= 64: M[r0:r0+64, a:a+d] <- M[r0:r0+64, a:a+d] Q_w, in kRSub-row
// sub-tiles; warp w owns output columns [16 wn, 16 wn + 16) (wn = w mod DW/16)
// of the sub-tile's row slice w / (DW/16).  (64-row sub-tiles:
// the 128 column copies of a stage are 512 bytes each -- 32-row stages of
// 256-byte copies left the ring starved, the TMA engine's per-copy cost.)
template <int Field>
__global__ void __launch_bounds__(kBulkThreads, 2)
update_right_bulk64_kernel(const WinDesc* __restrict__ wins, int nwin, int ntiles, const double* __restrict__ qw_pool,
                         double* __restrict__ M, long long ldm, long long alloc) {
    constexpr int DW = 64;
    using C = Right64Cfg;
    constexpr int kRightStage = C::kStage, kRStages = C::kStages, kMT = C::kMT, kKS = C::kKS;
    constexpr int FT = C::kFT;
    extern __shared__ __align__(128) double ring[];
    __shared__ __align__(8) uint64_t full[kRStages];
    init_ring(full, kRStages, ring, kRStages * kRightStage, DW / 32);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wn = warp % C::kNGroups, wm = warp / C::kNGroups;
    const int t0 = (int)((long long)ntiles * blockIdx.x / gridDim.x);
    const int t1 = (int)((long long)ntiles * (blockIdx.x + 1) / gridDim.x);
    auto tile_rows = [&](const TileWin& w, int t, int& r0, int& nrows) {
        r0 = w.r0 + (t - w.pref) * kRightBM;
        nrows = min(kRightBM, w.r1 - r0);
    };

    // every thread walks the (tile, sub-tile) sequence a ring depth ahead of the
    // one it computes; thread j < DW copies panel column j of each refilled
    // stage and arrives on its full barrier with its own byte count
    int pt = t0, psub = 0;
    TileWin pw;
    const int kk = threadIdx.x;
    auto produce = [&](int slot) {  // block-uniform
        while (pt < t1) {
            seek_win<Field>(pw, wins, nwin, pt);
            int r0, nrows;
            tile_rows(pw, pt, r0, nrows);
            if (psub * kRSub >= nrows) {
                ++pt;
                psub = 0;
                continue;
            }
            if (kk < DW) {
                const int rs = r0 + kRSub * psub, len = min(kRSub, nrows - kRSub * psub);
                double* dst = ring + slot * (kRightStage / 8) + kk * kLdA;
                long long st = 0;
                int n = 0;
                if (kk < pw.d)
                    n = plan_segment(dst, M, (long long)rs + (long long)(pw.a + kk) * ldm, len, alloc, st);
                warp_arrive(&full[slot], (unsigned)n * 8u);
                if (n > 0) bulk_copy(dst, M + st, (unsigned)n * 8u, &full[slot]);
            }
            ++psub;
            return;
        }
    };
    const int wi0 = window_of<Field>(wins, nwin, t0);
    load_win<Field>(pw, wins, nwin, wi0);
    for (int sl = 0; sl < kRStages; ++sl) produce(sl);

    const int gid = lane >> 2, tig = lane & 3;
    double bf[FT][kKS];
    unsigned nz[FT];  // bit ks: fragment bf[nt][ks] is nonzero in some lane (warp-uniform)
#pragma unroll
    for (int f = 0; f < FT; ++f) nz[f] = 0;
    unsigned long long ndmma = 0;
    TileWin wd;
    load_win<Field>(wd, wins, nwin, wi0);
    int cur = -1, stage = 0;
    unsigned phase = 0;
    for (int t = t0; t < t1; ++t) {
        seek_win<Field>(wd, wins, nwin, t);
        const int d = wd.d;
        if (wd.wi != cur) {  // B = Q_w: bf[nt][ks] = Q_w(k = 4ks + tig, n = 8 (FT wn + nt) + gid)
            const double* Qw = qw_pool + wd.qw_off;
#pragma unroll
            for (int nt = 0; nt < FT; ++nt) {
                const int nn = 8 * (FT * wn + nt) + gid;
#pragma unroll
                for (int ks = 0; ks < kKS; ++ks) {
                    const int k = 4 * ks + tig;
                    bf[nt][ks] = (nn < d && k < d) ? __ldg(Qw + k + (long long)nn * d) : 0.0;
                }
            }
#pragma unroll
            for (int nt = 0; nt < FT; ++nt) nz[nt] = 0;
#pragma unroll
            for (int ks = 0; ks < kKS; ++ks)
#pragma unroll
                for (int nt = 0; nt < FT; ++nt) nz[nt] |= (__any_sync(0xffffffffu, bf[nt][ks] != 0.0) ? 1u : 0u) << ks;
            cur = wd.wi;
        }
        int r0, nrows;
        tile_rows(wd, t, r0, nrows);
        double* P = M + (long long)r0 + (long long)wd.a * ldm;
        for (int sub = 0; kRSub * sub < nrows; ++sub) {
            double acc[kMT][FT][2];
#pragma unroll
            for (int i = 0; i < kMT; ++i)
#pragma unroll
                for (int j = 0; j < FT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
            // row 8 mt + gid, column k = 4 ks + tig (+ the sub-tile's shift)
            const int shift = (int)(((long long)r0 + kRSub * sub + (long long)wd.a * ldm) & 1);
            const double* sa = ring + stage * (kRightStage / 8) + tig * kLdA + 8 * kMT * wm + gid + shift;
            mbar_wait(&full[stage], phase);
#pragma unroll
            for (int nt = 0; nt < FT; ++nt) ndmma += (unsigned long long)__popc(nz[nt]) * kMT;
            // zero fragments of Q_w skipped (exact: see the left kernel)
#pragma unroll
            for (int ks = 0; ks < kKS; ++ks) {
                bool u[FT], any = false;
#pragma unroll
                for (int nt = 0; nt < FT; ++nt) {
                    u[nt] = (nz[nt] >> ks) & 1u;
                    any |= u[nt];
                }
                if (!any) continue;
                double a[kMT];
#pragma unroll
                for (int mt = 0; mt < kMT; ++mt) a[mt] = sa[4 * ks * kLdA + 8 * mt];
#pragma unroll
                for (int nt = 0; nt < FT; ++nt)
                    if (u[nt])
#pragma unroll
                        for (int mt = 0; mt < kMT; ++mt) dmma(acc[mt][nt][0], acc[mt][nt][1], a[mt], bf[nt][ks]);
            }
            // direct stores: with a 3-deep ring of 64-row stages the staged
            // (bulk-store) epilogue of the left kernel delays the refill by one
            // sub-tile and measured 2-3 % slower here
            __syncthreads();  // the stage is free
            produce(stage);
            if (++stage == kRStages) {
                stage = 0;
                phase ^= 1u;
            }
#pragma unroll
            for (int mt = 0; mt < kMT; ++mt) {
                const int r = kRSub * sub + 8 * (kMT * wm + mt) + gid;
                if (r >= nrows) continue;
#pragma unroll
                for (int nt = 0; nt < FT; ++nt) {
                    const int cc = 8 * (FT * wn + nt) + 2 * tig;
                    if (cc < d) P[r + (long long)cc * ldm] = acc[mt][nt][0];
                    if (cc + 1 < d) P[r + (long long)(cc + 1) * ldm] = acc[mt][nt][1];
                }
            }
        }
    }
    if (lane == 0 && ndmma) atomicAdd(&g_dmma_bulk, ndmma);
}

// ---------------------------------------------------------------------------
// host side

namespace {

bool bulk_disabled() {
    static const bool off = getenv("TEIG_NO_TMA") && atoi(getenv("TEIG_NO_TMA"));
    return off;
}

// `per_sm` CTAs per SM while every CTA gets >= kMinTilesPerCta tiles
int grid_for(int ntiles, int per_sm = 1) {
    const int sms = device_sm_count() * per_sm;
    return std::max(1, std::min(sms, (ntiles + kMinTilesPerCta - 1) / kMinTilesPerCta));
}

// TEIG_NO_BULK64=1: windows of order <= 64 take the cp.async kernels
bool bulk64_disabled() {
    static const bool off = getenv("TEIG_NO_BULK64") && atoi(getenv("TEIG_NO_BULK64"));
    return off;
}

bool bulk_eligible(int dmax, const double* base, long long ld, long long rows, long long cols) {
    return !bulk_disabled() && dmax >= 1 && dmax <= 128 && (dmax > 64 || !bulk64_disabled()) && rows > 0 &&
           cols > 0 && (ld % 2) == 0 && (reinterpret_cast<uintptr_t>(base) % 16) == 0 && kLeftBN == 64 &&
           kRightBM == 64;
}

template <int DW>
cudaError_t left_bulk(const WinDesc* wins, int nwin, int ntiles, const double* qw_pool, double* S, long long lds,
                      long long alloc, int grid, cudaStream_t stream) {
    if constexpr (DW == 64) {
        constexpr size_t smem = Left64Cfg::kSmem;
        cudaError_t e = ensure_dyn_smem((const void*)update_left_bulk64_kernel, smem);
        if (e != cudaSuccess) return e;
        update_left_bulk64_kernel<<<grid, kBulkThreads, smem, stream>>>(wins, nwin, ntiles, qw_pool, S, lds, alloc);
    } else {
        constexpr size_t smem = LeftCfg<DW>::kSmem;
        cudaError_t e = ensure_dyn_smem((const void*)update_left_bulk_kernel<DW>, smem);
        if (e != cudaSuccess) return e;
        update_left_bulk_kernel<DW><<<grid, kBulkThreads, smem, stream>>>(wins, nwin, ntiles, qw_pool, S, lds, alloc);
    }
    return cudaGetLastError();
}

template <int DW, int Field>
cudaError_t right_bulk(const WinDesc* wins, int nwin, int ntiles, const double* qw_pool, double* M, long long ldm,
                       long long alloc, int grid, cudaStream_t stream) {
    if constexpr (DW == 64) {
        constexpr size_t smem = Right64Cfg::kSmem;
        cudaError_t e = ensure_dyn_smem((const void*)update_right_bulk64_kernel<Field>, smem);
        if (e != cudaSuccess) return e;
        update_right_bulk64_kernel<Field><<<grid, kBulkThreads, smem, stream>>>(wins, nwin, ntiles, qw_pool, M, ldm,
                                                                                  alloc);
    } else {
        constexpr size_t smem = RightCfg<DW>::kSmem;
        cudaError_t e = ensure_dyn_smem((const void*)update_right_bulk_kernel<DW, Field>, smem);
        if (e != cudaSuccess) return e;
        update_right_bulk_kernel<DW, Field><<<grid, kBulkThreads, smem, stream>>>(wins, nwin, ntiles, qw_pool, M,
                                                                                  ldm, alloc);
    }
    return cudaGetLastError();
}

}  // namespace

bool launch_update_left_tma(const WinDesc* wins, int nwin, int ntiles, int dmax, const double* qw_pool, double* S,
                            long long lds, long long rows, long long cols, cudaStream_t stream, cudaError_t* err,
                            int max_ctas) {
    *err = cudaSuccess;
    if (ntiles <= 0) return true;
    if (!bulk_eligible(dmax, S, lds, rows, cols)) return false;
    const int per_sm = dmax > 64 ? 1 : 2;  // order <= 64: two CTAs per SM hide each other's barriers
    const int grid = max_ctas > 0   ? std::min(grid_for(ntiles, per_sm), max_ctas * per_sm)
                     : max_ctas < 0 ? std::min(ntiles, device_sm_count() * per_sm)
                                    : grid_for(ntiles, per_sm);
    const long long alloc = (cols - 1) * lds + rows;
    *err = dmax > 64 ? left_bulk<128>(wins, nwin, ntiles, qw_pool, S, lds, alloc, grid, stream)
                     : left_bulk<64>(wins, nwin, ntiles, qw_pool, S, lds, alloc, grid, stream);
    return true;
}

bool launch_update_right_tma(const WinDesc* wins, int nwin, int ntiles, int dmax, const double* qw_pool, double* M,
                             long long ldm, long long rows, long long cols, bool factor, cudaStream_t stream,
                             cudaError_t* err, bool short_ctas, int max_ctas, int short_tiles) {
    *err = cudaSuccess;
    if (ntiles <= 0) return true;
    if (!bulk_eligible(dmax, M, ldm, rows, cols)) return false;
    // short_ctas: the caller runs these updates on a low-priority stream beside
    // the critical path -- CTAs of short_tiles tiles, so critical-path CTAs can
    // take SMs as they free up; otherwise a persistent grid
    const int per_sm = dmax > 64 ? 1 : 2;
    const int st = std::max(1, short_tiles);
    int grid = short_ctas ? (ntiles + st - 1) / st : grid_for(ntiles, per_sm);
    if (max_ctas > 0 && !short_ctas) grid = std::min(grid, max_ctas * per_sm);
    if (max_ctas < 0 && !short_ctas) grid = std::min(ntiles, device_sm_count() * per_sm);
    const long long alloc = (cols - 1) * ldm + rows;
    if (dmax > 64)
        *err = factor ? right_bulk<128, 2>(wins, nwin, ntiles, qw_pool, M, ldm, alloc, grid, stream)
                      : right_bulk<128, 1>(wins, nwin, ntiles, qw_pool, M, ldm, alloc, grid, stream);
    else
        *err = factor ? right_bulk<64, 2>(wins, nwin, ntiles, qw_pool, M, ldm, alloc, grid, stream)
                      : right_bulk<64, 1>(wins, nwin, ntiles, qw_pool, M, ldm, alloc, grid, stream);
    return true;
}

unsigned long long dmma_count_bulk() {
    unsigned long long v = 0;
    if (cudaMemcpyFromSymbol(&v, g_dmma_bulk, sizeof v) != cudaSuccess) cudaGetLastError();
    return v;
}

}  // namespace teig
