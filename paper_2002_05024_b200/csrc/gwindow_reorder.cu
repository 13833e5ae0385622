// gwindow_reorder.cu -- batched single-CTA window kernel of the GENERALIZED
// Schur-pair reordering (S, T) with Q and Z (
// sm_100a).
//
// The window of the reference's reorder plan (reorder.cpp:271-324, the same
// planner serves the pair: block sizes come from S's subdiagonal) is moved in
// shared memory as a PAIR: S and T windows (T upper triangular) plus the two
// accumulators Q_w (left) and Z_w (right), d <= 64.  As in the standard
// window kernel (window_reorder.cu) the bubble of the reference's
// window_reorder (reorder.cpp:124-194) is scheduled as a parallel odd-even
// transposition: every step swaps ALL adjacent (unselected, selected & not
// stuck) block pairs at once -- their transformations act on disjoint index
// sets and commute.  A step is four barrier-separated phases:
//   1. warp 0 lists the pairs (ballot ranks, shuffle scan of the row starts);
//   2. one WARP per pair decides the swap (gswap_warp.cuh: generalized
//      Sylvester + QR of the deflating-subspace bases, DTGEX2 semantics,
//      the elimination and products spread over the lanes), pairs
//      round-robin over the 8 warps;
//   3. rows of every pair (S and T, columns right of the block) <- Q_m^T;
//   4. columns of every pair (S and T rows above; all rows of Q_w / Z_w)
//      <- Q_m / Z_m, and the new diagonal blocks;
// then warp 0 commits the arrangement (a rejected swap marks its selected
// block stuck: it stops, later blocks stack below it) and lists the next
// step's pairs behind the same barrier.
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "device_types.h"
#include "gswap_warp.cuh"
#include "launch.h"

namespace teig {

namespace {

constexpr int kGThreads = 256;
constexpr int kGMaxD = 64;
constexpr int kGMaxBlocks = 64;
constexpr int kGMaxPairs = 32;

struct GPair {
    int16_t pos, slot;
    int8_t p, q, ok, pad;
};

struct GShared {
    uint8_t arr[kGMaxBlocks], bsz[kGMaxBlocks], bsel[kGMaxBlocks], bstuck[kGMaxBlocks];
    GPair pairs[kGMaxPairs];
    int npairs;
    int executed;
    int skipped;
    double Qm[kGMaxPairs][16], Zm[kGMaxPairs][16], An[kGMaxPairs][16], Bn[kGMaxPairs][16];
    GSwapScratch ws[kGThreads / 32];
};

template <int P, int Q>
__device__ __forceinline__ void decide(GShared& sh, const double* Sw, const double* Tw, int ld, int pi, int lane,
                                       GSwapScratch& ws) {
    GPair& pr = sh.pairs[pi];
    const bool ok = wgswap<P, Q>(Sw, Tw, ld, pr.pos, ws, lane, sh.Qm[pi], sh.Zm[pi], sh.An[pi], sh.Bn[pi]);
    if (lane == 0) pr.ok = ok ? 1 : 0;
}

// rows pos.. of M (ld), columns [pos+D, d) <- U^T rows  (lanes over columns)
template <int D>
__device__ __forceinline__ void rows_apply(double* M, int ld, int d, int pos, const double* Ug, int lane) {
    double U[D][D];
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
        for (int i = 0; i < D; ++i) U[r][i] = Ug[r * D + i];
    for (int c = pos + D + lane; c < d; c += 32) {
        double* col = M + pos + c * ld;
        double x[D];
#pragma unroll
        for (int r = 0; r < D; ++r) x[r] = col[r];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double a = 0.0;
#pragma unroll
            for (int r = 0; r < D; ++r) a += U[r][i] * x[r];
            col[i] = a;
        }
    }
}

// columns pos.. of M (ld), rows [0, r1) <- rows V  (lanes over rows)
template <int D>
__device__ __forceinline__ void cols_apply(double* M, int ld, int r1, int pos, const double* Vg, int lane) {
    double V[D][D];
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
        for (int j = 0; j < D; ++j) V[r][j] = Vg[r * D + j];
    for (int i = lane; i < r1; i += 32) {
        double* row = M + i + pos * ld;
        double x[D];
#pragma unroll
        for (int r = 0; r < D; ++r) x[r] = row[r * ld];
#pragma unroll
        for (int j = 0; j < D; ++j) {
            double a = 0.0;
#pragma unroll
            for (int r = 0; r < D; ++r) a += x[r] * V[r][j];
            row[j * ld] = a;
        }
    }
}

template <int D>
__device__ __forceinline__ void pair_phase_rows(GShared& sh, double* Sw, double* Tw, int ld, int d, int pi, int lane) {
    const GPair pr = sh.pairs[pi];
    rows_apply<D>(Sw, ld, d, pr.pos, sh.Qm[pi], lane);
    rows_apply<D>(Tw, ld, d, pr.pos, sh.Qm[pi], lane);
}

template <int D>
__device__ __forceinline__ void pair_phase_cols(GShared& sh, double* Sw, double* Tw, double* Qw, double* Zw, int ld,
                                                int d, int pi, int lane) {
    const GPair pr = sh.pairs[pi];
    cols_apply<D>(Sw, ld, pr.pos, pr.pos, sh.Zm[pi], lane);
    cols_apply<D>(Tw, ld, pr.pos, pr.pos, sh.Zm[pi], lane);
    cols_apply<D>(Qw, ld, d, pr.pos, sh.Qm[pi], lane);
    cols_apply<D>(Zw, ld, d, pr.pos, sh.Zm[pi], lane);
    if (lane < D * D) {
        const int i = lane / D, j = lane % D;
        Sw[(pr.pos + i) + (pr.pos + j) * ld] = sh.An[pi][lane];
        Tw[(pr.pos + i) + (pr.pos + j) * ld] = sh.Bn[pi][lane];
    }
}

// warp 0: every adjacent (unselected, selected & not stuck) slot pair of the
// current arrangement.  Two candidates never overlap (the upper block of one
// is unselected, the lower of the other selected), so all slots are tested
// at once: a ballot ranks the pairs, a shuffle scan gives the row starts.
__device__ __forceinline__ void gfind_pairs(GShared& sh, int nb, int lane) {
    int loc[2], sum = 0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int s = lane * 2 + k;
        loc[k] = (s < nb) ? sh.bsz[sh.arr[s]] : 0;
        sum += loc[k];
    }
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    const int r0 = incl - sum;
    bool cand[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {  // slot s = 2 lane + k
        const int s = lane * 2 + k;
        cand[k] = s + 1 < nb && !sh.bsel[sh.arr[s]] && sh.bsel[sh.arr[s + 1]] && !sh.bstuck[sh.arr[s + 1]];
    }
    const unsigned c0 = __ballot_sync(0xffffffffu, cand[0]), c1 = __ballot_sync(0xffffffffu, cand[1]);
    const int np = __popc(c0) + __popc(c1);
    const unsigned below = (1u << lane) - 1u;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        if (!cand[k]) continue;
        const int s = lane * 2 + k;
        // rank in slot order: both slots of the lower lanes, and slot 2 lane before 2 lane + 1
        const int idx = __popc(c0 & below) + __popc(c1 & below) + (k == 1 && cand[0] ? 1 : 0);
        const int u = sh.arr[s], b = sh.arr[s + 1];
        GPair pr;
        pr.pos = (int16_t)(r0 + (k == 1 ? loc[0] : 0));
        pr.slot = (int16_t)s;
        pr.p = (int8_t)sh.bsz[u];
        pr.q = (int8_t)sh.bsz[b];
        pr.ok = 0;
        pr.pad = 0;
        sh.pairs[idx] = pr;
    }
    if (lane == 0) sh.npairs = np;
    __syncwarp();
}

}  // namespace

__global__ void __launch_bounds__(kGThreads, 1)
gwindow_reorder_kernel(const WinDesc* __restrict__ wins, double* __restrict__ S, long long lds, double* __restrict__ T,
                       long long ldt, double* __restrict__ qw_pool, const uint8_t* __restrict__ sizes_pool,
                       const uint8_t* __restrict__ sel_pool, uint8_t* __restrict__ order_pool,
                       uint8_t* __restrict__ stuck_pool, int32_t* __restrict__ status,
                       int32_t* __restrict__ dev_level) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    GShared& sh = *reinterpret_cast<GShared*>(smem_raw);
    const WinDesc wd = wins[blockIdx.x];
    const int d = wd.d, nb = wd.nb, a = wd.a;
    const int ld = d | 1;
    double* Sw = reinterpret_cast<double*>(smem_raw + ((sizeof(GShared) + 15) & ~size_t(15)));
    double* Tw = Sw + ld * d;
    double* Qw = Tw + ld * d;
    double* Zw = Qw + ld * d;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = kGThreads / 32;
    for (int idx = tid; idx < d * d; idx += kGThreads) {
        const int j = idx / d, i = idx - j * d;
        Sw[i + j * ld] = S[(long long)(a + i) + (long long)(a + j) * lds];
        Tw[i + j * ld] = T[(long long)(a + i) + (long long)(a + j) * ldt];
        Qw[i + j * ld] = (i == j) ? 1.0 : 0.0;
        Zw[i + j * ld] = (i == j) ? 1.0 : 0.0;
    }
    if (tid < nb) {
        sh.arr[tid] = (uint8_t)tid;
        sh.bsz[tid] = sizes_pool[wd.blk_off + tid];
        sh.bsel[tid] = sel_pool[wd.blk_off + tid];
        sh.bstuck[tid] = 0;
    }
    __syncthreads();
    if (tid == 0) {  // expected layout vs S's subdiagonal (reorder.cpp:132-154)
        // an earlier level deviated: this window's planned layout is stale
        const bool skip = dev_level && __ldcg(dev_level) < wd.level;
        int row = 0, ok = skip ? 0 : 1;
        sh.skipped = skip;
        for (int b = 0; b < nb && ok; ++b) {
            const int sz = sh.bsz[b];
            if (row + sz > d) ok = 0;
            else if (sz == 2 && Sw[(row + 1) + row * ld] == 0.0) ok = 0;
            else if (row + sz < d && Sw[(row + sz) + (row + sz - 1) * ld] != 0.0) ok = 0;
            row += sz;
        }
        if (ok && row != d) ok = 0;
        sh.executed = ok;
    }
    __syncthreads();
    if (sh.executed) {
        if (warp == 0) gfind_pairs(sh, nb, lane);  // list the first step's pairs
        __syncthreads();
        for (;;) {
            const int np = sh.npairs;
            if (np == 0) break;
            for (int pi = warp; pi < np; pi += NW) {  // decisions, one warp per pair
                const GPair pr = sh.pairs[pi];
                if (pr.p == 1 && pr.q == 1) decide<1, 1>(sh, Sw, Tw, ld, pi, lane, sh.ws[warp]);
                else if (pr.p == 1) decide<1, 2>(sh, Sw, Tw, ld, pi, lane, sh.ws[warp]);
                else if (pr.q == 1) decide<2, 1>(sh, Sw, Tw, ld, pi, lane, sh.ws[warp]);
                else decide<2, 2>(sh, Sw, Tw, ld, pi, lane, sh.ws[warp]);
            }
            __syncthreads();
            for (int pi = warp; pi < np; pi += NW) {
                const GPair pr = sh.pairs[pi];
                if (!pr.ok) continue;
                const int D = pr.p + pr.q;
                if (D == 2) pair_phase_rows<2>(sh, Sw, Tw, ld, d, pi, lane);
                else if (D == 3) pair_phase_rows<3>(sh, Sw, Tw, ld, d, pi, lane);
                else pair_phase_rows<4>(sh, Sw, Tw, ld, d, pi, lane);
            }
            __syncthreads();
            for (int pi = warp; pi < np; pi += NW) {
                const GPair pr = sh.pairs[pi];
                if (!pr.ok) continue;
                const int D = pr.p + pr.q;
                if (D == 2) pair_phase_cols<2>(sh, Sw, Tw, Qw, Zw, ld, d, pi, lane);
                else if (D == 3) pair_phase_cols<3>(sh, Sw, Tw, Qw, Zw, ld, d, pi, lane);
                else pair_phase_cols<4>(sh, Sw, Tw, Qw, Zw, ld, d, pi, lane);
            }
            __syncthreads();
            if (warp == 0) {  // commit (a lane per pair: disjoint slots), then the next step's pairs
                if (lane < np) {
                    const GPair pr = sh.pairs[lane];
                    const int u = sh.arr[pr.slot], b = sh.arr[pr.slot + 1];
                    if (pr.ok) {
                        sh.arr[pr.slot] = (uint8_t)b;
                        sh.arr[pr.slot + 1] = (uint8_t)u;
                    } else {
                        sh.bstuck[b] = 1;
                    }
                }
                __syncwarp();
                gfind_pairs(sh, nb, lane);
            }
            __syncthreads();
        }
    }
    // scatter the window pair and publish Q_w, Z_w (identity when not executed)
    for (int idx = tid; idx < d * d; idx += kGThreads) {
        const int j = idx / d, i = idx - j * d;
        if (sh.executed) {
            S[(long long)(a + i) + (long long)(a + j) * lds] = Sw[i + j * ld];
            T[(long long)(a + i) + (long long)(a + j) * ldt] = Tw[i + j * ld];
        }
        qw_pool[wd.qw_off + idx] = sh.executed ? Qw[i + j * ld] : (i == j ? 1.0 : 0.0);
        qw_pool[wd.qw_off + (long long)d * d + idx] = sh.executed ? Zw[i + j * ld] : (i == j ? 1.0 : 0.0);
    }
    if (tid < nb) {
        order_pool[wd.blk_off + tid] = sh.executed ? sh.arr[tid] : (uint8_t)tid;
        stuck_pool[wd.blk_off + tid] = sh.executed ? sh.bstuck[tid] : 0;
    }
    if (tid == 0) {
        int32_t st = sh.executed ? kWinExecuted : (sh.skipped ? kWinSkipped : 0);
        if (sh.executed)
            for (int b = 0; b < nb; ++b)
                if (sh.bstuck[b]) st |= kWinStuck;
        status[blockIdx.x] = st;
        if (dev_level && ((st & kWinStuck) || !(st & (kWinExecuted | kWinSkipped)))) atomicMin(dev_level, wd.level);
    }
}

size_t gwindow_smem_bytes(int d) {
    const size_t ld = (size_t)(d | 1);
    return ((sizeof(GShared) + 15) & ~size_t(15)) + 4 * ld * d * sizeof(double);
}

cudaError_t launch_gwindow_reorder(const WinDesc* wins, int nwin, int dmax, double* S, long long lds, double* T,
                                   long long ldt, double* qw_pool, const uint8_t* sizes_pool,
                                   const uint8_t* sel_pool, uint8_t* order_pool, uint8_t* stuck_pool,
                                   int32_t* status, cudaStream_t stream, int32_t* dev_level) {
    if (nwin <= 0) return cudaSuccess;
    if (dmax > kGMaxD) return cudaErrorInvalidValue;
    {
        cudaError_t e = ensure_dyn_smem((const void*)gwindow_reorder_kernel, gwindow_smem_bytes(kGMaxD));
        if (e != cudaSuccess) return e;
    }
    gwindow_reorder_kernel<<<nwin, kGThreads, gwindow_smem_bytes(dmax), stream>>>(
        wins, S, lds, T, ldt, qw_pool, sizes_pool, sel_pool, order_pool, stuck_pool, status, dev_level);
    return cudaGetLastError();
}

}  // namespace teig
