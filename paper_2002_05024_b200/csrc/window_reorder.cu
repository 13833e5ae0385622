// window_reorder.cu -- batched single-CTA window-reorder kernel (sm_100a).
//
// Device restatement of `window_reorder` (reference reorder.cpp:124-194):
// every CTA owns one diagonal window [a, a+d) of S (d <= 128), gathers it
// into shared memory (packed upper Hessenberg), moves the window's selected
// blocks to its top -- preserving the order among selected and among
// unselected blocks, stopping a block whose swap is rejected -- accumulates
// the d x d orthogonal Q_w in shared memory, scatters the window back and
// publishes Q_w for the update kernels.
//
// The reference bubbles one selected block at a time (a chain of dependent
// swaps, ~2000 per 128-wide window).  Here the swaps are scheduled as a
// parallel odd-even transposition: at every step ALL adjacent
// (unselected, selected) block pairs swap at once.  Such pairs never share a
// block, their similarity transformations act on disjoint index sets and
// commute, so the step is applied in three barrier-separated phases:
//   1. decision  -- one thread per pair evaluates its swap (Givens for 1x1 |
//                   1x1, register-resident direct swap otherwise; warps are
//                   specialised by block-size type, no divergence);
//   2. rows      -- M^T applied to each pair's rows right of its block;
//   3. columns   -- M applied to each pair's columns above its block, and to
//                   the pair's accumulator columns; the new diagonal block
//                   is written; the arrangement is updated.
// Every (unselected, selected) pair is swapped exactly once, as in the
// reference, and the final block order is identical; the depth drops from
// #swaps to ~#blocks.  Results agree with the reference to rounding (the
// swaps interleave differently), which the parity tests bound.
#include <cuda_runtime.h>

#include "device_types.h"
#include "launch.h"
#include "swap_math.cuh"

namespace teig {

namespace {

constexpr int kWinThreads = 256;
constexpr int kMaxBlocks = 128;
constexpr int kMaxPairs = 64;

__device__ __forceinline__ int pk(int i, int j) { return j * (j + 3) / 2 + i; }  // packed, i <= j+1

struct PairRec {
    int16_t pos;   // first row of the upper block
    int8_t p, q;   // upper (unselected) / lower (selected) block sizes
    int8_t slot;   // slot of the upper block
    int8_t ok;     // decision outcome
    int16_t pad;
};

struct WinShared {
    uint8_t arr[kMaxBlocks];     // arrangement: slot -> local block id
    uint8_t bsz[kMaxBlocks];     // block id -> size
    uint8_t bsel[kMaxBlocks];    // block id -> selected
    uint8_t bstuck[kMaxBlocks];  // block id -> rejected (stops moving)
    int16_t srow[kMaxBlocks + 1];
    PairRec pairs[kMaxPairs];
    int16_t type_list[4][kMaxPairs];
    int type_cnt[4];
    int npairs;
    int status;
    double M[kMaxPairs][16];     // row-major D x D, window <- M^T W M
    double B[kMaxPairs][16];     // new diagonal block, row-major D x D
};

template <int P, int Q>
__device__ __forceinline__ void decide_direct(const double* w, PairRec& pr, double* Mo, double* Bo) {
    constexpr int D = P + Q;
    double blk[D][D], M[D][D], nbk[D][D];
    const int pos = pr.pos;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) blk[i][j] = (i <= j + 1) ? w[pk(pos + i, pos + j)] : 0.0;
    const bool ok = direct_swap<P, Q>(blk, M, nbk);
    pr.ok = ok ? 1 : 0;
    if (ok) {
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) {
                Mo[i * D + j] = M[i][j];
                Bo[i * D + j] = nbk[i][j];
            }
    }
}

__device__ __forceinline__ void decide_givens(const double* w, PairRec& pr, double* Mo, double* Bo) {
    // reference kernels.cpp:515-527: Givens(t12, t22 - t11); t12 preserved
    const int pos = pr.pos;
    const double t11 = w[pk(pos, pos)], t12 = w[pk(pos, pos + 1)], t22 = w[pk(pos + 1, pos + 1)];
    double c, s;
    const double b = t22 - t11;
    if (b == 0.0) {
        c = 1.0;
        s = 0.0;
    } else if (t12 == 0.0) {
        c = 0.0;
        s = 1.0;
    } else {
        const double r = hypot(t12, b);
        c = t12 / r;
        s = b / r;
    }
    pr.ok = 1;
    if (t12 == 0.0 && b == 0.0) {  // equal values: no-op swap
        Mo[0] = 1.0; Mo[1] = 0.0; Mo[2] = 0.0; Mo[3] = 1.0;
        Bo[0] = t11; Bo[1] = t12; Bo[2] = 0.0; Bo[3] = t22;
        return;
    }
    Mo[0] = c; Mo[1] = -s; Mo[2] = s; Mo[3] = c;
    Bo[0] = t22; Bo[1] = t12; Bo[2] = 0.0; Bo[3] = t11;
}

}  // namespace

__global__ void __launch_bounds__(kWinThreads, 1)
window_reorder_kernel(const WinDesc* __restrict__ wins, double* __restrict__ S, long long lds,
                      double* __restrict__ qw_pool, const uint8_t* __restrict__ sizes_pool,
                      const uint8_t* __restrict__ sel_pool, uint8_t* __restrict__ order_pool,
                      uint8_t* __restrict__ stuck_pool, int32_t* __restrict__ status) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WinShared& sh = *reinterpret_cast<WinShared*>(smem_raw);
    double* w = reinterpret_cast<double*>(smem_raw + ((sizeof(WinShared) + 15) & ~size_t(15)));
    const WinDesc wd = wins[blockIdx.x];
    const int d = wd.d, nb = wd.nb;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = kWinThreads / 32;
    const int wpacked = d * (d + 3) / 2;
    double* acc = w + ((wpacked + 1) & ~1);

    // gather: column j keeps rows 0..min(j+1, d-1)
    const double* Sa = S + (long long)wd.a + (long long)wd.a * lds;
    for (int j = warp; j < d; j += NW) {
        const int len = min(j + 2, d);
        const double* src = Sa + (long long)j * lds;
        double* dst = w + pk(0, j);
        for (int i = lane; i < len; i += 32) dst[i] = src[i];
    }
    for (int idx = tid; idx < d * d; idx += kWinThreads) acc[idx] = ((idx % d) == (idx / d)) ? 1.0 : 0.0;
    for (int k = tid; k < nb; k += kWinThreads) {
        sh.arr[k] = (uint8_t)k;
        sh.bsz[k] = sizes_pool[wd.blk_off + k];
        sh.bsel[k] = sel_pool[wd.blk_off + k];
        sh.bstuck[k] = 0;
    }
    __syncthreads();
    if (tid == 0) {
        // layout check against the exact-zero subdiagonal (reorder.cpp:132-154)
        bool ok = true;
        int row = 0;
        for (int k = 0; k < nb && ok; ++k) {
            const int sz = sh.bsz[k];
            if (row + sz > d) ok = false;
            else if (sz == 2 && w[pk(row + 1, row)] == 0.0) ok = false;
            else if (row + sz < d && w[pk(row + sz, row + sz - 1)] != 0.0) ok = false;
            row += sz;
        }
        if (ok && row != d) ok = false;
        sh.status = ok ? kWinExecuted : 0;
    }
    __syncthreads();
    const bool executed = sh.status & kWinExecuted;

    if (executed) {
        for (;;) {
            // ---- find all adjacent (unselected, selected & not stuck) pairs ----
            if (warp == 0) {
                // row starts of the slots: per-lane chunk of 4 slots + warp scan
                int loc[4], sum = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int s = lane * 4 + k;
                    loc[k] = (s < nb) ? sh.bsz[sh.arr[s]] : 0;
                    sum += loc[k];
                }
                int incl = sum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += t;
                }
                int r = incl - sum;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int s = lane * 4 + k;
                    if (s < nb) sh.srow[s] = (int16_t)r;
                    r += loc[k];
                }
                if (lane == 31) sh.srow[nb] = (int16_t)incl;
                __syncwarp();
                if (lane < 4) sh.type_cnt[lane] = 0;
                __syncwarp();
                int np = 0;
                for (int base = 0; base < nb; base += 32) {
                    const int s = base + lane;
                    bool cand = false;
                    int ty = 0;
                    if (s + 1 < nb) {
                        const int u = sh.arr[s], b = sh.arr[s + 1];
                        cand = !sh.bsel[u] && sh.bsel[b] && !sh.bstuck[b];
                        ty = (sh.bsz[u] == 2 ? 2 : 0) + (sh.bsz[b] == 2 ? 1 : 0);
                    }
                    const unsigned m = __ballot_sync(0xffffffffu, cand);
                    if (cand) {
                        const int idx = np + __popc(m & ((1u << lane) - 1u));
                        PairRec pr;
                        pr.pos = sh.srow[s];
                        pr.p = (int8_t)sh.bsz[sh.arr[s]];
                        pr.q = (int8_t)sh.bsz[sh.arr[s + 1]];
                        pr.slot = (int8_t)s;
                        pr.ok = 0;
                        pr.pad = 0;
                        sh.pairs[idx] = pr;
                        const int t = atomicAdd(&sh.type_cnt[ty], 1);
                        sh.type_list[ty][t] = (int16_t)idx;
                    }
                    np += __popc(m);
                }
                if (lane == 0) sh.npairs = np;
            }
            __syncthreads();
            const int np = sh.npairs;
            if (np == 0) break;

            // ---- 1. decisions: warp t handles pair type t ----
            if (warp < 4) {
                const int cnt = sh.type_cnt[warp];
                for (int k = lane; k < cnt; k += 32) {
                    const int pi = sh.type_list[warp][k];
                    PairRec& pr = sh.pairs[pi];
                    if (warp == 0) decide_givens(w, pr, sh.M[pi], sh.B[pi]);
                    else if (warp == 1) decide_direct<1, 2>(w, pr, sh.M[pi], sh.B[pi]);
                    else if (warp == 2) decide_direct<2, 1>(w, pr, sh.M[pi], sh.B[pi]);
                    else decide_direct<2, 2>(w, pr, sh.M[pi], sh.B[pi]);
                }
            }
            __syncthreads();

            // ---- 2. rows: W[pos:pos+D, c] <- M^T W[pos:pos+D, c], c >= pos+D ----
            for (int pi = warp; pi < np; pi += NW) {
                const PairRec pr = sh.pairs[pi];
                if (!pr.ok) continue;
                const int D = pr.p + pr.q, pos = pr.pos;
                const double* M = sh.M[pi];
                for (int c = pos + D + lane; c < d; c += 32) {
                    double* col = w + pk(0, c) + pos;
                    if (D == 2) {
                        const double x0 = col[0], x1 = col[1];
                        col[0] = M[0] * x0 + M[2] * x1;
                        col[1] = M[1] * x0 + M[3] * x1;
                    } else if (D == 3) {
                        const double x0 = col[0], x1 = col[1], x2 = col[2];
                        col[0] = M[0] * x0 + M[3] * x1 + M[6] * x2;
                        col[1] = M[1] * x0 + M[4] * x1 + M[7] * x2;
                        col[2] = M[2] * x0 + M[5] * x1 + M[8] * x2;
                    } else {
                        const double x0 = col[0], x1 = col[1], x2 = col[2], x3 = col[3];
                        col[0] = M[0] * x0 + M[4] * x1 + M[8] * x2 + M[12] * x3;
                        col[1] = M[1] * x0 + M[5] * x1 + M[9] * x2 + M[13] * x3;
                        col[2] = M[2] * x0 + M[6] * x1 + M[10] * x2 + M[14] * x3;
                        col[3] = M[3] * x0 + M[7] * x1 + M[11] * x2 + M[15] * x3;
                    }
                }
            }
            __syncthreads();

            // ---- 3. columns above the block, accumulator columns, new block ----
            for (int pi = warp; pi < np; pi += NW) {
                const PairRec pr = sh.pairs[pi];
                if (!pr.ok) continue;
                const int D = pr.p + pr.q, pos = pr.pos;
                const double* M = sh.M[pi];
                // rows [0, pos) of W then rows [0, d) of ACC
                for (int r = lane; r < pos + d; r += 32) {
                    double* c0;
                    int stride_is_acc = r >= pos;
                    double x[4];
                    if (!stride_is_acc) {
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            if (j < D) x[j] = w[pk(r, pos + j)];
                    } else {
                        const int ra = r - pos;
                        c0 = acc + ra + pos * d;
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            if (j < D) x[j] = c0[j * d];
                    }
                    double y[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (j >= D) continue;
                        double s = 0.0;
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            if (k < D) s += x[k] * M[k * D + j];
                        y[j] = s;
                    }
                    if (!stride_is_acc) {
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            if (j < D) w[pk(r, pos + j)] = y[j];
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            if (j < D) c0[j * d] = y[j];
                    }
                }
                if (lane < D * D) {
                    const int i = lane / D, j = lane % D;
                    if (i <= j + 1) w[pk(pos + i, pos + j)] = sh.B[pi][i * D + j];
                }
            }
            if (tid == 0) {
                for (int pi = 0; pi < np; ++pi) {
                    const PairRec pr = sh.pairs[pi];
                    const int s = pr.slot;
                    if (pr.ok) {
                        const uint8_t t = sh.arr[s];
                        sh.arr[s] = sh.arr[s + 1];
                        sh.arr[s + 1] = t;
                    } else {
                        sh.bstuck[sh.arr[s + 1]] = 1;
                        sh.status |= kWinStuck;
                    }
                }
            }
            __syncthreads();
        }
    }

    const int st = sh.status;
    if (st & kWinExecuted) {
        double* dst0 = S + (long long)wd.a + (long long)wd.a * lds;
        for (int j = warp; j < d; j += NW) {
            const int len = min(j + 2, d);
            double* dst = dst0 + (long long)j * lds;
            const double* src = w + pk(0, j);
            for (int i = lane; i < len; i += 32) dst[i] = src[i];
        }
        for (int k = tid; k < nb; k += kWinThreads) {
            order_pool[wd.blk_off + k] = sh.arr[k];
            stuck_pool[wd.blk_off + k] = sh.bstuck[k];
        }
    }
    double* qw = qw_pool + wd.qw_off;
    for (int idx = tid; idx < d * d; idx += kWinThreads) qw[idx] = acc[idx];
    if (tid == 0) status[blockIdx.x] = st;
}

size_t window_reorder_smem_bytes(int dmax) {
    const size_t wpacked = (size_t)dmax * (dmax + 3) / 2;
    return ((sizeof(WinShared) + 15) & ~size_t(15)) + (((wpacked + 1) & ~size_t(1)) + (size_t)dmax * dmax) * sizeof(double);
}

cudaError_t launch_window_reorder(const WinDesc* wins, int nwin, int dmax, double* S, long long lds,
                                  double* qw_pool, const uint8_t* sizes_pool, const uint8_t* sel_pool,
                                  uint8_t* order_pool, uint8_t* stuck_pool, int32_t* status,
                                  cudaStream_t stream) {
    if (nwin <= 0) return cudaSuccess;
    const size_t smem = window_reorder_smem_bytes(dmax);
    static size_t configured = 0;
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(window_reorder_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    window_reorder_kernel<<<nwin, kWinThreads, smem, stream>>>(wins, S, lds, qw_pool, sizes_pool, sel_pool,
                                                               order_pool, stuck_pool, status);
    return cudaGetLastError();
}

}  // namespace teig
