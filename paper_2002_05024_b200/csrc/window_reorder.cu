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
// commute, so a step needs only two barrier-separated phases:
//   1. decisions (warps 0-3, one thread per pair, warps specialised by
//      block-size type: Givens for 1x1|1x1, register-resident direct swap
//      otherwise)  ||  the accumulator update of the PREVIOUS step
//      (warps 4-7; Q_w never feeds a decision, so it lags one step);
//   2. the window update of this step (warps 1-7): every element above or
//      right of a pair's block receives M_A^T (its row pair) and M_B (its
//      column pair) in one pass -- a cell shared by a row pair and a column
//      pair is transformed jointly, so no row/column phase split is needed
//      --  ||  warp 0 commits the arrangement and finds the next step's
//      pairs (pair state is double buffered).
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
    int8_t owner[3][kMaxBlocks]; // row/col index -> pair owning it (-1: none), per buffer
    int16_t acc_lo[kMaxBlocks];  // nonzero row range of each ACC column
    int16_t acc_hi[kMaxBlocks];
    int16_t srow[kMaxBlocks + 1];
    PairRec pairs[3][kMaxPairs];   // pair state of steps t-1, t, t+1 (index step % 3)
    int16_t type_list[3][4][kMaxPairs];
    int type_cnt[3][4];
    int npairs[3];
    int status;
    int redo;
    double M[2][kMaxPairs][16];  // row-major D x D, window <- M^T W M
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

// Warp 0: row starts of the slots and all adjacent (unselected, selected &
// not stuck) pairs of the current arrangement, into buffer `buf`.
__device__ __forceinline__ void find_pairs(WinShared& sh, int nb, int d, int buf, int lane) {
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
    if (lane < 4) sh.type_cnt[buf][lane] = 0;
    for (int i = lane; i < d; i += 32) sh.owner[buf][i] = -1;
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
            sh.pairs[buf][idx] = pr;
            for (int k = 0; k < pr.p + pr.q; ++k) sh.owner[buf][pr.pos + k] = (int8_t)idx;
            const int t = atomicAdd(&sh.type_cnt[buf][ty], 1);
            sh.type_list[buf][ty][t] = (int16_t)idx;
        }
        np += __popc(m);
    }
    if (lane == 0) sh.npairs[buf] = np;
    __syncwarp();
}

// x (D values) times M (row-major D x D): y_j = sum_k x_k M[k][j]
template <int D>
__device__ __forceinline__ void vec_mat(const double* x, const double* M, double* y) {
#pragma unroll
    for (int j = 0; j < D; ++j) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) s += x[k] * M[k * D + j];
        y[j] = s;
    }
}
// M^T x: y_i = sum_k M[k][i] x_k
template <int D>
__device__ __forceinline__ void matT_vec(const double* M, const double* x, double* y) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) s += M[k * D + i] * x[k];
        y[i] = s;
    }
}

// ACC[:, pos:pos+D] <- ACC[:, pos:pos+D] M for the pairs of buffer `buf`.
// One warp per pair (warp-uniform D, M in registers), lanes over the rows of
// the union of the columns' nonzero row ranges (ACC starts as I; a column's
// support only grows by mixing with its pair partner).
template <int D>
__device__ __forceinline__ void acc_pair(WinShared& sh, double* acc, int d, const double* Ms, int pos, int lane) {
    double M[D * D];
#pragma unroll
    for (int i = 0; i < D * D; ++i) M[i] = Ms[i];
    int lo = sh.acc_lo[pos], hi = sh.acc_hi[pos];
#pragma unroll
    for (int j = 1; j < D; ++j) {
        lo = min(lo, (int)sh.acc_lo[pos + j]);
        hi = max(hi, (int)sh.acc_hi[pos + j]);
    }
    double* c0 = acc + pos * d;
    for (int r = lo + lane; r <= hi; r += 32) {
        double x[D], y[D];
#pragma unroll
        for (int j = 0; j < D; ++j) x[j] = c0[r + j * d];
        vec_mat<D>(x, M, y);
#pragma unroll
        for (int j = 0; j < D; ++j) c0[r + j * d] = y[j];
    }
    __syncwarp();
    if (lane < D) {
        sh.acc_lo[pos + lane] = (int16_t)lo;
        sh.acc_hi[pos + lane] = (int16_t)hi;
    }
}

__device__ __forceinline__ void acc_update(WinShared& sh, double* acc, int d, int buf, int mbuf, int w0, int nw, int warp, int lane) {
    const int np = sh.npairs[buf];
    for (int pi = warp - w0; pi < np; pi += nw) {
        const PairRec pr = sh.pairs[buf][pi];
        if (!pr.ok) continue;
        const int D = pr.p + pr.q;
        const double* M = sh.M[mbuf][pi];
        if (D == 2) acc_pair<2>(sh, acc, d, M, pr.pos, lane);
        else if (D == 3) acc_pair<3>(sh, acc, d, M, pr.pos, lane);
        else acc_pair<4>(sh, acc, d, M, pr.pos, lane);
    }
}

// Rows of pair A: W[A, c] <- M_A^T W[A, c] for every column c right of A's
// block (lanes over columns).
template <int DA>
__device__ __forceinline__ void rows_pair(double* w, int d, int posA, const double* MAs, int lane) {
    double MA[DA * DA];
#pragma unroll
    for (int i = 0; i < DA * DA; ++i) MA[i] = MAs[i];
    for (int c = posA + DA + lane; c < d; c += 32) {
        double* col = w + pk(posA, c);
        double x[DA], y[DA];
#pragma unroll
        for (int i = 0; i < DA; ++i) x[i] = col[i];
        matT_vec<DA>(MA, x, y);
#pragma unroll
        for (int i = 0; i < DA; ++i) col[i] = y[i];
    }
}
// Columns of pair B: W[r, B] <- W[r, B] M_B for every row r above B's block
// (lanes over rows), then B's new diagonal block.
template <int DB>
__device__ __forceinline__ void cols_pair(double* w, int posB, const double* MBs, const double* Bblk, int lane) {
    double MB[DB * DB];
#pragma unroll
    for (int i = 0; i < DB * DB; ++i) MB[i] = MBs[i];
    for (int r = lane; r < posB; r += 32) {
        double x[DB], y[DB];
#pragma unroll
        for (int j = 0; j < DB; ++j) x[j] = w[pk(r, posB + j)];
        vec_mat<DB>(x, MB, y);
#pragma unroll
        for (int j = 0; j < DB; ++j) w[pk(r, posB + j)] = y[j];
    }
    if (lane < DB * DB) {
        const int i = lane / DB, j = lane % DB;
        if (i <= j + 1) w[pk(posB + i, posB + j)] = Bblk[i * DB + j];
    }
}

__device__ __forceinline__ void rows_phase(WinShared& sh, double* w, int d, int buf, int mbuf, int warp, int lane, int nw) {
    const int np = sh.npairs[buf];
    for (int pi = warp; pi < np; pi += nw) {
        const PairRec pa = sh.pairs[buf][pi];
        if (!pa.ok) continue;
        const int D = pa.p + pa.q;
        const double* M = sh.M[mbuf][pi];
        if (D == 2) rows_pair<2>(w, d, pa.pos, M, lane);
        else if (D == 3) rows_pair<3>(w, d, pa.pos, M, lane);
        else rows_pair<4>(w, d, pa.pos, M, lane);
    }
}

__device__ __forceinline__ void cols_phase(WinShared& sh, double* w, int buf, int mbuf, int warp, int lane, int nw) {
    const int np = sh.npairs[buf];
    for (int pi = warp; pi < np; pi += nw) {
        const PairRec pb = sh.pairs[buf][pi];
        if (!pb.ok) continue;
        const int D = pb.p + pb.q;
        const double* M = sh.M[mbuf][pi];
        if (D == 2) cols_pair<2>(w, pb.pos, M, sh.B[pi], lane);
        else if (D == 3) cols_pair<3>(w, pb.pos, M, sh.B[pi], lane);
        else cols_pair<4>(w, pb.pos, M, sh.B[pi], lane);
    }
}

__global__ void __launch_bounds__(kWinThreads, 1)
window_reorder_kernel(const WinDesc* __restrict__ wins, double* __restrict__ S, long long lds,
                      double* __restrict__ qw_pool, const uint8_t* __restrict__ sizes_pool,
                      const uint8_t* __restrict__ sel_pool, uint8_t* __restrict__ order_pool,
                      uint8_t* __restrict__ stuck_pool, int32_t* __restrict__ status,
                      unsigned long long* __restrict__ prof, int32_t* __restrict__ dev_level) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // optional per-warp phase timing (prof != nullptr): [warp][0] phase-1
    // busy cycles, [1] phase-2 busy cycles, [2] steps, [3] kernel cycles
    unsigned long long t_p1 = 0, t_p2 = 0, n_steps = 0;
    const unsigned long long t_k0 = clock64();
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
    for (int k = tid; k < d; k += kWinThreads) {
        sh.acc_lo[k] = (int16_t)k;
        sh.acc_hi[k] = (int16_t)k;
    }
    for (int k = tid; k < nb; k += kWinThreads) {
        sh.arr[k] = (uint8_t)k;
        sh.bsz[k] = sizes_pool[wd.blk_off + k];
        sh.bsel[k] = sel_pool[wd.blk_off + k];
        sh.bstuck[k] = 0;
    }
    if (tid == 0) sh.npairs[0] = sh.npairs[1] = sh.npairs[2] = 0;
    __syncthreads();
    if (warp == 0) {
        // layout check against the exact-zero subdiagonal (reorder.cpp:132-154)
        bool ok = true;
        if (lane == 0) {
            // an earlier level deviated: this window's planned layout is stale
            const bool skip = dev_level && __ldcg(dev_level) < wd.level;
            ok = !skip;
            int row = 0;
            for (int k = 0; k < nb && ok; ++k) {
                const int sz = sh.bsz[k];
                if (row + sz > d) ok = false;
                else if (sz == 2 && w[pk(row + 1, row)] == 0.0) ok = false;
                else if (row + sz < d && w[pk(row + sz, row + sz - 1)] != 0.0) ok = false;
                row += sz;
            }
            if (ok && row != d) ok = false;
            sh.status = ok ? kWinExecuted : (skip ? kWinSkipped : 0);
        }
        ok = __shfl_sync(0xffffffffu, ok, 0);
        if (ok) find_pairs(sh, nb, d, 0, lane);
    }
    __syncthreads();
    const bool executed = sh.status & kWinExecuted;

    if (executed) {
        int cur = 0, mb = 0;  // pair-state buffer (step % 3), M buffer (step % 2)
        bool have_prev = false;
        if (tid == 0) sh.redo = 0;
        __syncthreads();
        for (;;) {
            const int np = sh.npairs[cur];
            const int nxt = (cur + 1) % 3, prv = (cur + 2) % 3;
            const unsigned long long c0 = clock64();
            // ---- phase 1: decisions of this step || accumulator of the previous
            // step; warp 0 also commits the arrangement assuming every swap of
            // the step succeeds and finds the next step's pairs from it ----
            if (warp < 4) {
                const int cnt = sh.type_cnt[cur][warp];
                for (int k = lane; k < cnt; k += 32) {
                    const int pi = sh.type_list[cur][warp][k];
                    PairRec& pr = sh.pairs[cur][pi];
                    if (warp == 0) decide_givens(w, pr, sh.M[mb][pi], sh.B[pi]);
                    else if (warp == 1) decide_direct<1, 2>(w, pr, sh.M[mb][pi], sh.B[pi]);
                    else if (warp == 2) decide_direct<2, 1>(w, pr, sh.M[mb][pi], sh.B[pi]);
                    else decide_direct<2, 2>(w, pr, sh.M[mb][pi], sh.B[pi]);
                }
                if (warp == 0) {
                    for (int pi = lane; pi < np; pi += 32) {
                        const int s = sh.pairs[cur][pi].slot;
                        const uint8_t t = sh.arr[s];
                        sh.arr[s] = sh.arr[s + 1];
                        sh.arr[s + 1] = t;
                    }
                    __syncwarp();
                    find_pairs(sh, nb, d, nxt, lane);
                }
            } else if (have_prev) {
                acc_update(sh, acc, d, prv, mb ^ 1, 4, NW - 4, warp, lane);
            }
            const unsigned long long c1 = clock64();
            __syncthreads();
            const unsigned long long c2 = clock64();
            // ---- phase 2a: rows of every accepted pair ----
            rows_phase(sh, w, d, cur, mb, warp, lane, NW);
            if (lane == 0) {
                for (int pi = warp; pi < np; pi += NW)
                    if (!sh.pairs[cur][pi].ok) sh.redo = 1;
            }
            __syncthreads();
            // ---- phase 2b: columns + new diagonal blocks; rare fix-up of a
            // rejected swap (undo it in the arrangement, stop the block, redo
            // the next step's pairs) ----
            cols_phase(sh, w, cur, mb, warp, lane, NW);
            if (sh.redo && warp == 0) {
                if (lane == 0) {
                    for (int pi = 0; pi < np; ++pi) {
                        const PairRec pr = sh.pairs[cur][pi];
                        if (pr.ok) continue;
                        const int s = pr.slot;
                        const uint8_t t = sh.arr[s];  // undo the optimistic swap
                        sh.arr[s] = sh.arr[s + 1];
                        sh.arr[s + 1] = t;
                        sh.bstuck[sh.arr[s + 1]] = 1;
                        sh.status |= kWinStuck;
                    }
                    sh.redo = 0;
                }
                __syncwarp();
                find_pairs(sh, nb, d, nxt, lane);
            }
            const unsigned long long c3 = clock64();
            __syncthreads();
            t_p1 += c1 - c0;
            t_p2 += c3 - c2;
            ++n_steps;
            have_prev = true;
            cur = nxt;
            mb ^= 1;
            if (sh.npairs[cur] == 0) break;
        }
        // accumulator of the last step
        acc_update(sh, acc, d, (cur + 2) % 3, mb ^ 1, 0, NW, warp, lane);
        __syncthreads();
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
    if (tid == 0) {
        status[blockIdx.x] = st;
        // a rejected swap or a layout mismatch: later levels' plans are stale
        if (dev_level && ((st & kWinStuck) || !(st & (kWinExecuted | kWinSkipped)))) atomicMin(dev_level, wd.level);
    }
    if (prof && lane == 0) {
        unsigned long long* pw = prof + (blockIdx.x * (size_t)NW + warp) * 4;
        pw[0] = t_p1;
        pw[1] = t_p2;
        pw[2] = n_steps;
        pw[3] = clock64() - t_k0;
    }
}

size_t window_reorder_smem_bytes(int dmax) {
    const size_t wpacked = (size_t)dmax * (dmax + 3) / 2;
    return ((sizeof(WinShared) + 15) & ~size_t(15)) + (((wpacked + 1) & ~size_t(1)) + (size_t)dmax * dmax) * sizeof(double);
}

cudaError_t launch_window_reorder(const WinDesc* wins, int nwin, int dmax, double* S, long long lds,
                                  double* qw_pool, const uint8_t* sizes_pool, const uint8_t* sel_pool,
                                  uint8_t* order_pool, uint8_t* stuck_pool, int32_t* status,
                                  cudaStream_t stream, unsigned long long* prof, int32_t* dev_level) {
    if (nwin <= 0) return cudaSuccess;
    const size_t smem = window_reorder_smem_bytes(dmax);
    {
        cudaError_t e = ensure_dyn_smem((const void*)window_reorder_kernel, window_reorder_smem_bytes(128));
        if (e != cudaSuccess) return e;
    }
    window_reorder_kernel<<<nwin, kWinThreads, smem, stream>>>(wins, S, lds, qw_pool, sizes_pool, sel_pool,
                                                               order_pool, stuck_pool, status, prof, dev_level);
    return cudaGetLastError();
}

}  // namespace teig
