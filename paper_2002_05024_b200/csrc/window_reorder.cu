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
    int8_t owner[2][kMaxBlocks]; // row/col index -> pair owning it (-1: none), per buffer
    int16_t srow[kMaxBlocks + 1];
    PairRec pairs[2][kMaxPairs];
    int16_t type_list[2][4][kMaxPairs];
    int type_cnt[2][4];
    int npairs[2];
    int status;
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

// ACC[:, pos:pos+D] <- ACC[:, pos:pos+D] M for the pairs of buffer `buf`,
// threads [t0, t0+nt) of the CTA
__device__ __forceinline__ void acc_update(const WinShared& sh, double* acc, int d, int buf, int t0, int nt, int tid) {
    const int np = sh.npairs[buf];
    for (int item = tid - t0; item < np * d; item += nt) {
        const int pi = item / d, r = item - pi * d;
        const PairRec pr = sh.pairs[buf][pi];
        if (!pr.ok) continue;
        const int D = pr.p + pr.q;
        double* c0 = acc + r + pr.pos * d;
        double x[4], y[4];
        const double* M = sh.M[buf][pi];
        if (D == 2) {
            x[0] = c0[0]; x[1] = c0[d];
            vec_mat<2>(x, M, y);
            c0[0] = y[0]; c0[d] = y[1];
        } else if (D == 3) {
            x[0] = c0[0]; x[1] = c0[d]; x[2] = c0[2 * d];
            vec_mat<3>(x, M, y);
            c0[0] = y[0]; c0[d] = y[1]; c0[2 * d] = y[2];
        } else {
            x[0] = c0[0]; x[1] = c0[d]; x[2] = c0[2 * d]; x[3] = c0[3 * d];
            vec_mat<4>(x, M, y);
            c0[0] = y[0]; c0[d] = y[1]; c0[2 * d] = y[2]; c0[3 * d] = y[3];
        }
    }
}

// W[r, A] <- W[r, A] M_A for one row r above A's block
template <int DA>
__device__ __forceinline__ void upd_row(double* w, int r, int posA, const double* MA) {
    double x[DA], y[DA];
#pragma unroll
    for (int j = 0; j < DA; ++j) x[j] = w[pk(r, posA + j)];
    vec_mat<DA>(x, MA, y);
#pragma unroll
    for (int j = 0; j < DA; ++j) w[pk(r, posA + j)] = y[j];
}
// W[A, c] <- M_A^T W[A, c] for one column c right of A's block
template <int DA>
__device__ __forceinline__ void upd_col(double* w, int c, int posA, const double* MA) {
    double* col = w + pk(0, c) + posA;
    double x[DA], y[DA];
#pragma unroll
    for (int i = 0; i < DA; ++i) x[i] = col[i];
    matT_vec<DA>(MA, x, y);
#pragma unroll
    for (int i = 0; i < DA; ++i) col[i] = y[i];
}
// joint cell W[A, B] <- M_A^T W[A, B] M_B
template <int DA, int DB>
__device__ __forceinline__ void upd_joint(double* w, int posA, int posB, const double* MA, const double* MB) {
    double t[DA][DB];
#pragma unroll
    for (int j = 0; j < DB; ++j) {
        double cx[DA], cy[DA];
        const double* col = w + pk(0, posB + j) + posA;
#pragma unroll
        for (int i = 0; i < DA; ++i) cx[i] = col[i];
        matT_vec<DA>(MA, cx, cy);
#pragma unroll
        for (int i = 0; i < DA; ++i) t[i][j] = cy[i];
    }
#pragma unroll
    for (int i = 0; i < DA; ++i) {
        double ry[DB];
        vec_mat<DB>(t[i], MB, ry);
#pragma unroll
        for (int j = 0; j < DB; ++j) w[pk(posA + i, posB + j)] = ry[j];
    }
}
template <int DA>
__device__ __forceinline__ void upd_joint_a(double* w, int posA, int posB, int DB, const double* MA, const double* MB) {
    if (DB == 2) upd_joint<DA, 2>(w, posA, posB, MA, MB);
    else if (DB == 3) upd_joint<DA, 3>(w, posA, posB, MA, MB);
    else upd_joint<DA, 4>(w, posA, posB, MA, MB);
}

// Window update of one step (see the header): warps [1, NW) of the CTA.
__device__ __forceinline__ void window_update(WinShared& sh, double* w, int d, int buf, int warp, int lane, int nwarps) {
    const int np = sh.npairs[buf];
    for (int pi = warp - 1; pi < np; pi += nwarps - 1) {
        const PairRec pa = sh.pairs[buf][pi];
        if (!pa.ok) continue;
        const int DA = pa.p + pa.q, posA = pa.pos;
        const double* MA = sh.M[buf][pi];
        const int nitems = d - DA;  // rows [0, posA) then columns [posA+DA, d)
        for (int k = lane; k < nitems; k += 32) {
            if (k < posA) {
                // row k, columns of A (a row owned by another swapping pair is
                // handled there as a joint cell)
                const int ow = sh.owner[buf][k];
                if (ow >= 0 && sh.pairs[buf][ow].ok) continue;
                if (DA == 2) upd_row<2>(w, k, posA, MA);
                else if (DA == 3) upd_row<3>(w, k, posA, MA);
                else upd_row<4>(w, k, posA, MA);
            } else {
                const int c = k + DA;  // column right of A's block
                const int ob = sh.owner[buf][c];
                if (ob >= 0 && sh.pairs[buf][ob].ok) {
                    const PairRec pb = sh.pairs[buf][ob];
                    if (c != pb.pos) continue;  // the cell is handled at B's first column
                    const int DB = pb.p + pb.q;
                    const double* MB = sh.M[buf][ob];
                    if (DA == 2) upd_joint_a<2>(w, posA, c, DB, MA, MB);
                    else if (DA == 3) upd_joint_a<3>(w, posA, c, DB, MA, MB);
                    else upd_joint_a<4>(w, posA, c, DB, MA, MB);
                } else {
                    if (DA == 2) upd_col<2>(w, c, posA, MA);
                    else if (DA == 3) upd_col<3>(w, c, posA, MA);
                    else upd_col<4>(w, c, posA, MA);
                }
            }
        }
        if (lane < DA * DA) {
            const int i = lane / DA, j = lane % DA;
            if (i <= j + 1) w[pk(posA + i, posA + j)] = sh.B[pi][i * DA + j];
        }
    }
}

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
    if (tid == 0) sh.npairs[0] = sh.npairs[1] = 0;
    __syncthreads();
    if (warp == 0) {
        // layout check against the exact-zero subdiagonal (reorder.cpp:132-154)
        bool ok = true;
        if (lane == 0) {
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
        ok = __shfl_sync(0xffffffffu, ok, 0);
        if (ok) find_pairs(sh, nb, d, 0, lane);
    }
    __syncthreads();
    const bool executed = sh.status & kWinExecuted;

    if (executed) {
        int cur = 0;
        bool have_prev = false;
        for (;;) {
            const int np = sh.npairs[cur];
            // ---- phase 1: decisions of this step || accumulator of the previous step ----
            if (warp < 4) {
                const int cnt = sh.type_cnt[cur][warp];
                for (int k = lane; k < cnt; k += 32) {
                    const int pi = sh.type_list[cur][warp][k];
                    PairRec& pr = sh.pairs[cur][pi];
                    if (warp == 0) decide_givens(w, pr, sh.M[cur][pi], sh.B[pi]);
                    else if (warp == 1) decide_direct<1, 2>(w, pr, sh.M[cur][pi], sh.B[pi]);
                    else if (warp == 2) decide_direct<2, 1>(w, pr, sh.M[cur][pi], sh.B[pi]);
                    else decide_direct<2, 2>(w, pr, sh.M[cur][pi], sh.B[pi]);
                }
            } else if (have_prev) {
                acc_update(sh, acc, d, cur ^ 1, 4 * 32, kWinThreads - 4 * 32, tid);
            }
            __syncthreads();
            // ---- phase 2: window update || commit arrangement + next pairs ----
            if (warp == 0) {
                if (lane == 0) {
                    for (int pi = 0; pi < np; ++pi) {
                        const PairRec pr = sh.pairs[cur][pi];
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
                __syncwarp();
                find_pairs(sh, nb, d, cur ^ 1, lane);
            } else {
                window_update(sh, w, d, cur, warp, lane, NW);
            }
            __syncthreads();
            have_prev = true;
            cur ^= 1;
            if (sh.npairs[cur] == 0) break;
        }
        // accumulator of the last step
        acc_update(sh, acc, d, cur ^ 1, 0, kWinThreads, tid);
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
