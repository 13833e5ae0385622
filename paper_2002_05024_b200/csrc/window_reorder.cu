// window_reorder.cu -- batched single-CTA window-reorder kernel (sm_100a).
//
// Device restatement of `window_reorder` (reference reorder.cpp:124-194) and
// `kernels::swap_adjacent_blocks` (kernels.cpp:510-631): every CTA owns one
// diagonal window [a, a+d) of S, gathers it into shared memory (packed upper
// Hessenberg, see window_kernels.cuh), bubbles the window's selected blocks
// to its top with adjacent swaps -- preserving their order, stopping a block
// whose swap is rejected -- accumulates the d x d orthogonal Q_w in shared
// memory, scatters the window back and publishes Q_w for the update kernels.
//
// One launch processes all windows of one wavefront (level); they are
// disjoint along the diagonal, so the CTAs are independent.
#include <cuda_runtime.h>

#include "device_types.h"
#include "launch.h"
#include "window_kernels.cuh"

namespace teig {

constexpr int kWinThreads = 128;

__global__ void __launch_bounds__(kWinThreads, 1)
window_reorder_kernel(const WinDesc* __restrict__ wins, double* __restrict__ S, long long lds,
                      double* __restrict__ qw_pool, const uint8_t* __restrict__ sizes_pool,
                      const uint8_t* __restrict__ sel_pool, uint8_t* __restrict__ order_pool,
                      uint8_t* __restrict__ stuck_pool, int32_t* __restrict__ status) {
    extern __shared__ __align__(16) double smem[];
    const WinDesc wd = wins[blockIdx.x];
    const int d = wd.d, nb = wd.nb;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* w = smem;                              // packed window
    const int wpacked = d * (d + 3) / 2;
    double* acc = smem + ((wpacked + 1) & ~1);     // d x d
    uint8_t* arr = reinterpret_cast<uint8_t*>(acc + d * d);      // arrangement (nb)
    uint8_t* bsz = arr + 256;                                    // block sizes
    int* flag = reinterpret_cast<int*>(bsz + 256);

    const double* Sa = S + (long long)wd.a + (long long)wd.a * lds;
    // gather: column j keeps rows 0..min(j+1, d-1)
    for (int j = warp; j < d; j += kWinThreads / 32) {
        const int len = min(j + 2, d);
        const double* src = Sa + (long long)j * lds;
        double* dst = w + pk(0, j);
        for (int i = lane; i < len; i += 32) dst[i] = src[i];
    }
    for (int idx = tid; idx < d * d; idx += kWinThreads) acc[idx] = ((idx % d) == (idx / d)) ? 1.0 : 0.0;
    for (int k = tid; k < nb; k += kWinThreads) {
        arr[k] = (uint8_t)k;
        bsz[k] = sizes_pool[wd.blk_off + k];
    }
    __syncthreads();

    if (warp == 0) {
        WinView v{w, acc, d};
        // layout check against the exact-zero subdiagonal (reorder.cpp:132-154)
        bool ok = true;
        {
            int row = 0;
            for (int k = 0; k < nb && ok; ++k) {
                const int sz = bsz[k];
                if (row + sz > d) ok = false;
                else if (sz == 2 && v.W(row + 1, row) == 0.0) ok = false;
                else if (row + sz < d && v.W(row + sz, row + sz - 1) != 0.0) ok = false;
                row += sz;
            }
            if (ok && row != d) ok = false;
        }
        int st = 0;
        if (ok) {
            st = kWinExecuted;
            const uint8_t* sel = sel_pool + wd.blk_off;
            uint8_t* stuck = stuck_pool + wd.blk_off;
            int dest = 0;
            for (int blk = 0; blk < nb; ++blk) {
                if (lane == 0) stuck[blk] = 0;
                if (!sel[blk]) continue;
                int slot = 0, row = 0;
                while (arr[slot] != blk) row += bsz[arr[slot++]];
                bool stk = false;
                while (slot > dest) {
                    const int pred = arr[slot - 1];
                    const int prow = row - bsz[pred];
                    if (!swap_adjacent(v, prow, bsz[pred], bsz[blk], lane)) {
                        stk = true;
                        break;
                    }
                    __syncwarp();
                    if (lane == 0) {
                        arr[slot - 1] = (uint8_t)blk;
                        arr[slot] = (uint8_t)pred;
                    }
                    __syncwarp();
                    row = prow;
                    --slot;
                }
                if (stk) {
                    if (lane == 0) stuck[blk] = 1;
                    st |= kWinStuck;
                }
                dest = slot + 1;
            }
        }
        if (lane == 0) *flag = st;
    }
    __syncthreads();
    const int st = *flag;
    if (st & kWinExecuted) {
        double* dst0 = S + (long long)wd.a + (long long)wd.a * lds;
        for (int j = warp; j < d; j += kWinThreads / 32) {
            const int len = min(j + 2, d);
            double* dst = dst0 + (long long)j * lds;
            const double* src = w + pk(0, j);
            for (int i = lane; i < len; i += 32) dst[i] = src[i];
        }
        for (int k = tid; k < nb; k += kWinThreads) order_pool[wd.blk_off + k] = arr[k];
    }
    double* qw = qw_pool + wd.qw_off;
    for (int idx = tid; idx < d * d; idx += kWinThreads) qw[idx] = acc[idx];
    if (tid == 0) status[blockIdx.x] = st;
}

size_t window_reorder_smem_bytes(int dmax) {
    const size_t wpacked = (size_t)dmax * (dmax + 3) / 2;
    return (((wpacked + 1) & ~size_t(1)) + (size_t)dmax * dmax) * sizeof(double) + 512 + 16;
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
