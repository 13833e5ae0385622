// backtransform.cu -- eigenvector back-transformation X = Q * Y on the FP64
// tensor pipe (sm_100a: mma.sync.m8n8k4.f64 -> DMMA.8x8x4) plus the
// reference's per-column renormalisation (reference
// eigvec.cpp:448-516).
//
// Q (n x n) is the orthogonal factor a reorder / Schur call left in HBM, Y
// (n x k) the eigenvectors of the (reordered) Schur form: X = Q Y is a plain
// dense contraction, 2 n^2 k flops over 8 (n^2 + 2 n k) bytes, tensor-bound
// for k >~ 12: the DMMA GEMM of dgemm.cuh (also used by the Hessenberg
// reduction's trailing updates).
//
// Renormalisation (eigvec.cpp:494-512): every real eigenvector column, and
// every complex pair (real part, imaginary part), is scaled by sign(lead) /
// max_i |x_i| (pairs: max_i max(|re_i|, |im_i|)), lead = the entry at the
// FIRST index attaining the maximum (the imaginary part's if it is larger in
// magnitude there).  One CTA per column / pair: a first-index arg-max
// reduction, then the scale pass.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "dgemm.cuh"
#include "launch.h"

namespace teig {

namespace {

// one CTA per column (kind 0) or pair (kind 1); kind 2 columns are handled
// with their pair's first column; every other value leaves the column as is
constexpr int RT = 256;
__global__ void __launch_bounds__(RT) renorm_kernel(int n, double* __restrict__ X, long long ldx,
                                                    const int8_t* __restrict__ kind, int k, int* __restrict__ nonfinite) {
    const int j = blockIdx.x;
    if (j >= k) return;
    const int kd = kind ? kind[j] : -1;
    double* x = X + (long long)j * ldx;
    if (kd == 2) return;       // the pair's second column: its first column's CTA handles it
    if (kd != 0 && kd != 1) {  // not renormalised: finiteness only
        bool bad = false;
        for (int i = threadIdx.x; i < n; i += RT) bad |= !isfinite(x[i]);
        if (bad) atomicOr(nonfinite, 1);
        return;
    }
    const bool pair = kd == 1 && j + 1 < k;
    double* y = pair ? x + ldx : nullptr;
    // arg-max of |x_i| (pairs: max(|x_i|, |y_i|)), FIRST index on ties
    double best = 0.0;
    int arg = 0x7fffffff;
    bool bad = false;
    for (int i = threadIdx.x; i < n; i += RT) {
        double v = fabs(x[i]);
        if (pair) v = fmax(v, fabs(y[i]));
        bad |= !isfinite(v);
        if (v > best) {  // strictly greater: the thread keeps its first index
            best = v;
            arg = i;
        }
    }
    if (__syncthreads_or(bad)) {  // assert_finite (eigvec.cpp:485)
        if (threadIdx.x == 0) atomicOr(nonfinite, 1);
        return;
    }
    __shared__ double sb[RT / 32];
    __shared__ int sa[RT / 32];
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_down_sync(0xffffffffu, best, o);
        const int oa = __shfl_down_sync(0xffffffffu, arg, o);
        if (ob > best || (ob == best && oa < arg)) {
            best = ob;
            arg = oa;
        }
    }
    if ((threadIdx.x & 31) == 0) {
        sb[threadIdx.x >> 5] = best;
        sa[threadIdx.x >> 5] = arg;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < RT / 32; ++w)
            if (sb[w] > best || (sb[w] == best && sa[w] < arg)) {
                best = sb[w];
                arg = sa[w];
            }
        sb[0] = best;
        sa[0] = arg;
    }
    __syncthreads();
    best = sb[0];
    arg = sa[0];
    if (best == 0.0) return;
    double lead = x[arg];
    if (pair && fabs(y[arg]) > fabs(lead)) lead = y[arg];
    const double scale = (lead < 0.0 ? -1.0 : 1.0) / best;
    for (int i = threadIdx.x; i < n; i += RT) {
        x[i] *= scale;
        if (pair) y[i] *= scale;
    }
}

}  // namespace

cudaError_t launch_dgemm(bool ta, bool tb, int m, int n, int kdim, double alpha, const double* A, long long lda,
                         const double* B, long long ldb, double beta, double* C, long long ldc, cudaStream_t s,
                         double* work, size_t work_doubles) {
    if (m <= 0 || n <= 0) return cudaSuccess;
    dim3 grid((m + dg::BM - 1) / dg::BM, (n + dg::BN - 1) / dg::BN);
    // split K when the output has too few tiles to fill the GPU and K is long
    // (the Hessenberg panel products V^T G, A V: 64 columns, thousands of K)
    int kz = kdim;
    double* Cout = C;
    long long ldo = ldc, cz = 0;
    const long long tiles = (long long)grid.x * grid.y;
    if (work && tiles < 2 * 148 && kdim >= 1024) {
        int splits = (int)std::min<long long>(16, (2 * 148 + tiles - 1) / tiles);
        splits = std::min(splits, kdim / 256);
        kz = (((kdim + splits - 1) / splits) + dg::KC - 1) / dg::KC * dg::KC;
        splits = (kdim + kz - 1) / kz;
        if (splits > 1 && (size_t)splits * m * n <= work_doubles) {
            grid.z = splits;
            Cout = work;
            ldo = m;
            cz = (long long)m * n;
        } else {
            kz = kdim;
        }
    }
    const double a1 = grid.z > 1 ? 1.0 : alpha, b1 = grid.z > 1 ? 0.0 : beta;
    cudaError_t e = cudaSuccess;
#define TEIG_DG(TA, TB)                                                                                       \
    e = ensure_dyn_smem((const void*)dg::gemm_kernel<TA, TB>, dg::kSmem);                                      \
    if (e != cudaSuccess) return e;                                                                            \
    dg::gemm_kernel<TA, TB><<<grid, dg::NT, dg::kSmem, s>>>(m, n, kdim, a1, A, lda, B, ldb, b1, Cout, ldo, kz, cz);
    if (!ta && !tb) {
        TEIG_DG(false, false)
    } else if (!ta && tb) {
        TEIG_DG(false, true)
    } else if (ta && !tb) {
        TEIG_DG(true, false)
    } else {
        TEIG_DG(true, true)
    }
#undef TEIG_DG
    if (grid.z > 1) {
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        const long long tot = (long long)m * n;
        dg::dgemm_reduce<<<(unsigned)std::min<long long>((tot + 255) / 256, 4096), 256, 0, s>>>(
            m, n, (int)grid.z, alpha, work, m, cz, beta, C, ldc);
    }
    return cudaGetLastError();
}

cudaError_t launch_renorm_columns(int n, double* X, long long ldx, const int8_t* kind_dev, int k, int* nonfinite,
                                  cudaStream_t s) {
    if (n <= 0 || k <= 0) return cudaSuccess;
    renorm_kernel<<<k, RT, 0, s>>>(n, X, ldx, kind_dev, k, nonfinite);
    return cudaGetLastError();
}

}  // namespace teig
