// backtransform.cu -- eigenvector back-transformation X = Q * Y on the FP64
// tensor pipe (sm_100a: mma.sync.m8n8k4.f64 -> DMMA.8x8x4) plus the
// reference's per-column renormalisation (reference
// eigvec.cpp:448-516).
//
// Q (n x n) is the orthogonal factor a reorder / Schur call left in HBM, Y
// (n x k) the eigenvectors of the (reordered) Schur form: X = Q Y is a plain
// dense contraction, 2 n^2 k flops over 8 (n^2 + 2 n k) bytes, tensor-bound
// for k >~ 12.  One CTA owns a 128 x 64 tile of X and streams the K = n
// extent through a 3-stage cp.async ring in chunks of 32 (8-byte copies:
// arbitrary leading dimensions and offsets; edges zero-filled by cp.async's
// src-size operand); shared tiles use leading dimensions = 4 (mod 16)
// doubles so the m8n8k4 fragment loads are bank-conflict free; 8 warps of
// 32 x 32 (4 x 4 DMMA tiles each).
//
// Renormalisation (eigvec.cpp:494-512): every real eigenvector column, and
// every complex pair (real part, imaginary part), is scaled by sign(lead) /
// max_i |x_i| (pairs: max_i max(|re_i|, |im_i|)), lead = the entry at the
// FIRST index attaining the maximum (the imaginary part's if it is larger in
// magnitude there).  One CTA per column / pair: a first-index arg-max
// reduction, then the scale pass.
#include <cuda_runtime.h>

#include <cstdint>

#include "launch.h"

namespace teig {

namespace {

constexpr int BM = 128, BN = 64, KC = 32, ST = 3, NT = 256;
constexpr int LDA = BM + 4;  // As[kk][m], = 4 (mod 16)
constexpr int LDB = KC + 4;  // Bs[n][kk]
constexpr size_t kSmem = (size_t)ST * (KC * LDA + BN * LDB) * sizeof(double);

__device__ __forceinline__ void cp8(void* smem_dst, const void* gsrc, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gsrc), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// X[m0:m0+BM, n0:n0+BN] = Q[m0:, :] * Y[:, n0:]  (column-major, any ld)
__global__ void __launch_bounds__(NT) gemm_nn_kernel(int m, int n, int kdim, const double* __restrict__ A, long long lda,
                                                     const double* __restrict__ B, long long ldb, double* __restrict__ C,
                                                     long long ldc) {
    extern __shared__ __align__(16) double sm[];
    double* As = sm;                     // ST x KC x LDA
    double* Bs = sm + ST * KC * LDA;     // ST x BN x LDB
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    const int wm = warp & 3, wn = warp >> 2;  // 4 x 2 warps of 32 x 32
    const int nk = (kdim + KC - 1) / KC;

    auto load = [&](int stage, int kc) {
        const int k0 = kc * KC;
        double* as = As + stage * KC * LDA;
        double* bs = Bs + stage * BN * LDB;
        for (int idx = tid; idx < KC * BM; idx += NT) {  // coalesced along m
            const int kk = idx / BM, r = idx % BM;
            const bool v = (m0 + r < m) && (k0 + kk < kdim);
            cp8(as + kk * LDA + r, v ? (const void*)(A + (m0 + r) + (long long)(k0 + kk) * lda) : (const void*)A, v);
        }
        for (int idx = tid; idx < BN * KC; idx += NT) {  // coalesced along k
            const int nn = idx / KC, kk = idx % KC;
            const bool v = (n0 + nn < n) && (k0 + kk < kdim);
            cp8(bs + nn * LDB + kk, v ? (const void*)(B + (k0 + kk) + (long long)(n0 + nn) * ldb) : (const void*)B, v);
        }
    };

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
    for (int s = 0; s < ST - 1; ++s) {
        if (s < nk) load(s, s);
        cp_commit();
    }
    for (int kc = 0; kc < nk; ++kc) {
        cp_wait<ST - 2>();
        __syncthreads();
        const int nxt = kc + ST - 1;
        if (nxt < nk) load(nxt % ST, nxt);
        cp_commit();
        const double* as = As + (kc % ST) * KC * LDA;
        const double* bs = Bs + (kc % ST) * BN * LDB;
#pragma unroll
        for (int ks = 0; ks < KC; ks += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = as[(ks + tig) * LDA + wm * 32 + i * 8 + gid];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = bs[(wn * 32 + j * 8 + gid) * LDB + ks + tig];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
    }
    cp_wait<0>();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = m0 + wm * 32 + i * 8 + gid;
        if (r >= m) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = n0 + wn * 32 + j * 8 + 2 * tig;
            if (c < n) C[r + (long long)c * ldc] = acc[i][j][0];
            if (c + 1 < n) C[r + (long long)(c + 1) * ldc] = acc[i][j][1];
        }
    }
}

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

cudaError_t launch_gemm_nn(int m, int n, int kdim, const double* A, long long lda, const double* B, long long ldb,
                           double* C, long long ldc, cudaStream_t s) {
    if (m <= 0 || n <= 0) return cudaSuccess;
    cudaError_t e = ensure_dyn_smem((const void*)gemm_nn_kernel, kSmem);
    if (e != cudaSuccess) return e;
    const dim3 grid((m + BM - 1) / BM, (n + BN - 1) / BN);
    gemm_nn_kernel<<<grid, NT, kSmem, s>>>(m, n, kdim, A, lda, B, ldb, C, ldc);
    return cudaGetLastError();
}

cudaError_t launch_renorm_columns(int n, double* X, long long ldx, const int8_t* kind_dev, int k, int* nonfinite,
                                  cudaStream_t s) {
    if (n <= 0 || k <= 0) return cudaSuccess;
    renorm_kernel<<<k, RT, 0, s>>>(n, X, ldx, kind_dev, k, nonfinite);
    return cudaGetLastError();
}

}  // namespace teig
