// dgemm.cuh -- general FP64 GEMM on the tensor pipe for the dense phases
// (back-transformation, Hessenberg trailing / accumulator updates):
//   C = beta C + alpha op(A) op(B),   op(X) = X or X^T, column-major, any ld,
// beta in {0, 1}.  sm_100a: mma.sync.m8n8k4.f64 -> DMMA.8x8x4.
//
// One CTA owns a 128 x 64 tile of C and streams K through a 3-stage cp.async
// ring in chunks of 32 (8-byte copies: arbitrary leading dimensions and
// offsets; edges zero-filled by cp.async's src-size operand).  Shared tiles
// keep M (resp. N) contiguous with a leading dimension = 4 (mod 16) doubles:
// the m8n8k4 fragment loads are bank-conflict free.  The global loads walk
// the operand's contiguous dimension (M for A = N, K for A = T; K for B = N,
// N for B = T).  8 warps of 32 x 32 (4 x 4 DMMA tiles each).
#pragma once
#include <cuda_runtime.h>

namespace teig {
namespace dg {

constexpr int BM = 128, BN = 64, KC = 32, ST = 3, NT = 256;
constexpr int LDA = BM + 4;  // As[kk][m]
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

// gridDim.z > 1 (split K): slice z multiplies the K range [z*kz, (z+1)*kz)
// and writes its partial product to C + z*cz (beta must be 0; a fixed-order
// reduction of the slices follows, dgemm_reduce)
template <bool TA, bool TB>
__global__ void __launch_bounds__(NT) gemm_kernel(int m, int n, int kdim, double alpha, const double* __restrict__ A,
                                                  long long lda, const double* __restrict__ B, long long ldb,
                                                  double beta, double* __restrict__ C, long long ldc, int kz,
                                                  long long cz) {
    if (gridDim.z > 1) {
        const int z = blockIdx.z, k0 = z * kz;
        A += TA ? (long long)k0 : (long long)k0 * lda;
        B += TB ? (long long)k0 * ldb : (long long)k0;
        C += (long long)z * cz;
        kdim = min(kz, kdim - k0);
    }
    extern __shared__ __align__(16) double sm[];
    double* As = sm;                  // ST x KC x LDA   (As[kk * LDA + mm] = op(A)(m0+mm, k0+kk))
    double* Bs = sm + ST * KC * LDA;  // ST x BN x LDB   (Bs[nn * LDB + kk] = op(B)(k0+kk, n0+nn))
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    const int wm = warp & 3, wn = warp >> 2;
    const int nk = (kdim + KC - 1) / KC;

    auto load = [&](int stage, int kc) {
        const int k0 = kc * KC;
        double* as = As + stage * KC * LDA;
        double* bs = Bs + stage * BN * LDB;
        for (int idx = tid; idx < KC * BM; idx += NT) {
            int kk, mm;
            if (!TA) { kk = idx / BM; mm = idx % BM; }   // contiguous along m
            else { mm = idx / KC; kk = idx % KC; }       // contiguous along k
            const int gm = m0 + mm, gk = k0 + kk;
            const bool v = gm < m && gk < kdim;
            const double* src = TA ? A + gk + (long long)gm * lda : A + gm + (long long)gk * lda;
            cp8(as + kk * LDA + mm, v ? (const void*)src : (const void*)A, v);
        }
        for (int idx = tid; idx < BN * KC; idx += NT) {
            int kk, nn;
            if (!TB) { nn = idx / KC; kk = idx % KC; }   // contiguous along k
            else { kk = idx / BN; nn = idx % BN; }       // contiguous along n
            const int gn = n0 + nn, gk = k0 + kk;
            const bool v = gn < n && gk < kdim;
            const double* src = TB ? B + gn + (long long)gk * ldb : B + gk + (long long)gn * ldb;
            cp8(bs + nn * LDB + kk, v ? (const void*)src : (const void*)B, v);
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
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (c + h >= n) continue;
                double* dst = C + r + (long long)(c + h) * ldc;
                *dst = (beta != 0.0 ? *dst : 0.0) + alpha * acc[i][j][h];
            }
        }
    }
}

// C = beta C + alpha sum_z P[z] (z ascending: deterministic)
__global__ void dgemm_reduce(int m, int n, int nz, double alpha, const double* __restrict__ P, long long ldp,
                             long long pz, double beta, double* __restrict__ C, long long ldc) {
    const long long tot = (long long)m * n;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(t % m), j = (int)(t / m);
        double s = 0.0;
        for (int z = 0; z < nz; ++z) s += P[(long long)z * pz + i + (long long)j * ldp];
        double* dst = C + i + (long long)j * ldc;
        *dst = (beta != 0.0 ? *dst : 0.0) + alpha * s;
    }
}

}  // namespace dg
}  // namespace teig
