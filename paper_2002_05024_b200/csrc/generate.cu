// generate.cu -- on-device synthetic inputs (product side, used by bench.py
// and the tests to build the SURVEY.md 8d workloads directly in HBM).
//
// Counter-based Philox4x32-10 (the reference's generator, philox.hpp:18-84)
// lets every element compute its own draw index, so the fill is bit-identical
// to the reference's sequential row-major stream:
//   * schur input: `default_spectrum` + `build_quasi_triangular`
//     (generate.cpp:68-91, 115-150) -- reals on [-10,10] first, then 2x2
//     blocks [[re, im], [-im, re]], strictly-upper fill uniform [-1, 1];
//   * random upper Hessenberg (generate.cpp:192-198).
#include <cuda_runtime.h>

#include <cstdint>

#include "launch.h"

namespace teig {

namespace {

__device__ __forceinline__ void philox10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
        const uint32_t n1 = (uint32_t)p1;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
        const uint32_t n3 = (uint32_t)p0;
        c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

// k-th uniform_sym draw of Philox(seed)
__device__ __forceinline__ double draw_uniform_sym(uint64_t seed, uint64_t k) {
    const uint64_t blk = k >> 1;
    uint32_t c[4] = {(uint32_t)blk, (uint32_t)(blk >> 32), 0u, 0u};
    philox10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const int i = (int)(k & 1);
    const uint64_t u = (((uint64_t)c[2 * i + 1] << 32) | c[2 * i]) >> 11;
    return __dsub_rn(__dmul_rn((double)u, 2.0 / 9007199254740992.0), 1.0);
}

// k-th uniform [0, 1) draw of Philox(seed)
__device__ __forceinline__ double draw_u01(uint64_t seed, uint64_t k) {
    const uint64_t blk = k >> 1;
    uint32_t c[4] = {(uint32_t)blk, (uint32_t)(blk >> 32), 0u, 0u};
    philox10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const int i = (int)(k & 1);
    const uint64_t u = (((uint64_t)c[2 * i + 1] << 32) | c[2 * i]) >> 11;
    return __dmul_rn((double)u, 1.0 / 9007199254740992.0);
}

// C5 input T ("T upper triangular with a positive diagonal,
// uniform [-1, 1] upper fill"; no reference generator exists): on the block
// pattern of the synthetic S (reals first, then 2x2 blocks), diagonal 1 + u
// (both entries of a 2x2 block share the first one's draw and the in-block
// T(p, p+1) is 0, so every 2x2 block of the pencil keeps its complex pair),
// strictly upper fill uniform_sym.  Entry (i, j) uses draw i*n + j.
__global__ void gen_pair_t_kernel(double* T, long long ldt, long long n, uint64_t seed) {
    const long long j = blockIdx.y;
    const long long npairs = n / 4, nreal = n - 2 * npairs;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double v = 0.0;
        const bool pair_first_i = i >= nreal && ((i - nreal) & 1) == 0;
        if (i == j) {
            const bool second = j >= nreal && ((j - nreal) & 1) == 1;
            const long long r = second ? i - 1 : i;
            v = __dadd_rn(1.0, draw_u01(seed, (uint64_t)(r * n + r)));
        } else if (j > i) {
            if (!(pair_first_i && j == i + 1)) {
                const uint64_t k = (uint64_t)(i * n + j);
                v = __dsub_rn(__dmul_rn(2.0, draw_u01(seed, k)), 1.0);
            }
        }
        T[i + j * ldt] = v;
    }
}

__global__ void gen_schur_kernel(double* S, long long lds, long long n, uint64_t seed, long long c0) {
    const long long j = c0 + blockIdx.y;  // columns [c0, c0 + gridDim.y) into S[:, 0..)
    const long long npairs = n / 4, nreal = n - 2 * npairs;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double v = 0.0;
        auto first_of_pair = [&](long long r) { return r >= nreal && ((r - nreal) & 1) == 0; };
        if (i == j) {
            if (i < nreal) {
                v = (nreal == 1) ? 1.0 : __dadd_rn(-10.0, __ddiv_rn(__dmul_rn(20.0, (double)i), (double)(nreal - 1)));
            } else {
                const long long k = (i - nreal) >> 1;
                v = (npairs == 1) ? 0.5 : __dadd_rn(-9.7, __ddiv_rn(__dmul_rn(19.4, (double)k), (double)(npairs - 1)));
            }
        } else if (i == j + 1) {
            if (first_of_pair(j)) {
                const long long k = (j - nreal) >> 1;
                v = -(1.0 + 2.0 * (double)(k % 3));
            }
        } else if (j > i) {
            if (j == i + 1 && first_of_pair(i)) {
                const long long k = (i - nreal) >> 1;
                v = 1.0 + 2.0 * (double)(k % 3);
            } else {
                // draws consumed by rows < i, then the position inside row i
                const long long before = i * (n - 1) - i * (i - 1) / 2 - (i > nreal ? (i - nreal + 1) / 2 : 0);
                long long inrow = j - i - 1;
                if (first_of_pair(i)) inrow -= 1;  // the in-block entry is not drawn
                v = draw_uniform_sym(seed, (uint64_t)(before + inrow));
            }
        }
        S[i + (j - c0) * lds] = v;
    }
}

// rows [r0, r1) of the n x n identity into Q (ld ldq): Q[i - r0, j]
__global__ void identity_rows_kernel(double* Q, long long ldq, long long r0, long long r1) {
    const long long j = blockIdx.y;
    for (long long i = r0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < r1; i += (long long)gridDim.x * blockDim.x)
        Q[(i - r0) + j * ldq] = (i == j) ? 1.0 : 0.0;
}

__global__ void identity_kernel(double* Q, long long ldq, long long n) {
    const long long j = blockIdx.y;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        Q[i + j * ldq] = (i == j) ? 1.0 : 0.0;
}

__global__ void gen_hess_kernel(double* H, long long ldh, long long n, uint64_t seed) {
    const long long j = blockIdx.y;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double v = 0.0;
        if (i <= j + 1) {
            long long before;
            if (i == 0) before = 0;
            else before = n + (i - 1) * (n + 1) - (i - 1) * i / 2;
            const long long inrow = j - (i == 0 ? 0 : i - 1);
            v = draw_uniform_sym(seed, (uint64_t)(before + inrow));
        }
        H[i + j * ldh] = v;
    }
}

dim3 grid_for(long long n) {
    const long long bx = (n + 255) / 256;
    return dim3((unsigned)(bx < 64 ? bx : 64), (unsigned)n);
}

}  // namespace

cudaError_t launch_gen_schur_input(double* S, long long lds, long long n, uint64_t fill_seed, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    gen_schur_kernel<<<grid_for(n), 256, 0, stream>>>(S, lds, n, fill_seed, 0);
    return cudaGetLastError();
}

cudaError_t launch_gen_pair_t(double* T, long long ldt, long long n, uint64_t seed, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    gen_pair_t_kernel<<<grid_for(n), 256, 0, stream>>>(T, ldt, n, seed);
    return cudaGetLastError();
}

cudaError_t launch_gen_schur_cols(double* S, long long lds, long long n, uint64_t fill_seed, long long c0,
                                  long long c1, cudaStream_t stream) {
    if (n <= 0 || c1 <= c0) return cudaSuccess;
    dim3 g = grid_for(n);
    g.y = (unsigned)(c1 - c0);
    gen_schur_kernel<<<g, 256, 0, stream>>>(S, lds, n, fill_seed, c0);
    return cudaGetLastError();
}

cudaError_t launch_identity_rows(double* Q, long long ldq, long long n, long long r0, long long r1,
                                 cudaStream_t stream) {
    if (n <= 0 || r1 <= r0) return cudaSuccess;
    dim3 g = grid_for(r1 - r0);
    g.y = (unsigned)n;
    identity_rows_kernel<<<g, 256, 0, stream>>>(Q, ldq, r0, r1);
    return cudaGetLastError();
}

cudaError_t launch_set_identity(double* Q, long long ldq, long long n, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    identity_kernel<<<grid_for(n), 256, 0, stream>>>(Q, ldq, n);
    return cudaGetLastError();
}

cudaError_t launch_gen_hessenberg(double* H, long long ldh, long long n, uint64_t seed, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    gen_hess_kernel<<<grid_for(n), 256, 0, stream>>>(H, ldh, n, seed * 0x9E3779B97F4A7C15ull + 4ull);
    return cudaGetLastError();
}

// Row support of every column: the first and last row holding a nonzero
// (bit pattern != 0: +0.0 is the only zero) -- the factor-support tracking of
// the reorder drivers (plan.h FactorSupport).  One CTA per column.
__global__ void column_support_kernel(const double* __restrict__ Q, long long ldq, int rows, int32_t* __restrict__ lo,
                                      int32_t* __restrict__ hi) {
    const long long c = blockIdx.x;
    const unsigned long long* col = reinterpret_cast<const unsigned long long*>(Q + c * ldq);
    int l = rows, h = -1;
    for (int r = threadIdx.x; r < rows; r += blockDim.x)
        if (col[r] != 0ull) {
            l = min(l, r);
            h = max(h, r);
        }
    for (int o = 16; o > 0; o >>= 1) {
        l = min(l, __shfl_xor_sync(0xffffffffu, l, o));
        h = max(h, __shfl_xor_sync(0xffffffffu, h, o));
    }
    __shared__ int sl[32], sh[32];
    if ((threadIdx.x & 31) == 0) {
        sl[threadIdx.x >> 5] = l;
        sh[threadIdx.x >> 5] = h;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            l = min(l, sl[w]);
            h = max(h, sh[w]);
        }
        lo[c] = l;
        hi[c] = h;
    }
}

cudaError_t launch_column_support(const double* Q, long long ldq, long long rows, long long cols, int32_t* lo,
                                  int32_t* hi, cudaStream_t stream) {
    if (cols <= 0) return cudaSuccess;
    column_support_kernel<<<(unsigned)cols, 256, 0, stream>>>(Q, ldq, (int)rows, lo, hi);
    return cudaGetLastError();
}

}  // namespace teig
