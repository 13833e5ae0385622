// update_dmma.cu -- off-diagonal window updates on the FP64 tensor pipe
// (sm_100a: mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4).
//
// For a window [a, b) with accumulated orthogonal Q_w (d x d):
//   left  (row panel):    S[a:b, b:n]  <- Q_w^T S[a:b, b:n]       (reference window_tasks.cpp:12-20)
//   right (column panel): S[0:a, a:b]  <- S[0:a, a:b] Q_w          (window_tasks.cpp:22-30)
//   factor:               Q[0:n, a:b]  <- Q[0:n, a:b] Q_w          (window_tasks.cpp:72-86)
// Every CTA owns one in-place output tile and the full K = d extent of its
// panel tile, so no other CTA reads what it overwrites.  The index ranges
// come from WinDesc (lc0/lc1, rr0/rr1, qr0/qr1) so the same kernels update a
// column slab or row slab of a distributed matrix.  One launch covers
// all windows of a wavefront: the CTA locates its window by binary search
// over the per-level tile prefix sums carried in WinDesc.
//
// Operands are streamed through shared memory in K-chunks of 32 with 8-byte
// cp.async (panel row offsets are arbitrary, so 16-byte alignment is not
// guaranteed) in a 2-stage pipeline (A/B on B200: KC=32 x 2 stages beat
// KC=16 x 3 stages by 1.5 % on C4; 128-wide tiles lost 10-15 % to occupancy
// and tails); shared tiles are column-major with a
// leading dimension = 4 (mod 16) doubles, which makes the m8n8k4 fragment
// loads bank-conflict free.  Edges (k >= d, rows/cols past the panel) are
// zero-filled by cp.async's src-size operand.
#include <cuda_runtime.h>

#include "device_types.h"
#include "launch.h"

namespace teig {

// DMMA instructions issued by the update kernels of this file (every warp adds
// its count once, at its end): the profiled drivers report executed flops
__device__ unsigned long long g_dmma_cp = 0;

namespace {

#ifndef TEIG_UPD_KC
#define TEIG_UPD_KC 32
#endif
#ifndef TEIG_UPD_STAGES
#define TEIG_UPD_STAGES 2
#endif
constexpr int KC = TEIG_UPD_KC;  // K chunk
constexpr int LDK = KC + 4;      // smem ld for K-contiguous tiles (= 4 mod 16 doubles)
constexpr int STAGES = TEIG_UPD_STAGES;
constexpr int kUpdThreads = 256;

__device__ __forceinline__ void cp8(void* smem_dst, const void* gsrc, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
    const int nbytes = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gsrc), "r"(nbytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// locate the window owning tile t of this launch: largest k with pref[k] <= t
// (serial binary search: log2(nwin) dependent global loads)
template <int Field>
__device__ __forceinline__ int find_window_serial(const WinDesc* wins, int nwin, int t) {
    int lo = 0, hi = nwin - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        const int p = Field == 0 ? wins[mid].tl_pref : (Field == 1 ? wins[mid].tr_pref : wins[mid].tq_pref);
        if (p <= t) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// the same, CTA-cooperative: every thread reads one window's prefix (one
// global round trip instead of ~log2(nwin) dependent ones); ends with a barrier
template <int Field>
__device__ __forceinline__ int find_window(const WinDesc* wins, int nwin, int t, int* sh) {
    if (nwin > kUpdThreads) return find_window_serial<Field>(wins, nwin, t);
    if (threadIdx.x == 0) *sh = 0;
    __syncthreads();
    if ((int)threadIdx.x < nwin) {
        const WinDesc& w = wins[threadIdx.x];
        const int p = Field == 0 ? w.tl_pref : (Field == 1 ? w.tr_pref : w.tq_pref);
        if (p <= t) atomicMax(sh, (int)threadIdx.x);
    }
    __syncthreads();
    return *sh;
}

}  // namespace

// ---------------------------------------------------------------------------
// LEFT: out(d x BN) = Q_w^T (d x d) * P(d x BN), P = S[a:a+d, c:c+BN]
//   A[i][k] = Q_w[k][i]  -> smem As[i][kk] = Q_w[(k0+kk) + i*d]   (ld LDK)
//   B[k][n] = P[k][n]    -> smem Bs[n][kk] = S[a+k0+kk, c+n]       (ld LDK)
template <int DMAX>
__global__ void __launch_bounds__(kUpdThreads)
update_left_kernel(const WinDesc* __restrict__ wins, int nwin, const double* __restrict__ qw_pool,
                   double* __restrict__ S, long long lds, int n) {
    constexpr int BN = kLeftBN;
    constexpr int WM = (DMAX == 128) ? 4 : 2;   // warps along M
    constexpr int WN = 8 / WM;                  // warps along N
    constexpr int MT = DMAX / WM / 8;           // 8x8 tiles per warp along M (4)
    constexpr int NT = BN / WN / 8;             // along N (4 or 2)
    extern __shared__ __align__(16) double dsm[];
    double (*As)[DMAX * LDK] = reinterpret_cast<double (*)[DMAX * LDK]>(dsm);
    double (*Bs)[BN * LDK] = reinterpret_cast<double (*)[BN * LDK]>(dsm + STAGES * DMAX * LDK);

    const int t = blockIdx.x;
    __shared__ int sh_win;
    const int wi = find_window<0>(wins, nwin, t, &sh_win);
    const WinDesc wd = wins[wi];
    const int d = wd.d, a = wd.a;
    const int c = wd.lc0 + (t - wd.tl_pref) * BN;
    const int ncols = min(BN, wd.lc1 - c);
    const double* Qw = qw_pool + wd.qw_off;
    double* P = S + (long long)a + (long long)c * lds;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    const int wm = warp % WM, wn = warp / WM;
    const int nk = (d + KC - 1) / KC;

    auto load_stage = [&](int stage, int kc) {
        const int k0 = kc * KC;
        // A: DMAX x KC  (i major, kk minor in smem)
        for (int idx = tid; idx < DMAX * KC; idx += kUpdThreads) {
            const int i = idx / KC, kk = idx % KC;
            const int k = k0 + kk;
            const bool v = (i < d) && (k < d);
            cp8(&As[stage][i * LDK + kk], v ? (const void*)(Qw + k + (long long)i * d) : (const void*)Qw, v);
        }
        for (int idx = tid; idx < BN * KC; idx += kUpdThreads) {
            const int nn = idx / KC, kk = idx % KC;
            const int k = k0 + kk;
            const bool v = (nn < ncols) && (k < d);
            cp8(&Bs[stage][nn * LDK + kk], v ? (const void*)(P + k + (long long)nn * lds) : (const void*)P, v);
        }
    };

    double acc[MT][NT][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nk) load_stage(s, s);
        cp_commit();
    }
    const int m_base = wm * (MT * 8);
    const int n_base = wn * (NT * 8);
    const bool warp_active = m_base < d;
    int nlive = 0;  // executed fragment rows (DMMA count / NT)
    for (int kc = 0; kc < nk; ++kc) {
        cp_wait<STAGES - 2>();
        __syncthreads();
        const int nxt = kc + STAGES - 1;
        if (nxt < nk) load_stage(nxt % STAGES, nxt);
        cp_commit();
        const double* as = As[kc % STAGES];
        const double* bs = Bs[kc % STAGES];
        if (warp_active) {
#pragma unroll
            for (int ks = 0; ks < KC; ks += 4) {
                double af[MT], bf[NT];
#pragma unroll
                for (int i = 0; i < MT; ++i) af[i] = as[(m_base + i * 8 + gid) * LDK + ks + tig];
#pragma unroll
                for (int j = 0; j < NT; ++j) bf[j] = bs[(n_base + j * 8 + gid) * LDK + ks + tig];
                // all-zero 8x4 fragments of Q_w^T contribute exact zeros: skip
                // them (warp-uniform vote; the sums start at +0, bitwise equal)
                unsigned live = 0;
#pragma unroll
                for (int i = 0; i < MT; ++i) live |= (__any_sync(0xffffffffu, af[i] != 0.0) ? 1u : 0u) << i;
                nlive += __popc(live);
#pragma unroll
                for (int i = 0; i < MT; ++i)
                    if (live >> i & 1u)
#pragma unroll
                        for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
            }
        }
    }
    cp_wait<0>();
    if (warp_active && (threadIdx.x & 31) == 0) atomicAdd(&g_dmma_cp, (unsigned long long)nlive * NT);
    // all K of this CTA's panel tile has been consumed: write in place
    if (warp_active) {
#pragma unroll
        for (int i = 0; i < MT; ++i) {
            const int r = m_base + i * 8 + gid;
            if (r >= d) continue;
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                const int cc = n_base + j * 8 + 2 * tig;
                if (cc < ncols) P[r + (long long)cc * lds] = acc[i][j][0];
                if (cc + 1 < ncols) P[r + (long long)(cc + 1) * lds] = acc[i][j][1];
            }
        }
    }
}

// ---------------------------------------------------------------------------
// RIGHT: out(BM x d) = P(BM x d) * Q_w(d x d), P = M[r:r+BM, a:a+d]
//   A[r][k] = P[r][k]   -> smem As[kk][r] = M[r0+r, a+k0+kk]  (ld BM+4)
//   B[k][n] = Q_w[k][n] -> smem Bs[n][kk] = Q_w[(k0+kk) + n*d] (ld LDK)
// Field selects the prefix (1: S column panel rows [0,a); 2: factor rows [0,n)).
template <int DMAX, int Field>
__global__ void __launch_bounds__(kUpdThreads)
update_right_kernel(const WinDesc* __restrict__ wins, int nwin, const double* __restrict__ qw_pool,
                    double* __restrict__ M, long long ldm, int nrows_total) {
    constexpr int BM = kRightBM;
    constexpr int LDM = BM + 4;
    constexpr int WM = 2, WN = 4;
    constexpr int MT = BM / WM / 8;     // 4
    constexpr int NT = DMAX / WN / 8;   // 4 or 2
    extern __shared__ __align__(16) double dsm[];
    double (*As)[KC * LDM] = reinterpret_cast<double (*)[KC * LDM]>(dsm);
    double (*Bs)[DMAX * LDK] = reinterpret_cast<double (*)[DMAX * LDK]>(dsm + STAGES * KC * LDM);

    const int t = blockIdx.x;
    __shared__ int sh_win;
    const int wi = find_window<Field>(wins, nwin, t, &sh_win);
    const WinDesc wd = wins[wi];
    const int d = wd.d, a = wd.a;
    const int pref = (Field == 1) ? wd.tr_pref : wd.tq_pref;
    const int r0 = ((Field == 1) ? wd.rr0 : wd.qr0) + (t - pref) * BM;
    const int row_end = (Field == 1) ? wd.rr1 : wd.qr1;
    const int nrows = min(BM, row_end - r0);
    const double* Qw = qw_pool + wd.qw_off;
    double* P = M + (long long)r0 + (long long)a * ldm;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    const int wm = warp % WM, wn = warp / WM;
    const int nk = (d + KC - 1) / KC;

    auto load_stage = [&](int stage, int kc) {
        const int k0 = kc * KC;
        for (int idx = tid; idx < KC * BM; idx += kUpdThreads) {
            const int kk = idx / BM, r = idx % BM;
            const int k = k0 + kk;
            const bool v = (r < nrows) && (k < d);
            cp8(&As[stage][kk * LDM + r], v ? (const void*)(P + r + (long long)k * ldm) : (const void*)P, v);
        }
        for (int idx = tid; idx < DMAX * KC; idx += kUpdThreads) {
            const int nn = idx / KC, kk = idx % KC;
            const int k = k0 + kk;
            const bool v = (nn < d) && (k < d);
            cp8(&Bs[stage][nn * LDK + kk], v ? (const void*)(Qw + k + (long long)nn * d) : (const void*)Qw, v);
        }
    };

    double acc[MT][NT][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nk) load_stage(s, s);
        cp_commit();
    }
    const int m_base = wm * (MT * 8);
    const int n_base = wn * (NT * 8);
    const bool warp_active = (n_base < d) && (m_base < nrows);
    int nlive = 0;  // executed fragment columns (DMMA count / MT)
    for (int kc = 0; kc < nk; ++kc) {
        cp_wait<STAGES - 2>();
        __syncthreads();
        const int nxt = kc + STAGES - 1;
        if (nxt < nk) load_stage(nxt % STAGES, nxt);
        cp_commit();
        const double* as = As[kc % STAGES];
        const double* bs = Bs[kc % STAGES];
        if (warp_active) {
#pragma unroll
            for (int ks = 0; ks < KC; ks += 4) {
                double af[MT], bf[NT];
#pragma unroll
                for (int i = 0; i < MT; ++i) af[i] = as[(ks + tig) * LDM + m_base + i * 8 + gid];
#pragma unroll
                for (int j = 0; j < NT; ++j) bf[j] = bs[(n_base + j * 8 + gid) * LDK + ks + tig];
                unsigned live = 0;  // zero Q_w fragments skipped, as in the left kernel
#pragma unroll
                for (int j = 0; j < NT; ++j) live |= (__any_sync(0xffffffffu, bf[j] != 0.0) ? 1u : 0u) << j;
                nlive += __popc(live);
#pragma unroll
                for (int j = 0; j < NT; ++j)
                    if (live >> j & 1u)
#pragma unroll
                        for (int i = 0; i < MT; ++i) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
            }
        }
    }
    cp_wait<0>();
    if (warp_active && (threadIdx.x & 31) == 0) atomicAdd(&g_dmma_cp, (unsigned long long)nlive * MT);
    if (warp_active) {
#pragma unroll
        for (int i = 0; i < MT; ++i) {
            const int r = m_base + i * 8 + gid;
            if (r >= nrows) continue;
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                const int cc = n_base + j * 8 + 2 * tig;
                if (cc < d) P[r + (long long)cc * ldm] = acc[i][j][0];
                if (cc + 1 < d) P[r + (long long)(cc + 1) * ldm] = acc[i][j][1];
            }
        }
    }
}

template <typename K>
static cudaError_t set_smem(K kernel, size_t bytes) {
    return ensure_dyn_smem((const void*)kernel, bytes);
}

constexpr size_t left_smem(int dmax) { return (size_t)STAGES * (dmax * LDK + kLeftBN * LDK) * sizeof(double); }
constexpr size_t right_smem(int dmax) { return (size_t)STAGES * (KC * (kRightBM + 4) + dmax * LDK) * sizeof(double); }

cudaError_t launch_update_left(const WinDesc* wins, int nwin, int ntiles, int dmax, const double* qw_pool,
                               double* S, long long lds, int n, cudaStream_t stream, long long rows, long long cols,
                               int max_ctas) {
    if (ntiles <= 0) return cudaSuccess;
    if (rows > 0) {
        cudaError_t err;
        if (launch_update_left_tma(wins, nwin, ntiles, dmax, qw_pool, S, lds, rows, cols, stream, &err, max_ctas))
            return err;
    }
    {
        cudaError_t e = set_smem(update_left_kernel<64>, left_smem(64));
        if (e == cudaSuccess) e = set_smem(update_left_kernel<128>, left_smem(128));
        if (e != cudaSuccess) return e;
    }
    if (dmax <= 64)
        update_left_kernel<64><<<ntiles, kUpdThreads, left_smem(64), stream>>>(wins, nwin, qw_pool, S, lds, n);
    else
        update_left_kernel<128><<<ntiles, kUpdThreads, left_smem(128), stream>>>(wins, nwin, qw_pool, S, lds, n);
    return cudaGetLastError();
}

cudaError_t launch_update_right(const WinDesc* wins, int nwin, int ntiles, int dmax, const double* qw_pool,
                                double* M, long long ldm, int nrows_total, bool factor, cudaStream_t stream,
                                long long rows, long long cols, bool short_ctas, int max_ctas, int short_tiles) {
    if (ntiles <= 0) return cudaSuccess;
    if (rows > 0) {
        cudaError_t err;
        if (launch_update_right_tma(wins, nwin, ntiles, dmax, qw_pool, M, ldm, rows, cols, factor, stream, &err,
                                    short_ctas, max_ctas, short_tiles))
            return err;
    }
    {
        cudaError_t e = set_smem(update_right_kernel<64, 1>, right_smem(64));
        if (e == cudaSuccess) e = set_smem(update_right_kernel<64, 2>, right_smem(64));
        if (e == cudaSuccess) e = set_smem(update_right_kernel<128, 1>, right_smem(128));
        if (e == cudaSuccess) e = set_smem(update_right_kernel<128, 2>, right_smem(128));
        if (e != cudaSuccess) return e;
    }
    const size_t sm = right_smem(dmax <= 64 ? 64 : 128);
    if (dmax <= 64) {
        if (factor)
            update_right_kernel<64, 2><<<ntiles, kUpdThreads, sm, stream>>>(wins, nwin, qw_pool, M, ldm, nrows_total);
        else
            update_right_kernel<64, 1><<<ntiles, kUpdThreads, sm, stream>>>(wins, nwin, qw_pool, M, ldm, nrows_total);
    } else {
        if (factor)
            update_right_kernel<128, 2><<<ntiles, kUpdThreads, sm, stream>>>(wins, nwin, qw_pool, M, ldm, nrows_total);
        else
            update_right_kernel<128, 1><<<ntiles, kUpdThreads, sm, stream>>>(wins, nwin, qw_pool, M, ldm, nrows_total);
    }
    return cudaGetLastError();
}

unsigned long long dmma_count_cp() {
    unsigned long long v = 0;
    if (cudaMemcpyFromSymbol(&v, g_dmma_cp, sizeof v) != cudaSuccess) cudaGetLastError();
    return v;
}

}  // namespace teig
