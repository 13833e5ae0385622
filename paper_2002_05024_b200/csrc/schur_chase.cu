// schur_chase.cu -- the bulge-chain window kernel of the multishift-QR Schur
// reduction and the whole-matrix helpers of its driver (sm_100a).
//
// chase_window_kernel -- one window of a bulge chain (intro window,
// reference schur.cpp:833-867 / introduce_bulges :611-648; chase windows,
// run_chase_window :507-523).  The reference moves the bulges one after the
// other (the bottom bulge over the whole hop, then the next).  Bulges sit
// exactly 3 rows apart, so a step of bulge k and the same step of its
// neighbours act on disjoint index sets; the kernel advances ALL bulges of the
// window one position per step in three barrier-separated phases
// (reflectors; left applications + accumulator; right applications), which
// reorders only commuting left/right multiplications of the reference's
// sequence.  The window lives packed in shared memory (column j keeps rows
// 0..j+3: the Hessenberg band plus the bulges' fill), Q_w densely (odd
// leading dimension: conflict-free row access).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "device_types.h"
#include "launch.h"
#include "swap_math.cuh"

namespace teig {

namespace {
constexpr int NTC = kChaseThreads;
__device__ __forceinline__ int tid() { return (int)threadIdx.x; }
}  // namespace

// ---------------------------------------------------------------------------
// chase window kernel (one CTA per window, all bulges advance together)

namespace {

struct BulgeRefl {
    double v1, v2, tau, beta;
    int ri, len, kind, pad;  // kind: 0 inactive, 1 chase step, 2 intro
};

// packed column-major window: column j holds rows 0..min(j+3, d-1)
struct Packed {
    double* p;
    const int* off;
    __device__ __forceinline__ double& operator()(int i, int j) const { return p[off[j] + i]; }
};

}  // namespace

__global__ void __launch_bounds__(NTC) chase_window_kernel(double* __restrict__ Hg, long long ldh,
                                                           const ChaseWin* __restrict__ wins,
                                                           const double* __restrict__ shift_pairs,
                                                           double* __restrict__ qw_pool) {
    const ChaseWin cw = wins[blockIdx.x];
    const int a = cw.a, d = cw.d;
    extern __shared__ __align__(16) double sm[];
    const int lda = d | 1;
    double* acc = sm;
    double* win = acc + (size_t)lda * d;
    BulgeRefl* br = reinterpret_cast<BulgeRefl*>(win + cw.packed_len);  // 8-byte aligned
    int* off = reinterpret_cast<int*>(br + 64);
    // column offsets of the packed layout
    if (tid() == 0) {
        int o = 0;
        for (int j = 0; j < d; ++j) {
            off[j] = o;
            o += min(j + 4, d);
        }
        off[d] = o;
    }
    __syncthreads();
    Packed W{win, off};
    for (int j = threadIdx.x >> 5; j < d; j += NTC / 32) {
        const int rows = min(j + 4, d);
        for (int i = threadIdx.x & 31; i < rows; i += 32) W(i, j) = Hg[(long long)(a + i) + (long long)(a + j) * ldh];
    }
    for (int idx = tid(); idx < d * d; idx += NTC) {
        const int j = idx / d, i = idx - j * d;
        acc[i + j * lda] = (i == j) ? 1.0 : 0.0;
    }
    __syncthreads();

    const int nb = cw.nb;
    const int ihi_l = cw.ihi - a;  // local end of the active range
    // schedule: bulge k (k = 0 bottom-most) -- first step time t0[k], step count
    // cnt[k], local row of its first reflector r0[k]:
    //   intro (mode 2): k = nb-1-j for bulge j: t0 = 3j, cnt = 3(nb-1-j)+1 (intro + chase)
    //   chase (mode 0): t0 = 0, cnt = hop, r0 = p_k - a
    //   final (mode 1): t0 = 0, cnt = ihi-1-p_k
    int T;
    if (cw.mode == kChaseIntro) T = 3 * nb - 2;
    else if (cw.mode == kChaseHop) T = cw.hop;
    else T = cw.ihi - 1 - (cw.p_bot - 3 * (nb - 1));
    const int lane = tid() & 31, warp = tid() >> 5;
    constexpr int NW = NTC / 32;
    for (int t = 0; t < T; ++t) {
        // phase R: reflectors (thread k for bulge k)
        if (tid() < nb) {
            const int k = tid();
            BulgeRefl b{0, 0, 0, 0, 0, 0, 0, 0};
            int ri = -1;
            bool intro = false;
            if (cw.mode == kChaseIntro) {
                const int j = nb - 1 - k;
                const int s = t - 3 * j;  // step index of bulge j
                if (s >= 0 && s <= 3 * (nb - 1 - j)) {
                    if (s == 0) intro = true;
                    ri = s;  // intro at local row 0, then chase from row 1
                }
            } else {
                const int p = cw.p_bot - 3 * k;
                const int cnt = (cw.mode == kChaseHop) ? cw.hop : (cw.ihi - 1 - p);
                if (t < cnt) ri = p + t - a;
            }
            if (ri >= 0) {
                if (intro) {
                    const int j = nb - 1 - k;
                    const double re1 = shift_pairs[cw.shift_off + 4 * j], im1 = shift_pairs[cw.shift_off + 4 * j + 1];
                    const double re2 = shift_pairs[cw.shift_off + 4 * j + 2], im2 = shift_pairs[cw.shift_off + 4 * j + 3];
                    const double ssum = re1 + re2, sprod = re1 * re2 - im1 * im2;
                    const double a11 = W(0, 0), a12 = W(0, 1), a21 = W(1, 0), a22 = W(1, 1);
                    const double a32 = d > 2 ? W(2, 1) : 0.0;
                    double sv[3] = {a11 * a11 + a12 * a21 - ssum * a11 + sprod, a21 * (a11 + a22 - ssum), a21 * a32};
                    const double vm = fmax(fabs(sv[0]), fmax(fabs(sv[1]), fabs(sv[2])));
                    if (vm != 0.0) {
                        sv[0] /= vm;
                        sv[1] /= vm;
                        sv[2] /= vm;
                    }
                    double v[3], tau;
                    b.beta = reflector_fast<3>(sv, v, tau);
                    b.v1 = v[1];
                    b.v2 = v[2];
                    b.tau = tau;
                    b.ri = 0;
                    b.len = 3;
                    b.kind = 2;
                } else {
                    const int len = min(3, ihi_l - ri);
                    if (len >= 2 && ri + 1 < ihi_l) {
                        if (len == 3) {
                            double x[3] = {W(ri, ri - 1), W(ri + 1, ri - 1), W(ri + 2, ri - 1)}, v[3], tau;
                            b.beta = reflector_fast<3>(x, v, tau);
                            b.v1 = v[1];
                            b.v2 = v[2];
                            b.tau = tau;
                        } else {
                            double x[2] = {W(ri, ri - 1), W(ri + 1, ri - 1)}, v[2], tau;
                            b.beta = reflector_fast<2>(x, v, tau);
                            b.v1 = v[1];
                            b.v2 = 0.0;
                            b.tau = tau;
                        }
                        b.ri = ri;
                        b.len = len;
                        b.kind = 1;
                    }
                }
            }
            br[k] = b;
        }
        __syncthreads();
        // phase L: annihilated columns, left applications, accumulator
        for (int k = warp; k < nb; k += NW) {
            const BulgeRefl b = br[k];
            if (!b.kind) continue;
            const int ri = b.ri;
            if (b.kind == 1 && lane < b.len) W(ri + lane, ri - 1) = (lane == 0) ? b.beta : 0.0;
            if (b.tau == 0.0) continue;
            const double v1 = b.v1, v2 = b.v2, tau = b.tau;
            if (b.len == 3) {
                for (int j = ri + lane; j < d; j += 32) {
                    double* col = &W(ri, j);
                    double w = (col[0] + v1 * col[1] + v2 * col[2]) * tau;
                    col[0] -= w;
                    col[1] -= w * v1;
                    col[2] -= w * v2;
                }
                for (int i = lane; i < d; i += 32) {
                    double* r = acc + i + ri * lda;
                    double w = (r[0] + r[lda] * v1 + r[2 * lda] * v2) * tau;
                    r[0] -= w;
                    r[lda] -= w * v1;
                    r[2 * lda] -= w * v2;
                }
            } else {
                for (int j = ri + lane; j < d; j += 32) {
                    double* col = &W(ri, j);
                    double w = (col[0] + v1 * col[1]) * tau;
                    col[0] -= w;
                    col[1] -= w * v1;
                }
                for (int i = lane; i < d; i += 32) {
                    double* r = acc + i + ri * lda;
                    double w = (r[0] + r[lda] * v1) * tau;
                    r[0] -= w;
                    r[lda] -= w * v1;
                }
            }
        }
        __syncthreads();
        // phase Rt: right applications on the window rows above each bulge
        for (int k = warp; k < nb; k += NW) {
            const BulgeRefl b = br[k];
            if (!b.kind || b.tau == 0.0) continue;
            const int ri = b.ri;
            const int r1 = min(ri + b.len + 1, d);
            const double v1 = b.v1, v2 = b.v2, tau = b.tau;
            double* c0 = win + off[ri];
            double* c1 = win + off[ri + 1];
            if (b.len == 3) {
                double* c2 = win + off[ri + 2];
                for (int i = lane; i < r1; i += 32) {
                    double w = (c0[i] + c1[i] * v1 + c2[i] * v2) * tau;
                    c0[i] -= w;
                    c1[i] -= w * v1;
                    c2[i] -= w * v2;
                }
            } else {
                for (int i = lane; i < r1; i += 32) {
                    double w = (c0[i] + c1[i] * v1) * tau;
                    c0[i] -= w;
                    c1[i] -= w * v1;
                }
            }
        }
        __syncthreads();
    }
    // scatter the window band and publish Q_w
    for (int j = threadIdx.x >> 5; j < d; j += NTC / 32) {
        const int rows = min(j + 4, d);
        for (int i = threadIdx.x & 31; i < rows; i += 32) Hg[(long long)(a + i) + (long long)(a + j) * ldh] = W(i, j);
    }
    double* qw = qw_pool + cw.qw_off;
    for (int idx = tid(); idx < d * d; idx += NTC) {
        const int j = idx / d, i = idx - j * d;
        qw[idx] = acc[i + j * lda];
    }
}

size_t chase_window_smem_bytes(int d) {
    const size_t lda = (size_t)(d | 1);
    size_t packed = 0;
    for (int j = 0; j < d; ++j) packed += (size_t)std::min(j + 4, d);
    return (lda * d + packed) * sizeof(double) + (size_t)(d + 2) * sizeof(int) + 64 * sizeof(BulgeRefl) + 64;
}

int chase_window_packed_len(int d) {
    int o = 0;
    for (int j = 0; j < d; ++j) o += std::min(j + 4, d);
    return o;
}

cudaError_t launch_chase_window(double* H, long long ldh, const ChaseWin* wins_dev, int idx, int d,
                                const double* shift_pairs, double* qw_pool, cudaStream_t stream) {
    {
        cudaError_t err = ensure_dyn_smem((const void*)chase_window_kernel, chase_window_smem_bytes(kChaseMaxWindow));
        if (err != cudaSuccess) return err;
    }
    chase_window_kernel<<<1, NTC, chase_window_smem_bytes(d), stream>>>(H, ldh, wins_dev + idx, shift_pairs, qw_pool);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// whole-matrix helpers of the driver

// max |h_ij| over the Hessenberg part (schur.cpp:682-685)
__global__ void hess_norm_kernel(const double* __restrict__ H, long long ldh, int n,
                                 unsigned long long* __restrict__ out) {
    double m = 0.0;
    for (long long j = blockIdx.x; j < n; j += gridDim.x) {
        const int rows = min((int)j + 2, n);
        for (int i = threadIdx.x; i < rows; i += blockDim.x) m = fmax(m, fabs(H[i + j * ldh]));
    }
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// scan_active_start_tiled (schur.cpp:581-595): largest l in (0, ihi) with a
// negligible subdiagonal, zeroed; *out = l (0 if none)
__global__ void scan_active_kernel(double* __restrict__ H, long long ldh, int n, int ihi, double hnorm,
                                   int* __restrict__ out) {
    __shared__ int best;
    if (threadIdx.x == 0) best = 0;
    __syncthreads();
    const double smlnum = kSafeMinD * ((double)n / kEpsD);
    for (int l = ihi - 1 - (int)threadIdx.x; l > 0; l -= blockDim.x) {
        double tst = fabs(H[(l - 1) + (long long)(l - 1) * ldh]) + fabs(H[l + (long long)l * ldh]);
        if (tst == 0.0) tst = hnorm;
        if (fabs(H[l + (long long)(l - 1) * ldh]) <= fmax(kEpsD * tst, smlnum)) atomicMax(&best, l);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int l = best;
        if (l > 0) H[l + (long long)(l - 1) * ldh] = 0.0;
        *out = l;
    }
}

cudaError_t launch_hess_norm(const double* H, long long ldh, int n, unsigned long long* out, cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned long long), stream);
    if (e != cudaSuccess) return e;
    hess_norm_kernel<<<std::min(n, 2048), 256, 0, stream>>>(H, ldh, n, out);
    return cudaGetLastError();
}

cudaError_t launch_scan_active(double* H, long long ldh, int n, int ihi, double hnorm, int* out,
                               cudaStream_t stream) {
    scan_active_kernel<<<1, 1024, 0, stream>>>(H, ldh, n, ihi, hnorm, out);
    return cudaGetLastError();
}

}  // namespace teig
