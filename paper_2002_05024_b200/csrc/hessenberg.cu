// hessenberg.cu -- blocked Householder reduction to upper Hessenberg form on
// the B200 (the phase that feeds schur_reduce; reference
// hessenberg.cpp:15-280), Q1 accumulated on request.
//
// The reference's algorithm, unchanged (so its results are reproduced to
// rounding): panels of b = min(tile, 64) columns; inside a panel, column i
// of the compact-WY factorisation (V, T, Y) is
//   x  = A[k+1:, k+i] - Y V(i-1, :)^T - V T^T V^T x          (bring up to date)
//   (v, tau, beta) = make_reflector(x[i:])                    (kernels.cpp:24-58)
//   T(:, i) = -tau T(:i, :i) V^T v,  T(i, i) = tau
//   Y(:, i) = tau (A_trail v - Y V^T v)                        (A_trail: columns
//             right of the panel column, as at the panel start)
// then the trailing block A[k+1:, k+b:] <- (I - V T V^T)^T (A - Y V_s^T), the
// rows above, A[:k+1, k+1:] <- A (I - V T V^T), and Q[:, k+1:] <- Q (I - V T V^T).
//
// B200 mapping.  The column step is a chain of grid-wide reductions over the
// m = n-k-1 panel rows -- latency-bound -- plus one GEMV with the trailing
// block (m x (m-i) doubles read once: the HBM-bound part, ~n^3/3 x 8 bytes
// over the whole reduction).  Five stream-ordered kernels per column, every
// reduction deterministic (per-CTA partials summed in a fixed order, no
// atomics): col_prep (x update, partial V^T x), col_apply (x -= V T^T V^T x,
// partial max |x|), col_sumsq (partial sum (x/max)^2: the reference's
// two-pass scaled nrm2), col_reflect (every CTA forms the same beta / tau,
// writes v and the finalised panel column, partial V^T v), col_matvec (GEMV
// over row blocks x column chunks, partials per chunk), col_y (Y column; CTA
// 0 also the T column; then the next column's col_prep for the same rows).  The panel's trailing, top-right and Q updates
// are FP64 tensor-core GEMMs (DMMA, dgemm.cuh).
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/taskeig_b200.h"
#include "launch.h"

namespace teig {

int set_error(int code, const std::string& msg);

namespace {

constexpr int HT = 256;        // threads per CTA of the column kernels
constexpr int HB = 64;         // max panel width
constexpr int MV_COLS = 128;   // max columns per GEMV chunk
constexpr int MV_MIN = 16;     // min columns per GEMV chunk
constexpr int MV_CTAS = 4 * 148;  // GEMV CTAs aimed for (four per SM)
constexpr double kSafe = DBL_MIN / 2.220446049250313e-16;  // safmin / eps (kernels.cpp:45)

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// per-CTA partials of sum_r V(r, j) * w_r for j < cnt (w_r = 0 outside)
__device__ void block_dots(const double* V, long long ldv, int m, int cnt, int r, double w, double* part_out,
                           double* sh /* HT/32 x HB */) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int j = 0; j < cnt; ++j) {
        const double p = warp_sum(r < m ? V[r + (long long)j * ldv] * w : 0.0);
        if (lane == 0) sh[warp * HB + j] = p;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < cnt; j += HT) {
        double s = 0.0;
        for (int w8 = 0; w8 < HT / 32; ++w8) s += sh[w8 * HB + j];
        part_out[j] = s;
    }
}

// column work state, device resident
struct Col {
    double* A;        // &A(k+1, 0): row r of the panel block at A[r + c*lda] for global column c
    long long lda;
    double* V;        // m x b, ld ldv
    double* Y;        // m x b, ld ldv
    double* T;        // b x b, ld HB
    long long ldv;
    double* x;        // m
    double* part;     // NB x HB partials of V^T v (col_reflect -> col_y)
    double* pprep;    // NB x HB partials of V^T x (col_prep / col_y_prep -> col_apply)
    double* pscal;    // NB partials: max |x_r|
    double* psum;     // NB partials: sum (x_r / max)^2
    double* scal;     // [0] tau, [1] beta, [2] mx, [3] inv, [4] rescale count
    double* s2;       // HB: V^T v
    double* ww;       // nchunk x m GEMV partials
    int k, m, nb_cta;
};

// x = A[k+1:, k+i] - Y V(i-1, :)^T ; partial (V^T x)_j  (row r of the CTA)
__device__ __forceinline__ void prep_row(const Col& c, int i, int r, double* sh) {
    double x = 0.0;
    if (r < c.m) {
        x = c.A[r + (long long)(c.k + i) * c.lda];
        for (int j = 0; j < i; ++j) {
            const double vr = c.V[(i - 1) + (long long)j * c.ldv];
            if (vr != 0.0) x -= c.Y[r + (long long)j * c.ldv] * vr;
        }
        c.x[r] = x;
    }
    if (i > 0) block_dots(c.V, c.ldv, c.m, i, r, x, c.pprep + (long long)blockIdx.x * HB, sh);
}

__global__ void __launch_bounds__(HT) col_prep(Col c, int i) {
    __shared__ double sh[HT / 32 * HB];
    prep_row(c, i, blockIdx.x * HT + threadIdx.x, sh);
}

// x -= V (T^T s), s = sum of the partials; partial max |x_r|, r > i
__global__ void __launch_bounds__(HT) col_apply(Col c, int i) {
    __shared__ double s[HB], tw[HB], red[HT / 32];
    for (int j = threadIdx.x; j < i; j += HT) {
        double a = 0.0;
        for (int b = 0; b < c.nb_cta; ++b) a += c.pprep[(long long)b * HB + j];
        s[j] = a;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < i; j += HT) {
        double a = 0.0;
        for (int l = 0; l <= j; ++l) a += c.T[l + j * HB] * s[l];
        tw[j] = a;
    }
    __syncthreads();
    const int r = blockIdx.x * HT + threadIdx.x;
    double mx = 0.0;
    if (r < c.m) {
        double x = c.x[r];
        for (int j = 0; j < i; ++j) {
            const double f = tw[j];
            if (f != 0.0) x -= c.V[r + (long long)j * c.ldv] * f;
        }
        c.x[r] = x;
        if (r > i) mx = fabs(x);
    }
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m2 = 0.0;
        for (int w = 0; w < HT / 32; ++w) m2 = fmax(m2, red[w]);
        c.pscal[blockIdx.x] = m2;
    }
}

// partial sum (x_r / mx)^2, r > i (the reference's two-pass nrm2, dense.hpp:112-123)
__global__ void __launch_bounds__(HT) col_sumsq(Col c, int i) {
    __shared__ double red[HT / 32];
    __shared__ double smx;
    if (threadIdx.x == 0) {
        double m2 = 0.0;
        for (int b = 0; b < c.nb_cta; ++b) m2 = fmax(m2, c.pscal[b]);
        smx = m2;
    }
    __syncthreads();
    const double mx = smx;
    const int r = blockIdx.x * HT + threadIdx.x;
    double t = 0.0;
    if (r < c.m && r > i && mx != 0.0) {
        const double q = c.x[r] / mx;
        t = q * q;
    }
    t = warp_sum(t);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (int w = 0; w < HT / 32; ++w) a += red[w];
        c.psum[blockIdx.x] = a;
        if (blockIdx.x == 0) c.scal[2] = mx;
    }
}

// make_reflector(x[i:]) (kernels.cpp:24-58), identically in every CTA; v and
// the finalised panel column; partial (V^T v)_j
__global__ void __launch_bounds__(HT) col_reflect(Col c, int i) {
    __shared__ double sh[HT / 32 * HB];
    __shared__ double st[4];  // tau, beta, inv, scale
    __shared__ int slow;
    __shared__ double red[HT / 32];
    if (threadIdx.x == 0) {
        double mx = 0.0;
        for (int b = 0; b < c.nb_cta; ++b) mx = fmax(mx, c.pscal[b]);
        const double alpha = c.x[i];
        double tau = 0.0, beta = alpha, inv = 0.0;
        int sl = 0;
        if (c.m - i > 1) {
            double acc = 0.0;
            for (int b = 0; b < c.nb_cta; ++b) acc += c.psum[b];
            const double tail = mx == 0.0 ? 0.0 : mx * sqrt(acc);
            if (tail != 0.0) {  // (tail == 0: zero vector or already collapsed, tau = 0)
                beta = -(alpha >= 0.0 ? 1.0 : -1.0) * hypot(alpha, tail);
                if (fabs(beta) >= kSafe) {
                    tau = (beta - alpha) / beta;
                    inv = 1.0 / (alpha - beta);
                } else {
                    sl = 1;
                }
            }
        }
        st[0] = tau;
        st[1] = beta;
        st[2] = inv;
        st[3] = 1.0;
        slow = sl;
    }
    __syncthreads();
    if (slow) {
        // tiny beta: scale the tail by 1/(safmin/eps) (a power of two: exact)
        // until |beta| >= safmin/eps, at most 20 times, recomputing the scaled
        // nrm2 (kernels.cpp:44-57); every CTA repeats it over the whole tail
        const double big = 1.0 / kSafe;
        double a = c.x[i], beta = st[1], scale = 1.0;
        int rescale = 0;
        while (fabs(beta) < kSafe && rescale < 20) {
            scale *= big;
            a *= big;
            double m2 = 0.0;
            for (int r = i + 1 + threadIdx.x; r < c.m; r += HT) m2 = fmax(m2, fabs(c.x[r] * scale));
            m2 = warp_max(m2);
            if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m2;
            __syncthreads();
            m2 = 0.0;
            for (int w = 0; w < HT / 32; ++w) m2 = fmax(m2, red[w]);
            __syncthreads();
            double ss = 0.0;
            if (m2 != 0.0)
                for (int r = i + 1 + threadIdx.x; r < c.m; r += HT) {
                    const double q = (c.x[r] * scale) / m2;
                    ss += q * q;
                }
            ss = warp_sum(ss);
            if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
            __syncthreads();
            ss = 0.0;
            for (int w = 0; w < HT / 32; ++w) ss += red[w];
            __syncthreads();
            beta = -(a >= 0.0 ? 1.0 : -1.0) * hypot(a, m2 * sqrt(ss));
            ++rescale;
        }
        if (threadIdx.x == 0) {
            st[0] = (beta - a) / beta;
            st[2] = 1.0 / (a - beta);
            st[3] = scale;
            for (int q = 0; q < rescale; ++q) beta *= kSafe;
            st[1] = beta;
        }
        __syncthreads();
    }
    const double tau = st[0], beta = st[1], inv = st[2], scale = st[3];
    const int r = blockIdx.x * HT + threadIdx.x;
    double v = 0.0;
    if (r < c.m) {
        const double x = c.x[r];
        if (r == i) v = 1.0;
        else if (r > i) v = tau == 0.0 ? 0.0 : (x * scale) * inv;
        c.V[r + (long long)i * c.ldv] = v;
        // finalised panel column: updated head, beta, explicit zeros
        c.A[r + (long long)(c.k + i) * c.lda] = r < i ? x : (r == i ? beta : 0.0);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        c.scal[0] = tau;
        c.scal[1] = beta;
    }
    if (i > 0) block_dots(c.V, c.ldv, c.m, i, r, v, c.part + (long long)blockIdx.x * HB, sh);
}

// ww[chunk][r] = sum over the chunk's columns c >= i of A(k+1+r, k+1+c) v_c
__global__ void __launch_bounds__(HT) col_matvec(Col c, int i, int chunk) {
    __shared__ double vs[MV_COLS];
    const int c0 = i + blockIdx.y * chunk;
    const int cn = min(chunk, c.m - c0);
    for (int t = threadIdx.x; t < cn; t += HT) vs[t] = c.V[(c0 + t) + (long long)i * c.ldv];
    __syncthreads();
    const int r = blockIdx.x * HT + threadIdx.x;
    if (r >= c.m) return;
    const double* a = c.A + r + (long long)(c.k + 1 + c0) * c.lda;
    double acc = 0.0;
#pragma unroll 4
    for (int t = 0; t < cn; ++t) acc += a[(long long)t * c.lda] * vs[t];
    c.ww[(long long)blockIdx.y * c.m + r] = acc;
}

// Y(:, i) = tau (ww - Y s2), s2 = V^T v summed from col_reflect's partials
// in every CTA (the order of col_tcol's sum); CTA 0 also writes T(:, i) =
// -tau T(:i, :i) s2, T(i, i) = tau -- col_tcol folded in, one launch less
// per column
__global__ void __launch_bounds__(HT) col_y(Col c, int i, int nchunk, int prep_next) {
    __shared__ double s2[HB];
    __shared__ double sh[HT / 32 * HB];
    for (int j = threadIdx.x; j < i; j += HT) {
        double a = 0.0;
        for (int b = 0; b < c.nb_cta; ++b) a += c.part[(long long)b * HB + j];
        s2[j] = a;
    }
    __syncthreads();
    const double tau = c.scal[0];
    if (blockIdx.x == 0) {
        for (int j = threadIdx.x; j < i; j += HT) {
            double a = 0.0;
            for (int l = j; l < i; ++l) a += c.T[j + l * HB] * s2[l];
            c.T[j + i * HB] = -tau * a;
        }
        if (threadIdx.x == 0) c.T[i + i * HB] = tau;
    }
    const int r = blockIdx.x * HT + threadIdx.x;
    if (r < c.m) {
        double w = 0.0;
        for (int q = 0; q < nchunk; ++q) w += c.ww[(long long)q * c.m + r];
        for (int j = 0; j < i; ++j) {
            const double f = s2[j];
            if (f != 0.0) w -= c.Y[r + (long long)j * c.ldv] * f;
        }
        c.Y[r + (long long)i * c.ldv] = tau * w;
    }
    // the next column's col_prep, fused: row r only needs Y(r, 0..i) (this
    // thread's) and V's row i (earlier kernels); its partials go to pprep
    if (prep_next) prep_row(c, i + 1, r, sh);
}

__global__ void zero_kernel(double* p, long long n) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
        p[t] = 0.0;
}

#define HCUDA(expr)                                                                                 \
    do {                                                                                            \
        cudaError_t _e = (expr);                                                                    \
        if (_e != cudaSuccess)                                                                      \
            throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(_e) + " at " + \
                                     __FILE__ + ":" + std::to_string(__LINE__));                    \
    } while (0)

struct Buf {
    double* p = nullptr;
    cudaStream_t s;
    Buf(size_t n, cudaStream_t st) : s(st) {
        if (n) HCUDA(lib_malloc_async(reinterpret_cast<void**>(&p), n * sizeof(double), st));
    }
    ~Buf() {
        if (p) cudaFreeAsync(p, s);
    }
};

}  // namespace

int hessenberg_reduce_device(int64_t n, double* dA, int64_t lda, double* dQ, int64_t ldq, int64_t panel_width,
                             teig_hessenberg_info* info, cudaStream_t s) {
    if (n < 1) return set_error(-1, "n must be >= 1");
    if (!dA || lda < n) return set_error(-3, "bad A");
    if (dQ && ldq < n) return set_error(-5, "bad Q");
    if (panel_width < 0) return set_error(-6, "panel_width must be >= 0");
    if (n > 2147483647LL) return set_error(TEIG_ERR_UNSUPPORTED, "n too large");
    // panel width as the reference picks it (hessenberg.cpp:193-195):
    // min(tile, 64) by default; the column kernels hold up to 64 columns
    const int64_t ts = n >= 1000 ? 128 : std::max<int64_t>(32, ((std::max<int64_t>(32, n / 8) + 7) / 8) * 8);
    const int bdef = (int)std::min<int64_t>(panel_width ? panel_width : std::min<int64_t>(ts, 64), HB);
    teig_hessenberg_info inf{};
    try {
        if (dQ) HCUDA(launch_set_identity(dQ, ldq, n, s));
        if (n >= 3) {
            const int64_t mmax = n - 1;
            const int nb_cta = (int)((mmax + HT - 1) / HT);
            const int nchunk_max = (int)((mmax + MV_MIN - 1) / MV_MIN);
            Buf V(mmax * HB, s), Y(mmax * HB, s), T(HB * HB, s), X(mmax, s), part((size_t)nb_cta * HB, s),
                pprep((size_t)nb_cta * HB, s),
                pscal(nb_cta, s), psum(nb_cta, s), scal(8, s), s2(HB, s), ww((size_t)nchunk_max * mmax, s), W(HB * n, s),
                W2(HB * n, s), P(n * HB, s), P2(n * HB, s), K(16 * HB * n, s);
            for (int64_t k = 0; k + 2 < n; k += bdef) {
                const int b = (int)std::min<int64_t>(bdef, n - 2 - k);
                const int m = (int)(n - k - 1);
                Col c{dA + (k + 1), lda, V.p, Y.p, T.p, (long long)m, X.p, part.p, pprep.p, pscal.p, psum.p, scal.p, s2.p,
                      ww.p, (int)k, m, (m + HT - 1) / HT};
                zero_kernel<<<64, 256, 0, s>>>(V.p, (long long)m * b);
                zero_kernel<<<1, 256, 0, s>>>(T.p, HB * HB);
                inf.launches += 2;
                col_prep<<<c.nb_cta, HT, 0, s>>>(c, 0);  // later columns: fused into col_y
                inf.launches += 1;
                for (int i = 0; i < b; ++i) {
                    col_apply<<<c.nb_cta, HT, 0, s>>>(c, i);
                    col_sumsq<<<c.nb_cta, HT, 0, s>>>(c, i);
                    col_reflect<<<c.nb_cta, HT, 0, s>>>(c, i);
                    // column chunks: enough CTAs to fill the GPU at every panel size
                    const int want = std::max(1, MV_CTAS / c.nb_cta);
                    const int chunk = std::min(MV_COLS, std::max(MV_MIN, (m - i + want - 1) / want));
                    const int nchunk = (m - i + chunk - 1) / chunk;
                    col_matvec<<<dim3(c.nb_cta, nchunk), HT, 0, s>>>(c, i, chunk);
                    col_y<<<c.nb_cta, HT, 0, s>>>(c, i, nchunk, i + 1 < b ? 1 : 0);
                    inf.launches += 5;
                }
                HCUDA(cudaGetLastError());
                // trailing block (hessenberg.cpp:110-138): G = A[k+1:, k+b:]
                //   G -= Y V_s^T  (V_s: V rows b-1.. = columns k+b..);  G -= V (T^T (V^T G))
                const int cw = (int)(n - k - b);
                double* G = dA + (k + 1) + (k + b) * lda;
                HCUDA(launch_dgemm(false, true, m, cw, b, -1.0, Y.p, m, V.p + (b - 1), m, 1.0, G, lda, s));
                HCUDA(launch_dgemm(true, false, b, cw, m, 1.0, V.p, m, G, lda, 0.0, W.p, HB, s, K.p, 16 * HB * n));
                HCUDA(launch_dgemm(true, false, b, cw, b, 1.0, T.p, HB, W.p, HB, 0.0, W2.p, HB, s));
                HCUDA(launch_dgemm(false, false, m, cw, b, -1.0, V.p, m, W2.p, HB, 1.0, G, lda, s));
                // rows above (hessenberg.cpp:140-160): A[:k+1, k+1:] -= ((A V) T) V^T
                const int rt = (int)(k + 1);
                double* Gt = dA + (k + 1) * lda;
                HCUDA(launch_dgemm(false, false, rt, b, m, 1.0, Gt, lda, V.p, m, 0.0, P.p, n, s, K.p, 16 * HB * n));
                HCUDA(launch_dgemm(false, false, rt, b, b, 1.0, P.p, n, T.p, HB, 0.0, P2.p, n, s));
                HCUDA(launch_dgemm(false, true, rt, m, b, -1.0, P2.p, n, V.p, m, 1.0, Gt, lda, s));
                inf.launches += 7;
                if (dQ) {  // Q[:, k+1:] <- Q (I - V T V^T) (hessenberg.cpp:165-181)
                    double* Gq = dQ + (k + 1) * ldq;
                    HCUDA(launch_dgemm(false, false, (int)n, b, m, 1.0, Gq, ldq, V.p, m, 0.0, P.p, n, s, K.p, 16 * HB * n));
                    HCUDA(launch_dgemm(false, false, (int)n, b, b, 1.0, P.p, n, T.p, HB, 0.0, P2.p, n, s));
                    HCUDA(launch_dgemm(false, true, (int)n, m, b, -1.0, P2.p, n, V.p, m, 1.0, Gq, ldq, s));
                    inf.launches += 3;
                }
                inf.panels += 1;
                const double dm = m, db = b;
                inf.flops += 2.0 * dm * (dm - db / 2) * db   // panel GEMVs
                             + 6.0 * dm * cw * db + 2.0 * rt * dm * db * 2.0 + (dQ ? 4.0 * (double)n * dm * db : 0.0);
            }
        }
        HCUDA(cudaStreamSynchronize(s));
    } catch (const std::exception& e) {
        return set_error(TEIG_ERR_CUDA, e.what());
    }
    inf.panel_width = bdef;
    if (info) *info = inf;
    return 0;
}

}  // namespace teig

using namespace teig;

extern "C" {

int teig_hessenberg_reduce_device(int64_t n, double* dA, int64_t lda, double* dQ, int64_t ldq, int64_t panel_width,
                                  teig_hessenberg_info* info, void* stream) {
    DeviceGuard device_guard(dA);
    return hessenberg_reduce_device(n, dA, lda, dQ, ldq, panel_width, info, (cudaStream_t)stream);
}

}  // extern "C"
