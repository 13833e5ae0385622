// schur_window.cu -- single-CTA window kernels of the multishift-QR Schur
// reduction (sm_100a).
//
// The AED window kernel owns ONE diagonal window of H in shared memory and
// accumulates the window's orthogonal similarity Q_w for the DMMA update
// kernels (update_dmma.cu), which apply it to the row panel right of the
// window, the column panel above it and the Schur-vector factor -- the
// reference's L/R/Q tasks (window_tasks.cpp:12-102).
//
// aed_window_kernel -- the AED window task (reference schur.cpp:421-459,
//   aed_process_window :147-248), the direct small-block solve (:554-579,
//   kernels.cpp:260-381) and the 2x2 standardization round (:728-757).
//   The reference gathers every nested window (recursive multishift QR,
//   :304-399, down to small_schur) into fresh dense matrices and propagates
//   their similarities with dense GEMMs.  Here everything happens IN PLACE on
//   the one shared-memory copy of the top window: every reflector/rotation is
//   applied to the full rows right of and the full columns above the
//   affected indices (which is what gather + apply_similarity_dense compute),
//   to Q_w, and to the first row of every enclosing nested AED window's
//   accumulator -- the only part of a nested accumulator the algorithm ever
//   reads (the spike beta*q(0,:)).  Nested levels therefore cost no extra
//   storage and no GEMMs.  Control flow is uniform: every decision is taken
//   by all threads from the same shared-memory values.
//
// The bulge-chain window kernel lives in schur_chase.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "device_types.h"
#include "launch.h"
#include "swap_math.cuh"

namespace teig {

namespace {

constexpr int NT = kAedThreads;      // threads of the AED / small-solve kernel
constexpr int kMaxSpk = 5;           // nested AED levels (depth 0, 2, 4, 6, 8)

__device__ __forceinline__ int tid() { return (int)threadIdx.x; }

struct Mat {
    double* p;
    int ld;
    __device__ __forceinline__ double& operator()(int i, int j) const { return p[i + j * ld]; }
};

// first row of a nested AED window's accumulator (window starts at `off`)
struct Spk {
    double* p;
    int off;
};

struct Ctx {
    Mat H;        // the top window, N x N
    int N;
    Mat Q;        // its accumulator, N x N
    Spk spk[kMaxSpk];
    int nspk;
    double* red;  // >= 32 doubles: block reductions
    double* scr;  // >= N + 8 doubles: reflector broadcast
    int* iscr;    // >= 8 ints
    double* shb;  // harvested shifts, per level 2*N doubles
    double* pkb;  // picked shifts, per level 2*(N+4) doubles
    double* spkb; // spike rows, per level N doubles
    int* nsh;     // harvested shift count per level
    SchurDevOpts o;
    unsigned long long* prof;  // shared-memory cycle counters (nullptr: off)
    double* brf;  // per-bulge reflector table of the pipelined sweeps (64 entries)
    int* wave_i;     // swap-wave bookkeeping (block list, pairs)
    double* wave_d;  // swap-wave pair transforms (kWaveMaxPairs x 32)
    double* snap;    // global scratch: H and Q snapshot of the top window (2 N^2)
    double* loc;     // kLocalAedDoubles: a small nested window gathered for one warp
};

// nested AED windows up to this order run gathered (aed_local)
#ifndef TEIG_LOCAL_AED_MAX
#define TEIG_LOCAL_AED_MAX 16
#endif
constexpr int kLocalAedMax = TEIG_LOCAL_AED_MAX;
constexpr int kLocalAedDoubles = 2 * kLocalAedMax * kLocalAedMax + kLocalAedMax + 8 + 32 + 8;

constexpr int kWaveMaxPairs = 56;
constexpr int kWaveMinWindow = 24;  // smaller AED windows use the sequential order

// diagnostics (TEIG_AED_PROF=1): cycle counters kept by thread 0
enum { kPfTotal, kPfSmall, kPfSwap, kPfSwapN, kPfSweep, kPfSpike, kPfSteps, kPfSmallSweeps, kPfWaveSteps, kPfWaveDecide, kPfWavePlan, kPfLocal, kPfLocalSmall, kPfLocalDefl, kPfLocalN, kPfN };
#define PF_T0() const long long _pf0 = clock64()
#define PF_ADD(i) do { if (c.prof && tid() == 0) c.prof[i] += (unsigned long long)(clock64() - _pf0); } while (0)
#define PF_INC(i) do { if (c.prof && tid() == 0) c.prof[i] += 1ull; } while (0)

__device__ double block_max(double v, double* red) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if ((tid() & 31) == 0) red[tid() >> 5] = v;
    __syncthreads();
    double r = red[0];
    for (int i = 1; i < NT / 32; ++i) r = fmax(r, red[i]);
    return r;
}

__device__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((tid() & 31) == 0) red[tid() >> 5] = v;
    __syncthreads();
    double r = 0.0;
    for (int i = 0; i < NT / 32; ++i) r += red[i];
    return r;
}

// ---------------------------------------------------------------------------
// in-place similarity primitives (all threads call; no barrier inside)

// rows r0..r0+L-1 of H <- (I - tau v v^T) rows, columns [c0, N)
template <int L>
__device__ __forceinline__ void left_apply(const Ctx& c, int r0, const double (&v)[L], double tau, int c0) {
    if (tau == 0.0) return;
    for (int j = c0 + tid(); j < c.N; j += NT) {
        double* col = &c.H(r0, j);
        double w = 0.0;
#pragma unroll
        for (int i = 0; i < L; ++i) w += v[i] * col[i];
        w *= tau;
#pragma unroll
        for (int i = 0; i < L; ++i) col[i] -= w * v[i];
    }
}

// the row vector starting at p (column stride cs) <- row (I - tau v v^T)
template <int L>
__device__ __forceinline__ void row_apply(double* p, int cs, const double (&v)[L], double tau) {
    double w = 0.0;
#pragma unroll
    for (int j = 0; j < L; ++j) w += p[j * cs] * v[j];
    w *= tau;
#pragma unroll
    for (int j = 0; j < L; ++j) p[j * cs] -= w * v[j];
}

// columns c0..c0+L-1: H rows [0, r1), all rows of Q, every spike row
template <int L>
__device__ __forceinline__ void right_apply(const Ctx& c, int c0, const double (&v)[L], double tau, int r1) {
    if (tau == 0.0) return;
    const int total = r1 + c.N + c.nspk;
    for (int t = tid(); t < total; t += NT) {
        if (t < r1) row_apply<L>(&c.H(t, c0), c.H.ld, v, tau);
        else if (t < r1 + c.N) row_apply<L>(&c.Q(t - r1, c0), c.Q.ld, v, tau);
        else {
            const Spk& s = c.spk[t - r1 - c.N];
            row_apply<L>(s.p + (c0 - s.off), 1, v, tau);
        }
    }
}

// general-length reflector held in c.scr[0..len) (v), c.scr[len] = tau
__device__ void left_apply_n(const Ctx& c, int r0, int len, int c0) {
    const double tau = c.scr[len];
    if (tau == 0.0) return;
    for (int j = c0 + tid(); j < c.N; j += NT) {
        double* col = &c.H(r0, j);
        double w = 0.0;
        for (int i = 0; i < len; ++i) w += c.scr[i] * col[i];
        w *= tau;
        for (int i = 0; i < len; ++i) col[i] -= w * c.scr[i];
    }
}

__device__ void right_apply_n(const Ctx& c, int c0, int len, int r1) {
    const double tau = c.scr[len];
    if (tau == 0.0) return;
    const int total = r1 + c.N + c.nspk;
    for (int t = tid(); t < total; t += NT) {
        double* p;
        int cs;
        if (t < r1) {
            p = &c.H(t, c0);
            cs = c.H.ld;
        } else if (t < r1 + c.N) {
            p = &c.Q(t - r1, c0);
            cs = c.Q.ld;
        } else {
            const Spk& s = c.spk[t - r1 - c.N];
            p = s.p + (c0 - s.off);
            cs = 1;
        }
        double w = 0.0;
        for (int j = 0; j < len; ++j) w += p[j * cs] * c.scr[j];
        w *= tau;
        for (int j = 0; j < len; ++j) p[j * cs] -= w * c.scr[j];
    }
}

// make_reflector (kernels.cpp:24-58) of x[0..len) in place by one warp: on
// return (after __syncwarp) x[0..len) = v, x[len] = tau, x[len+1] = beta.
__device__ void make_refl_warp(double* x, int len, int lane) {
    double tau = 0.0, beta;
    if (len == 1) {
        beta = x[0];
    } else {
        const double alpha = x[0];
        auto tailnorm = [&]() {
            double mx = 0.0;
            for (int i = 1 + lane; i < len; i += 32) mx = fmax(mx, fabs(x[i]));
#pragma unroll
            for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            if (mx == 0.0) return 0.0;
            double acc = 0.0;
            for (int i = 1 + lane; i < len; i += 32) {
                const double t = x[i] / mx;
                acc += t * t;
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            return mx * sqrt(acc);
        };
        const double tail = tailnorm();
        if (tail == 0.0) {
            beta = (alpha == 0.0) ? 0.0 : alpha;
            __syncwarp();
            for (int i = 1 + lane; i < len; i += 32) x[i] = 0.0;
        } else {
            beta = -sgnd(alpha) * hypot(alpha, tail);
            double a = alpha;
            int rescale = 0;
            while (fabs(beta) < kSafeMinD / kEpsD && rescale < 20) {
                const double big = 1.0 / (kSafeMinD / kEpsD);
                __syncwarp();
                for (int i = 1 + lane; i < len; i += 32) x[i] *= big;
                __syncwarp();
                a *= big;
                beta = -sgnd(a) * hypot(a, tailnorm());
                ++rescale;
            }
            tau = (beta - a) / beta;
            const double inv = 1.0 / (a - beta);
            __syncwarp();
            for (int i = 1 + lane; i < len; i += 32) x[i] *= inv;
            for (int r = 0; r < rescale; ++r) beta *= kSafeMinD / kEpsD;
        }
    }
    __syncwarp();
    if (lane == 0) {
        x[0] = 1.0;
        x[len] = tau;
        x[len + 1] = beta;
    }
    __syncwarp();
}

// the same for the whole CTA (warp 0 computes): c.scr[0..len) = x on entry
__device__ void make_refl_block(const Ctx& c, int len) {
    __syncthreads();  // x written by the caller
    if (tid() < 32) make_refl_warp(c.scr, len, tid());
    __syncthreads();
}

// ---------------------------------------------------------------------------
// negligible-subdiagonal scan of the block [lo, lo+ihi) (schur.cpp:286-300,
// kernels.cpp:283-292): largest l in (0, ihi) with a negligible H(l, l-1),
// zeroed; 0 if none.
__device__ int scan_block(const Ctx& c, int lo, int ihi, double hnorm, double smlnum) {
    __syncthreads();
    if (tid() == 0) c.iscr[0] = 0;
    __syncthreads();
    for (int l = ihi - 1 - tid(); l > 0; l -= NT) {
        double tst = fabs(c.H(lo + l - 1, lo + l - 1)) + fabs(c.H(lo + l, lo + l));
        if (tst == 0.0) tst = hnorm;
        if (fabs(c.H(lo + l, lo + l - 1)) <= fmax(kEpsD * tst, smlnum)) atomicMax(c.iscr, l);
    }
    __syncthreads();
    const int l = c.iscr[0];
    __syncthreads();
    if (l > 0 && tid() == 0) c.H(lo + l, lo + l - 1) = 0.0;
    __syncthreads();
    return l;
}

__device__ double hess_norm_block(const Ctx& c, int lo, int n) {
    double m = 0.0;
    for (int idx = tid(); idx < n * n; idx += NT) {
        const int j = idx / n, i = idx - j * n;
        if (i <= min(j + 1, n - 1)) m = fmax(m, fabs(c.H(lo + i, lo + j)));
    }
    return block_max(m, c.red);
}

// standardize the 2x2 block at p (kernels.cpp:245-256 / schur.cpp:82-94)
__device__ void std_block_dev(const Ctx& c, int p) {
    double st[6];
    std2x2(c.H(p, p), c.H(p, p + 1), c.H(p + 1, p), c.H(p + 1, p + 1), st);
    __syncthreads();
    const double cs = st[0], sn = st[1];
    const int ncol = c.N - p - 2;
    const int total = ncol + p + c.N + c.nspk;
    for (int t = tid(); t < total; t += NT) {
        if (t < ncol) {
            const int k = p + 2 + t;
            const double x = c.H(p, k), y = c.H(p + 1, k);
            c.H(p, k) = cs * x + sn * y;
            c.H(p + 1, k) = -sn * x + cs * y;
        } else {
            double* a;
            int s;
            const int u = t - ncol;
            if (u < p) {
                a = &c.H(u, p);
                s = c.H.ld;
            } else if (u < p + c.N) {
                a = &c.Q(u - p, p);
                s = c.Q.ld;
            } else {
                const Spk& sp = c.spk[u - p - c.N];
                a = sp.p + (p - sp.off);
                s = 1;
            }
            const double x = a[0], y = a[s];
            a[0] = cs * x + sn * y;
            a[s] = -sn * x + cs * y;
        }
    }
    if (tid() == 0) {
        c.H(p, p) = st[2];
        c.H(p, p + 1) = st[3];
        c.H(p + 1, p) = st[4];
        c.H(p + 1, p + 1) = st[5];
    }
    __syncthreads();
}

// one similarity step with a length-L reflector at index k0: left on rows
// k0.. for columns [k0, N), right on columns k0.. for rows [0, r1).  When
// annih >= 0, column annih (rows k0..k0+L-1) is set to (beta, 0, ..).
template <int L>
__device__ __forceinline__ void sim_step(const Ctx& c, int k0, const double (&v)[L], double tau, double beta,
                                         int annih, int r1) {
    PF_INC(kPfSteps);
    left_apply<L>(c, k0, v, tau, k0);
    __syncthreads();
    if (annih >= 0 && tid() == 0) {
        c.H(k0, annih) = beta;
#pragma unroll
        for (int i = 1; i < L; ++i) c.H(k0 + i, annih) = 0.0;
    }
    right_apply<L>(c, k0, v, tau, r1);
    __syncthreads();
}

// ---------------------------------------------------------------------------
// small_schur (kernels.cpp:260-381) on the block [lo, lo+n), in place, run by
// ONE WARP: a double-shift sweep is a chain of dependent 3-element reflector
// steps whose per-step work (<= 96 columns left, <= 2*96 rows right) is a
// few items per lane, so warp-synchronous steps (__syncwarp) beat CTA-wide
// barriers.  The other warps wait at the closing barrier.

struct WCtx {  // the fields the warp path touches, held in registers
    double* H;
    int ldh, N;
    double* Q;
    int ldq, nspk;
    double* sp[kMaxSpk];
    int spoff[kMaxSpk];
    unsigned long long* prof;
};

__device__ __forceinline__ WCtx wctx(const Ctx& c) {
    WCtx w;
    w.H = c.H.p;
    w.ldh = c.H.ld;
    w.N = c.N;
    w.Q = c.Q.p;
    w.ldq = c.Q.ld;
    w.nspk = c.nspk;
#pragma unroll
    for (int k = 0; k < kMaxSpk; ++k) {
        w.sp[k] = c.spk[k].p;
        w.spoff[k] = c.spk[k].off;
    }
    w.prof = c.prof;
    return w;
}

#define WH(i, j) W.H[(i) + (j) * W.ldh]

template <int G>
__device__ __forceinline__ void gsync() {
    if (G == 32) __syncwarp();
    else __syncthreads();
}

template <int L, int G>
__device__ __forceinline__ void w_step(const WCtx& W, int lane, int k0, const double (&v)[L], double tau,
                                       double beta, int annih, int r1) {
    if (W.prof && lane == 0) W.prof[kPfSteps] += 1ull;
    if (tau != 0.0) {
        for (int j = k0 + lane; j < W.N; j += G) {
            double* col = &WH(k0, j);
            double w = 0.0;
#pragma unroll
            for (int i = 0; i < L; ++i) w += v[i] * col[i];
            w *= tau;
#pragma unroll
            for (int i = 0; i < L; ++i) col[i] -= w * v[i];
        }
    }
    gsync<G>();
    if (annih >= 0 && lane == 0) {
        WH(k0, annih) = beta;
#pragma unroll
        for (int i = 1; i < L; ++i) WH(k0 + i, annih) = 0.0;
    }
    if (tau != 0.0) {
        const int total = r1 + W.N + W.nspk;
        for (int t = lane; t < total; t += G) {
            double* p;
            int cs;
            if (t < r1) {
                p = &WH(t, k0);
                cs = W.ldh;
            } else if (t < r1 + W.N) {
                p = W.Q + (t - r1) + (size_t)k0 * W.ldq;
                cs = W.ldq;
            } else {
                const int k = t - r1 - W.N;
                p = W.sp[k] + (k0 - W.spoff[k]);
                cs = 1;
            }
            double w = 0.0;
#pragma unroll
            for (int j = 0; j < L; ++j) w += p[j * cs] * v[j];
            w *= tau;
#pragma unroll
            for (int j = 0; j < L; ++j) p[j * cs] -= w * v[j];
        }
    }
    gsync<G>();
}

template <int G>
__device__ void w_std_block(const WCtx& W, int lane, int p) {
    double st[6];
    std2x2(WH(p, p), WH(p, p + 1), WH(p + 1, p), WH(p + 1, p + 1), st);
    gsync<G>();
    const double cs = st[0], sn = st[1];
    const int ncol = W.N - p - 2;
    const int total = ncol + p + W.N + W.nspk;
    for (int t = lane; t < total; t += G) {
        if (t < ncol) {
            const int k = p + 2 + t;
            const double x = WH(p, k), y = WH(p + 1, k);
            WH(p, k) = cs * x + sn * y;
            WH(p + 1, k) = -sn * x + cs * y;
        } else {
            double* a;
            int s;
            const int u = t - ncol;
            if (u < p) {
                a = &WH(u, p);
                s = W.ldh;
            } else if (u < p + W.N) {
                a = W.Q + (u - p) + (size_t)p * W.ldq;
                s = W.ldq;
            } else {
                const int k = u - p - W.N;
                a = W.sp[k] + (p - W.spoff[k]);
                s = 1;
            }
            const double x = a[0], y = a[s];
            a[0] = cs * x + sn * y;
            a[s] = -sn * x + cs * y;
        }
    }
    if (lane == 0) {
        WH(p, p) = st[2];
        WH(p, p + 1) = st[3];
        WH(p + 1, p) = st[4];
        WH(p + 1, p + 1) = st[5];
    }
    gsync<G>();
}

template <int G>
__device__ bool small_schur_grp(const WCtx& W, int lane, int lo, int n, double* red, int* iscr) {
    if (n <= 1) return true;
    double hm = 0.0;
    for (int idx = lane; idx < n * n; idx += G) {
        const int j = idx / n, i = idx - j * n;
        if (i <= min(j + 1, n - 1)) hm = fmax(hm, fabs(WH(lo + i, lo + j)));
    }
    double hnorm;
    if (G == 32) {
#pragma unroll
        for (int o = 16; o; o >>= 1) hm = fmax(hm, __shfl_xor_sync(0xffffffffu, hm, o));
        hnorm = hm;
    } else {
        hnorm = block_max(hm, red);
    }
    if (hnorm == 0.0) return true;
    const double smlnum = kSafeMinD * ((double)n / kEpsD);
    const int max_sweeps = 30 * n;
    int ihi = n, its = 0, sweeps = 0;
    while (ihi > 0) {
        if (ihi == 1) {
            ihi = 0;
            its = 0;
            continue;
        }
        int best = 0;  // negligible-subdiagonal scan (kernels.cpp:283-292)
        for (int l = ihi - 1 - lane; l > 0; l -= G) {
            double tst = fabs(WH(lo + l - 1, lo + l - 1)) + fabs(WH(lo + l, lo + l));
            if (tst == 0.0) tst = hnorm;
            if (fabs(WH(lo + l, lo + l - 1)) <= fmax(kEpsD * tst, smlnum)) best = max(best, l);
        }
        int l;
        if (G == 32) {
            l = __reduce_max_sync(0xffffffffu, best);
        } else {
            best = __reduce_max_sync(0xffffffffu, best);
            if (lane == 0) iscr[0] = 0;
            __syncthreads();
            if ((lane & 31) == 0 && best > 0) atomicMax(iscr, best);
            __syncthreads();
            l = iscr[0];
            __syncthreads();
        }
        if (l > 0 && lane == 0) WH(lo + l, lo + l - 1) = 0.0;
        gsync<G>();
        if (l == ihi - 1) {
            ihi = l;
            its = 0;
            continue;
        }
        if (l == ihi - 2) {
            w_std_block<G>(W, lane, lo + l);
            ihi = l;
            its = 0;
            continue;
        }
        ++its;
        ++sweeps;
        if (W.prof && lane == 0) W.prof[kPfSmallSweeps] += 1ull;
        if (sweeps > max_sweeps) return false;
        double s11, s12, s21, s22;
        if (its % 10 == 0) {
            const double sp = fabs(WH(lo + ihi - 1, lo + ihi - 2)) +
                              ((ihi >= l + 3) ? fabs(WH(lo + ihi - 2, lo + ihi - 3)) : 0.0);
            s11 = 0.75 * sp + WH(lo + ihi - 1, lo + ihi - 1);
            s12 = -0.4375 * sp;
            s21 = sp;
            s22 = s11;
        } else {
            s11 = WH(lo + ihi - 2, lo + ihi - 2);
            s12 = WH(lo + ihi - 2, lo + ihi - 1);
            s21 = WH(lo + ihi - 1, lo + ihi - 2);
            s22 = WH(lo + ihi - 1, lo + ihi - 1);
        }
        const double ssum = s11 + s22, sprod = s11 * s22 - s12 * s21;
        double v0[3];
        {
            const int b = lo + l;
            const double a11 = WH(b, b), a12 = WH(b, b + 1), a21 = WH(b + 1, b), a22 = WH(b + 1, b + 1);
            const double a32 = WH(b + 2, b + 1);
            v0[0] = a11 * a11 + a12 * a21 - ssum * a11 + sprod;
            v0[1] = a21 * (a11 + a22 - ssum);
            v0[2] = a21 * a32;
            const double vm = fmax(fabs(v0[0]), fmax(fabs(v0[1]), fabs(v0[2])));
            if (vm != 0.0) {
                v0[0] /= vm;
                v0[1] /= vm;
                v0[2] /= vm;
            }
        }
        for (int i = l; i + 3 <= ihi; ++i) {
            double x[3];
            if (i == l) {
                x[0] = v0[0];
                x[1] = v0[1];
                x[2] = v0[2];
            } else {
                x[0] = WH(lo + i, lo + i - 1);
                x[1] = WH(lo + i + 1, lo + i - 1);
                x[2] = WH(lo + i + 2, lo + i - 1);
            }
            double v[3], tau;
            const double beta = reflector_fast<3>(x, v, tau);
            w_step<3, G>(W, lane, lo + i, v, tau, beta, i > l ? lo + i - 1 : -1, lo + min(i + 4, ihi));
        }
        {
            const int i = ihi - 2;
            double x[2] = {WH(lo + i, lo + i - 1), WH(lo + i + 1, lo + i - 1)};
            double v[2], tau;
            const double beta = reflector_fast<2>(x, v, tau);
            w_step<2, G>(W, lane, lo + i, v, tau, beta, lo + i - 1, lo + ihi);
        }
    }
    return true;
}

#undef WH

__device__ bool small_schur_dev(const Ctx& c, int lo, int n) {
    PF_T0();
    __syncthreads();
    // the whole CTA (a one-warp variant measured 1.7x slower: more items per
    // thread on the full-width rows/columns), context held in registers
    const WCtx W = wctx(c);
    const bool ok = small_schur_grp<NT>(W, tid(), lo, n, c.red, c.iscr);
    PF_ADD(kPfSmall);
    return ok;
}

// ---------------------------------------------------------------------------
// adjacent block swap (kernels.cpp:510-631) at absolute index pos, applied to
// the rows right of / columns above the block, to Q and the spike rows.
// one swap's transform M (row-major D x D) on the rows of its block, columns
// right of the block (M^T), by one warp
template <int D>
__device__ __forceinline__ void pair_left(const Ctx& c, const double* Mg, int pos, int lane) {
    double M[D][D];
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
        for (int i = 0; i < D; ++i) M[r][i] = Mg[r * D + i];
    for (int k = pos + D + lane; k < c.N; k += 32) {
        double* col = &c.H(pos, k);
        double x[D];
#pragma unroll
        for (int r = 0; r < D; ++r) x[r] = col[r];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double a = 0.0;
#pragma unroll
            for (int r = 0; r < D; ++r) a += M[r][i] * x[r];
            col[i] = a;
        }
    }
}

// ... on the columns of its block: H rows above, all Q rows, spike rows (M),
// and the new block NB
template <int D>
__device__ __forceinline__ void pair_right(const Ctx& c, const double* Mg, int pos, int lane) {
    double M[D][D];
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
        for (int j = 0; j < D; ++j) M[r][j] = Mg[r * D + j];
    const int total = pos + c.N + c.nspk;
    for (int t = lane; t < total; t += 32) {
        double* a;
        int st;
        if (t < pos) {
            a = &c.H(t, pos);
            st = c.H.ld;
        } else if (t < pos + c.N) {
            a = &c.Q(t - pos, pos);
            st = c.Q.ld;
        } else {
            const Spk& sk = c.spk[t - pos - c.N];
            a = sk.p + (pos - sk.off);
            st = 1;
        }
        double x[D];
#pragma unroll
        for (int r = 0; r < D; ++r) x[r] = a[r * st];
#pragma unroll
        for (int j = 0; j < D; ++j) {
            double acc = 0.0;
#pragma unroll
            for (int r = 0; r < D; ++r) acc += x[r] * M[r][j];
            a[j * st] = acc;
        }
    }
    const double* NB = Mg + 16;
    if (lane < D * D) c.H(pos + lane / D, pos + lane % D) = NB[lane];
}

// One thread's swap decision (kernels.cpp:510-631) for the adjacent p x p /
// q x q blocks at pos of H: M (row-major D x D, window <- M^T W M) and the new
// block NB.  Returns 0 rejected, 1 ok, 2 no-op (equal 1x1 values).
__device__ __noinline__ int swap_decide(const double* H, int ldh, int pos, int p, int q, double* M, double* NB) {
    if (p == 1 && q == 1) {
        const double t11 = H[pos + pos * ldh], t12 = H[pos + (pos + 1) * ldh], t22 = H[(pos + 1) + (pos + 1) * ldh];
        double cs = 1.0, sn = 0.0;
        const double bb = t22 - t11;
        if (bb == 0.0) {
            cs = 1.0;
            sn = 0.0;
        } else if (t12 == 0.0) {
            cs = 0.0;
            sn = 1.0;
        } else {
            const double r = hypot(t12, bb);
            cs = t12 / r;
            sn = bb / r;
        }
        if (t12 == 0.0 && bb == 0.0) return 2;  // equal values: no-op (kernels.cpp:517)
        M[0] = cs;
        M[1] = -sn;
        M[2] = sn;
        M[3] = cs;
        NB[0] = t22;
        NB[1] = t12;
        NB[2] = 0.0;
        NB[3] = t11;
        return 1;
    }
    auto run = [&](auto P_, auto Q_) {
        constexpr int P = decltype(P_)::value, Qn = decltype(Q_)::value, D = P + Qn;
        double blk[D][D], Mm[D][D], nb[D][D];
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) blk[i][j] = H[(pos + i) + (pos + j) * ldh];
        const bool ok = direct_swap<P, Qn>(blk, Mm, nb);
        if (ok) {
#pragma unroll
            for (int i = 0; i < D; ++i)
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    M[i * D + j] = Mm[i][j];
                    NB[i * D + j] = nb[i][j];
                }
        }
        return ok;
    };
    bool ok;
    if (p == 1) ok = run(std::integral_constant<int, 1>(), std::integral_constant<int, 2>());
    else if (q == 1) ok = run(std::integral_constant<int, 2>(), std::integral_constant<int, 1>());
    else ok = run(std::integral_constant<int, 2>(), std::integral_constant<int, 2>());
    return ok ? 1 : 0;
}

__device__ __noinline__ bool swap_dev(const Ctx& c, int pos, int p, int q) {
    __syncthreads();
    double* M = c.scr;        // row-major D x D
    double* NB = c.scr + 16;  // new block, row-major
    if (tid() == 0) {
        const int st = swap_decide(c.H.p, c.H.ld, pos, p, q, M, NB);
        c.iscr[1] = st;
    }
    __syncthreads();
    const int st = c.iscr[1];
    if (st != 1) return st == 2;
    const int D = p + q;
    // left part on warps 0..3, right part (and the block) on warps 4..7
    const int lane = tid() & 31, warp = tid() >> 5;
    if (warp == 0) {
        if (D == 2) pair_left<2>(c, M, pos, lane);
        else if (D == 3) pair_left<3>(c, M, pos, lane);
        else pair_left<4>(c, M, pos, lane);
    } else if (warp == 1) {
        if (D == 2) pair_right<2>(c, M, pos, lane);
        else if (D == 3) pair_right<3>(c, M, pos, lane);
        else pair_right<4>(c, M, pos, lane);
    }
    __syncthreads();
    return true;
}

__device__ __forceinline__ int default_shift_count_dev(int active) {  // schur.cpp:119-129
    int m = (active / 16) & ~1;
    m = max(m, 4);
    m = min(m, 64);
    if (3 * (m / 2) + 2 > active) {
        const int nb = (active >= 6) ? (active - 2) / 3 : 1;
        m = min(max(2, 2 * nb), 64);
    }
    return m;
}

__device__ __forceinline__ bool deflation_check_dev(double spike, double dsum, int norm_stable, double wnorm) {
    if (!norm_stable) return spike <= fmax(kEpsD * dsum, kSafeMinD);  // schur.cpp:406-411
    return spike <= kEpsD * wnorm;
}

struct AedCoreDev {
    int deflated;
    int converged;
    int swap_rejected;
    int spike_eliminated;
    double newbeta;
};

template <int D>
__device__ AedCoreDev aed_dev(Ctx& c, int e, int w, double beta);
template <int D>
__device__ AedCoreDev aed_local(Ctx& c, int e, int w, double beta);

// shift_vector (schur.cpp:29-43) at the top of the window starting at b
__device__ __forceinline__ void shift_vec_dev(const Ctx& c, int b, int rows, double ssum, double sprod,
                                              double (&v)[3]) {
    const double a11 = c.H(b, b), a12 = c.H(b, b + 1), a21 = c.H(b + 1, b), a22 = c.H(b + 1, b + 1);
    const double a32 = rows > 2 ? c.H(b + 2, b + 1) : 0.0;
    v[0] = a11 * a11 + a12 * a21 - ssum * a11 + sprod;
    v[1] = a21 * (a11 + a22 - ssum);
    v[2] = a21 * a32;
    const double vm = fmax(fabs(v[0]), fmax(fabs(v[1]), fabs(v[2])));
    if (vm != 0.0) {
        v[0] /= vm;
        v[1] /= vm;
        v[2] /= vm;
    }
}

// chase_one_step (schur.cpp:48-63) in place: the window is [lo+l, lo+ihi);
// r is in block coordinates.  Returns the new r.
__device__ int chase_step_dev(const Ctx& c, int lo, int ihi, int r) {
    const int len = min(3, ihi - r);
    if (len < 2 || r + 1 >= ihi) return ihi - 1;
    const int g = lo + r;
    const int r1 = lo + min(r + len + 1, ihi);
    if (len == 3) {
        double x[3] = {c.H(g, g - 1), c.H(g + 1, g - 1), c.H(g + 2, g - 1)}, v[3], tau;
        const double beta = reflector_fast<3>(x, v, tau);
        sim_step<3>(c, g, v, tau, beta, g - 1, r1);
    } else {
        double x[2] = {c.H(g, g - 1), c.H(g + 1, g - 1)}, v[2], tau;
        const double beta = reflector_fast<2>(x, v, tau);
        sim_step<2>(c, g, v, tau, beta, g - 1, r1);
    }
    return r + 1;
}

// one bulge's reflector at one step of a pipelined sweep
struct BRf {
    double v1, v2, tau, beta;
    int g, len, kind, r1;  // kind: 0 idle, 1 chase step, 2 intro
};

// The multishift sweep of multishift_schur_dense (schur.cpp:374-393) on the
// active block [l, ihi) of the block at lo, in place, with the nb bulges
// PIPELINED: bulge j is introduced at time 3j and then moves one row per time
// step (the reference introduces and partially chases them one by one, then
// chases each to the end).  At every position the lower bulge still acts
// first, and bulges 3 rows apart act on disjoint index sets, so this only
// reorders commuting left/right multiplications; depth 3nb + active instead
// of ~nb * active.  pairs: (re1, im1, re2, im2) per bulge.
//
// A time step is two barrier-separated phases: the left reflections (all
// warps), then the right ones (warps 0-6) while the last warp builds every
// bulge's reflector for the NEXT step -- lane j applies bulge j's right
// reflection to rows g+1..g+3 (the only ones of column g its next reflector
// reads; no other bulge touches column g) and reads them back, or, for an
// introduction, the active block's top-left entries (final after this step's
// left phase).  Same values as a separate reflector phase, one barrier less.
__device__ __forceinline__ BRf sweep_refl(const Ctx& c, int lo, int l, int ihi, int aw, int j, int t,
                                          const double* pairs) {
    const int s = t - 3 * j;
    BRf b{0.0, 0.0, 0.0, 0.0, 0, 0, 0, 0};
    if (s == 0) {
        const double re1 = pairs[4 * j], im1 = pairs[4 * j + 1], re2 = pairs[4 * j + 2], im2 = pairs[4 * j + 3];
        double sv[3], v[3], tau;
        shift_vec_dev(c, lo + l, aw, re1 + re2, re1 * re2 - im1 * im2, sv);
        b.beta = reflector_fast<3>(sv, v, tau);
        b.v1 = v[1];
        b.v2 = v[2];
        b.tau = tau;
        b.g = lo + l;
        b.len = 3;
        b.kind = 2;
        b.r1 = lo + l + min(4, aw);
    } else if (s > 0 && l + s < ihi - 1) {
        const int r = l + s, len = min(3, ihi - r), g = lo + r;
        if (len == 3) {
            double x[3] = {c.H(g, g - 1), c.H(g + 1, g - 1), c.H(g + 2, g - 1)}, v[3], tau;
            b.beta = reflector_fast<3>(x, v, tau);
            b.v1 = v[1];
            b.v2 = v[2];
            b.tau = tau;
        } else {
            double x[2] = {c.H(g, g - 1), c.H(g + 1, g - 1)}, v[2], tau;
            b.beta = reflector_fast<2>(x, v, tau);
            b.v1 = v[1];
            b.tau = tau;
        }
        b.g = g;
        b.len = len;
        b.kind = 1;
        b.r1 = lo + min(r + len + 1, ihi);
    }
    return b;
}

__device__ __forceinline__ void sweep_right_row(double* p, int cs, const BRf& b) {
    if (b.len == 3) {
        const double w = (p[0] + p[cs] * b.v1 + p[2 * cs] * b.v2) * b.tau;
        p[0] -= w;
        p[cs] -= w * b.v1;
        p[2 * cs] -= w * b.v2;
    } else {
        const double w = (p[0] + p[cs] * b.v1) * b.tau;
        p[0] -= w;
        p[cs] -= w * b.v1;
    }
}

__device__ void sweep_pipelined(const Ctx& c, int lo, int l, int ihi, int nb, const double* pairs) {
    BRf* tbuf = reinterpret_cast<BRf*>(c.brf);  // two tables of 32 (nb <= 31)
    const int aw = ihi - l;
    const int T = 3 * (nb - 1) + (ihi - 1 - l);
    const int M = 2 * c.N + c.nspk;
    constexpr int NG = NT - 32;      // threads of the general right phase (warps 0-6)
    const int owner = tid() - NG;    // last warp: lane j owns bulge j
    if (owner >= 0 && owner < nb) tbuf[owner] = sweep_refl(c, lo, l, ihi, aw, owner, 0, pairs);
    __syncthreads();
    for (int t = 0; t < T; ++t) {
        const BRf* tb = tbuf + (t & 1) * 32;
        BRf* tn = tbuf + ((t + 1) & 1) * 32;
        for (int it = tid(); it < nb * c.N; it += NT) {
            const int j = it / c.N, col = it - j * c.N;
            const BRf b = tb[j];
            if (!b.kind) continue;
            if (b.kind == 1 && col < b.len) c.H(b.g + col, b.g - 1) = (col == 0) ? b.beta : 0.0;
            if (b.tau == 0.0 || col < b.g) continue;
            double* p = &c.H(b.g, col);
            if (b.len == 3) {
                const double w = (p[0] + b.v1 * p[1] + b.v2 * p[2]) * b.tau;
                p[0] -= w;
                p[1] -= w * b.v1;
                p[2] -= w * b.v2;
            } else {
                const double w = (p[0] + b.v1 * p[1]) * b.tau;
                p[0] -= w;
                p[1] -= w * b.v1;
            }
        }
        __syncthreads();
        if (owner < 0) {
            for (int it = tid(); it < nb * M; it += NG) {
                const int j = it / M, k = it - j * M;
                const BRf b = tb[j];
                if (!b.kind || b.tau == 0.0) continue;
                double* p;
                int cs;
                if (k < c.N) {
                    if (k >= b.r1 || (k > b.g && k <= b.g + 3)) continue;  // rows g+1..g+3: the owner
                    p = &c.H(k, b.g);
                    cs = c.H.ld;
                } else if (k < 2 * c.N) {
                    p = &c.Q(k - c.N, b.g);
                    cs = c.Q.ld;
                } else {
                    const Spk& sp = c.spk[k - 2 * c.N];
                    p = sp.p + (b.g - sp.off);
                    cs = 1;
                }
                sweep_right_row(p, cs, b);
            }
        } else if (owner < nb) {
            const BRf b = tb[owner];
            if (b.kind && b.tau != 0.0)
                for (int k = b.g + 1; k <= b.g + 3 && k < b.r1; ++k) sweep_right_row(&c.H(k, b.g), c.H.ld, b);
            if (t + 1 < T) tn[owner] = sweep_refl(c, lo, l, ihi, aw, owner, t + 1, pairs);
        }
        __syncthreads();
    }
}


// ---------------------------------------------------------------------------
// AED deflation as a SWAP WAVE.  The reference (schur.cpp:169-204) tests the
// bottom block of the undecided range; a failed block is moved to the top of
// the window by a chain of adjacent swaps before the next block is tested.
// A block's test only reads its own diagonal and its spike entries
// beta*q(0, rows), which the failed blocks change only while passing it, so
// the next block can be tested as soon as the last failed block has passed
// it.  Here every failed block ("mover") climbs one block per step, movers
// trail each other, every mover's swap of the step is decided by its own
// thread and all are applied in one two-phase pass (rows, then columns:
// disjoint pairs commute).  The final arrangement and every decision are the
// reference's; the depth drops from #swaps (~800 per 96-window) to
// ~#blocks + #failures.  A rejected swap (where the reference stops the
// whole loop) makes the caller restore a snapshot and rerun the reference
// order.  Returns false on a rejection; ns_out = top of the deflated part.
__device__ bool deflate_wave(const Ctx& c, int e, int w, double beta, double wnorm, const double* sp, int sps,
                             int& ns_out) {
    int* wi = c.wave_i;     // [0] nblk [1] npairs [2] done [3] ns [4] rejected
    int* bsz = wi + 8;      // block sizes, top to bottom
    int* bst = bsz + 128;   // 0 undecided, 1 mover, 2 settled (top), 3 deflated (bottom)
    int* pr = bst + 128;    // per pair: upper block index, pos, p, q
    int* pt = pr + 4 * kWaveMaxPairs;  // per type: count[4], then the pair lists
    double* pm = c.wave_d;  // per pair: M[16], NB[16]
    const int lane = tid() & 31, warp = tid() >> 5;
    constexpr int NW = NT / 32;
    __syncthreads();
    if (tid() == 0) {
        int i = 0, k = 0;
        while (i < w) {
            const int sz = (i + 1 < w && c.H(e + i + 1, e + i) != 0.0) ? 2 : 1;
            bsz[k] = sz;
            bst[k] = 0;
            i += sz;
            ++k;
        }
        wi[0] = k;
        wi[3] = w;
        wi[4] = 0;
    }
    __syncthreads();
    const int nblk = wi[0];
    for (;;) {
        long long _pfp = clock64();
        if (tid() == 0) {
            // test the bottom undecided block(s) nobody still has to pass
            for (;;) {
                int k = nblk - 1;
                while (k >= 0 && bst[k] == 3) --k;
                if (k < 0 || bst[k] != 0) break;
                int pos = 0;
                for (int t = 0; t < k; ++t) pos += bsz[t];
                double spike = 0.0, dsum = 0.0;
                for (int r = pos; r < pos + bsz[k]; ++r) {
                    spike = fmax(spike, fabs(beta * sp[(e + r) * sps]));
                    dsum += fabs(c.H(e + r, e + r));
                }
                if (deflation_check_dev(spike, dsum, c.o.deflation, wnorm)) {
                    bst[k] = 3;
                    wi[3] = pos;
                } else {
                    bst[k] = 1;
                    break;
                }
            }
            // movers: settle at the top or pair with the undecided block above
            int np = 0, pos = 0;
            bool any = false;
            for (int k = 0; k < nblk; ++k) {
                if (bst[k] == 1) {
                    if (k == 0 || bst[k - 1] == 2) {
                        bst[k] = 2;
                    } else if (bst[k - 1] == 0 && np < kWaveMaxPairs) {
                        pr[4 * np] = k - 1;
                        pr[4 * np + 1] = e + pos - bsz[k - 1];
                        pr[4 * np + 2] = bsz[k - 1];
                        pr[4 * np + 3] = bsz[k];
                        ++np;
                    }
                }
                if (bst[k] == 0 || bst[k] == 1) any = true;
                pos += bsz[k];
            }
            wi[1] = np;
            wi[2] = any ? 0 : 1;
            for (int ty = 0; ty < 4; ++ty) pt[ty] = 0;
            for (int q = 0; q < np; ++q) {
                const int ty = (pr[4 * q + 2] - 1) * 2 + (pr[4 * q + 3] - 1);  // (p,q) -> 0..3
                pt[4 + ty * kWaveMaxPairs + pt[ty]++] = q;
            }
        }
        __syncthreads();
        if (c.prof && tid() == 0) {
            c.prof[kPfWavePlan] += (unsigned long long)(clock64() - _pfp);
            c.prof[kPfWaveSteps] += 1ull;
        }
        if (wi[2]) break;
        const int np = wi[1];
        _pfp = clock64();
        // every mover's swap decision on its own thread; warp w takes the pairs
        // of block-size type w so the four decision code paths run on
        // different warps concurrently instead of diverging inside one
        for (int li = lane; warp < 4 && li < pt[warp]; li += 32) {
            const int t = pt[4 + warp * kWaveMaxPairs + li];
            double* M = pm + 32 * t;
            double* NB = M + 16;
            const int pos = pr[4 * t + 1], p = pr[4 * t + 2], q = pr[4 * t + 3];
            const int st = swap_decide(c.H.p, c.H.ld, pos, p, q, M, NB);
            if (st == 0) wi[4] = 1;
            if (st == 2) {  // equal 1x1 values: the swap is the identity
                M[0] = 1.0; M[1] = 0.0; M[2] = 0.0; M[3] = 1.0;
                NB[0] = c.H(pos, pos); NB[1] = c.H(pos, pos + 1); NB[2] = 0.0; NB[3] = c.H(pos + 1, pos + 1);
            }
        }
        __syncthreads();
        if (c.prof && tid() == 0) c.prof[kPfWaveDecide] += (unsigned long long)(clock64() - _pfp);
        if (wi[4]) return false;
        if (c.prof && tid() == 0) c.prof[kPfSwapN] += (unsigned long long)np;
        for (int q = warp; q < np; q += NW) {  // rows of each pair, columns right of its block
            const double* M = pm + 32 * q;
            const int pos = pr[4 * q + 1], D = pr[4 * q + 2] + pr[4 * q + 3];
            if (D == 2) pair_left<2>(c, M, pos, lane);
            else if (D == 3) pair_left<3>(c, M, pos, lane);
            else pair_left<4>(c, M, pos, lane);
        }
        __syncthreads();
        for (int q = warp; q < np; q += NW) {  // columns of each pair: rows above, Q, spikes; the block
            const double* M = pm + 32 * q;
            const int pos = pr[4 * q + 1], D = pr[4 * q + 2] + pr[4 * q + 3];
            if (D == 2) pair_right<2>(c, M, pos, lane);
            else if (D == 3) pair_right<3>(c, M, pos, lane);
            else pair_right<4>(c, M, pos, lane);
        }
        __syncthreads();
        if (tid() == 0)
            for (int q = 0; q < np; ++q) {  // the pair's blocks changed places
                const int k = pr[4 * q];
                const int ts = bsz[k], tt = bst[k];
                bsz[k] = bsz[k + 1];
                bst[k] = bst[k + 1];
                bsz[k + 1] = ts;
                bst[k + 1] = tt;
            }
    }
    ns_out = wi[3] - 0;
    return true;
}

// top-window snapshot (H and Q, N x N each) to global scratch and back
__device__ void snap_copy(const Ctx& c, bool save) {
    const int N = c.N;
    for (int idx = tid(); idx < N * N; idx += NT) {
        const int j = idx / N, i = idx - j * N;
        if (save) {
            c.snap[idx] = c.H(i, j);
            c.snap[N * N + idx] = c.Q(i, j);
        } else {
            c.H(i, j) = c.snap[idx];
            c.Q(i, j) = c.snap[N * N + idx];
        }
    }
    __syncthreads();
}

// multishift_schur_dense (schur.cpp:304-399) on the block [lo, lo+n), in place
template <int D>
__device__ bool mshift_dev(Ctx& c, int lo, int n) {
    if (n <= 1) return true;
    const double hnorm = hess_norm_block(c, lo, n);
    const double smlnum = kSafeMinD * ((double)n / kEpsD);
    const int limit = 30 * n;
    int sweeps = 0, stagnation = 0, ihi = n;
    const int lvl = (D + 1) / 2;  // level of the AED windows this call opens
    while (ihi > 0) {
        if (ihi == 1) {
            ihi = 0;
            continue;
        }
        const int l = scan_block(c, lo, ihi, hnorm, smlnum);
        const int active = ihi - l;
        if (active == 1) {
            ihi = l;
            continue;
        }
        if (active == 2) {
            std_block_dev(c, lo + l);
            ihi = l;
            continue;
        }
        if (active <= c.o.small_threshold || D >= 8) {
            if (!small_schur_dev(c, lo + l, active)) return false;
            ihi = l;
            continue;
        }
        const int m = c.o.shift_count ? c.o.shift_count : default_shift_count_dev(active);
        int w = c.o.aed_window ? c.o.aed_window : (3 * m) / 2;
        w = min(max(w, 4), active);
        const int e = ihi - w;
        const double beta = (e > l) ? c.H(lo + e, lo + e - 1) : 0.0;
        AedCoreDev core{0, 0, 0, 0, 0.0};
        if constexpr (D < 8) {
            if (w <= kLocalAedMax && !(c.o.flags & kSchurFlagNoLocal)) core = aed_local<D + 1>(c, lo + e, w, beta);
            else core = aed_dev<D + 1>(c, lo + e, w, beta);
        }
        if (!core.converged) return false;
        if (e > l && tid() == 0) c.H(lo + e, lo + e - 1) = core.newbeta;
        __syncthreads();
        stagnation = (core.deflated == 0) ? stagnation + 1 : 0;
        ihi -= core.deflated;
        if (core.deflated > 0 && 100 * core.deflated >= 14 * w) continue;
        if (ihi - l < 4) continue;
        // pick_shifts (schur.cpp:97-117) by thread 0 into the level's buffer
        double* sh = c.shb + lvl * 2 * c.N;
        double* pk = c.pkb + lvl * 2 * (c.N + 4);
        if (tid() == 0) {
            int no = 0;
            const int nh = c.nsh[lvl];
            for (int i = 0; i < nh && no + 1 < m + 1; ++i) {
                const double re = sh[2 * i], im = sh[2 * i + 1];
                if (im > 0.0) {
                    if (no + 2 <= m) {
                        pk[2 * no] = re;
                        pk[2 * no + 1] = im;
                        pk[2 * no + 2] = re;
                        pk[2 * no + 3] = -im;
                        no += 2;
                    }
                }
            }
            // reals in harvest order, taken in pairs
            int nr = 0;
            double r0 = 0.0;
            for (int i = 0; i < nh; ++i) {
                if (sh[2 * i + 1] != 0.0) continue;
                if (nr % 2 == 0) {
                    r0 = sh[2 * i];
                } else if (no + 2 <= m) {
                    pk[2 * no] = r0;
                    pk[2 * no + 1] = 0.0;
                    pk[2 * no + 2] = sh[2 * i];
                    pk[2 * no + 3] = 0.0;
                    no += 2;
                }
                ++nr;
            }
            c.iscr[2] = no;
        }
        __syncthreads();
        int np = c.iscr[2];
        double ex[4];
        const bool exc = (stagnation >= 6 || np < 2);
        if (exc) {
            const double sp = fabs(c.H(lo + ihi - 1, lo + ihi - 2)) +
                              ((ihi >= l + 3) ? fabs(c.H(lo + ihi - 2, lo + ihi - 3)) : 0.0);
            const double h11 = 0.75 * sp + c.H(lo + ihi - 1, lo + ihi - 1);
            double st[6];
            std2x2(h11, -0.4375 * sp, sp, h11, st);
            // eigenvalues of the standardized block (kernels.cpp:210-217)
            if (st[4] == 0.0) {
                ex[0] = st[2];
                ex[1] = 0.0;
                ex[2] = st[5];
                ex[3] = 0.0;
            } else {
                const double bt = sqrt(fabs(st[3])) * sqrt(fabs(st[4]));
                ex[0] = st[2];
                ex[1] = bt;
                ex[2] = st[2];
                ex[3] = -bt;
            }
            np = 2;
            stagnation = 0;
        }
        if (++sweeps > limit) return false;
        const int nb = min(np / 2, (ihi - l - 2) / 3);
        if (nb == 0) continue;
        const int aw = ihi - l;
        PF_T0();
        if (exc) {
            if (tid() == 0)
                for (int q = 0; q < 4; ++q) pk[q] = ex[q];
            __syncthreads();
        }
        sweep_pipelined(c, lo, l, ihi, nb, pk);
        PF_ADD(kPfSweep);
    }
    return true;
}

// aed_process_window (schur.cpp:147-248) for a small nested window, gathered:
// warp 0 runs the whole window procedure on a private copy Hl with its own
// accumulator Ql (no block barrier per reflector, rows of length w instead of
// the enclosing window's), then the CTA applies the one similarity Ql to the
// enclosing context: rows right of / columns above the window, Q and the
// tracked spike rows.  Same decisions as the in-place aed_dev (the deflation
// test reads Ql's first row, which is the nested spike row it tracks).
template <int D>
__device__ AedCoreDev aed_local(Ctx& c, int e, int w, double beta) {
    PF_T0();
    const int lvl = D / 2;
    double* Hl = c.loc;
    double* Ql = Hl + kLocalAedMax * kLocalAedMax;
    double* xs = Ql + kLocalAedMax * kLocalAedMax;  // reflector, len + 2
    double* MB = xs + kLocalAedMax + 8;             // swap transform + new block
    int* res = reinterpret_cast<int*>(MB + 32);     // converged, deflated, rejected
    double* nbeta = MB + 36;
    __syncthreads();
    for (int idx = tid(); idx < w * w; idx += NT) {
        const int j = idx / w, i = idx - j * w;
        Hl[idx] = c.H(e + i, e + j);
        Ql[idx] = (i == j) ? 1.0 : 0.0;
    }
    __syncthreads();
    if (tid() < 32) {
        const int lane = tid();
        Ctx L = c;
        L.H = Mat{Hl, w};
        L.Q = Mat{Ql, w};
        L.N = w;
        L.nspk = 0;
        double mx = 0.0;
        for (int idx = lane; idx < w * w; idx += 32) mx = fmax(mx, fabs(Hl[idx]));
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        double wnorm = 0.0;
        if (mx != 0.0) {
            double acc = 0.0;
            for (int idx = lane; idx < w * w; idx += 32) {
                const double t = Hl[idx] / mx;
                acc += t * t;
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            wnorm = mx * sqrt(acc);
        }
        const long long t_s = clock64();
        const bool conv = small_schur_grp<32>(wctx(L), lane, 0, w, nullptr, nullptr);
        const long long t_d = clock64();
        if (c.prof && lane == 0) {
            c.prof[kPfLocalSmall] += (unsigned long long)(t_d - t_s);
            c.prof[kPfLocalN] += 1ull;
        }
        int deflated = 0, rejected = 0;
        double newbeta = 0.0;
        if (conv && beta == 0.0) {
            deflated = w;
        } else if (conv) {
            int ktop = 0, ns = w;
            while (ns > ktop) {
                const int bsize = (ns >= 2 && ns - 2 >= ktop && Hl[(ns - 1) + (ns - 2) * w] != 0.0) ? 2 : 1;
                const int bs = ns - bsize;
                double spike = 0.0, dsum = 0.0;
                for (int r = bs; r < ns; ++r) {
                    spike = fmax(spike, fabs(beta * Ql[r * w]));
                    dsum += fabs(Hl[r + r * w]);
                }
                if (deflation_check_dev(spike, dsum, c.o.deflation, wnorm)) {
                    ns = bs;
                    continue;
                }
                int cur = bs;
                bool stuck = false;
                while (cur > ktop) {
                    const int psize = (cur >= 2 && cur - 2 >= ktop && Hl[(cur - 1) + (cur - 2) * w] != 0.0) ? 2 : 1;
                    const int ps = cur - psize;
                    int st = 0;
                    if (lane == 0) st = swap_decide(Hl, w, ps, psize, bsize, MB, MB + 16);
                    st = __shfl_sync(0xffffffffu, st, 0);
                    __syncwarp();
                    if (st == 0) {
                        stuck = true;
                        break;
                    }
                    if (st == 1) {
                        const int Dd = psize + bsize;
                        if (Dd == 2) pair_left<2>(L, MB, ps, lane);
                        else if (Dd == 3) pair_left<3>(L, MB, ps, lane);
                        else pair_left<4>(L, MB, ps, lane);
                        __syncwarp();
                        if (Dd == 2) pair_right<2>(L, MB, ps, lane);
                        else if (Dd == 3) pair_right<3>(L, MB, ps, lane);
                        else pair_right<4>(L, MB, ps, lane);
                        __syncwarp();
                    }
                    cur = ps;
                }
                if (stuck) {
                    rejected = 1;
                    break;
                }
                ktop += bsize;
            }
            deflated = w - ns;
            if (c.prof && lane == 0) c.prof[kPfLocalDefl] += (unsigned long long)(clock64() - t_d);
            if (lane == 0) {  // harvest (schur.cpp:206-219)
                double* sh = c.shb + lvl * 2 * c.N;
                int nsh = 0;
                for (int i = 0; i < ns;) {
                    if (i + 1 < ns && Hl[(i + 1) + i * w] != 0.0) {
                        const double a = Hl[i + i * w], b = Hl[i + (i + 1) * w], cc = Hl[(i + 1) + i * w];
                        const double im = sqrt(fabs(b)) * sqrt(fabs(cc));
                        sh[2 * nsh] = a;
                        sh[2 * nsh + 1] = im;
                        sh[2 * nsh + 2] = a;
                        sh[2 * nsh + 3] = -im;
                        nsh += 2;
                        i += 2;
                    } else {
                        sh[2 * nsh] = Hl[i + i * w];
                        sh[2 * nsh + 1] = 0.0;
                        nsh += 1;
                        i += 1;
                    }
                }
                c.nsh[lvl] = nsh;
            }
            // spike elimination and Hessenberg restore (schur.cpp:222-245)
            auto left = [&](int r0, int len, int c0) {  // rows r0.., columns [c0, w)
                const double tau = xs[len];
                if (tau != 0.0)
                    for (int j = c0 + lane; j < w; j += 32) {
                        double* col = Hl + r0 + j * w;
                        double a = 0.0;
                        for (int i = 0; i < len; ++i) a += xs[i] * col[i];
                        a *= tau;
                        for (int i = 0; i < len; ++i) col[i] -= a * xs[i];
                    }
                __syncwarp();
            };
            auto right = [&](int c0, int len, int r1) {  // columns c0.., Hl rows [0, r1) and Ql
                const double tau = xs[len];
                if (tau != 0.0)
                    for (int t = lane; t < r1 + w; t += 32) {
                        double* p = (t < r1) ? Hl + t + c0 * w : Ql + (t - r1) + c0 * w;
                        double a = 0.0;
                        for (int j = 0; j < len; ++j) a += p[j * w] * xs[j];
                        a *= tau;
                        for (int j = 0; j < len; ++j) p[j * w] -= a * xs[j];
                    }
                __syncwarp();
            };
            if (ns == 1) {
                newbeta = beta * Ql[0];
            } else if (ns > 1) {
                for (int i = lane; i < ns; i += 32) xs[i] = beta * Ql[i * w];
                make_refl_warp(xs, ns, lane);
                newbeta = xs[ns + 1];
                left(0, ns, 0);
                right(0, ns, ns);
                for (int j = 0; j + 2 < ns; ++j) {
                    const int len = ns - j - 1;
                    for (int i = lane; i < len; i += 32) xs[i] = Hl[(j + 1 + i) + j * w];
                    make_refl_warp(xs, len, lane);
                    if (xs[len] == 0.0) continue;
                    const double hb = xs[len + 1];
                    left(j + 1, len, j + 1);
                    for (int i = lane; i < len; i += 32) Hl[(j + 1 + i) + j * w] = (i == 0) ? hb : 0.0;
                    __syncwarp();
                    right(j + 1, len, ns);
                }
            }
        }
        if (lane == 0) {
            res[0] = conv ? 1 : 0;
            res[1] = deflated;
            res[2] = rejected;
            *nbeta = newbeta;
        }
    }
    __syncthreads();
    AedCoreDev core{res[1], res[0], res[2], res[0], *nbeta};
    if (!core.converged) {
        core.spike_eliminated = 0;
        __syncthreads();
        return core;
    }
    // the similarity on the enclosing context: H rows [e, e+w) right of the
    // window (Ql^T x), H rows above it, Q and the spike rows (x Ql)
    const int ncol = c.N - e - w;
    const int total = ncol + e + c.N + c.nspk;
    for (int t = tid(); t < total + w * w; t += NT) {
        if (t >= total) {
            const int idx = t - total, j = idx / w, i = idx - j * w;
            c.H(e + i, e + j) = Hl[idx];
            continue;
        }
        double* a;  // a length-w vector (stride st): x <- Ql^T x (H rows) or x^T Ql (columns)
        int st;
        if (t < ncol) {
            a = &c.H(e, e + w + t);
            st = 1;
        } else {
            const int u = t - ncol;
            if (u < e) {
                a = &c.H(u, e);
                st = c.H.ld;
            } else if (u < e + c.N) {
                a = &c.Q(u - e, e);
                st = c.Q.ld;
            } else {
                const Spk& sk = c.spk[u - e - c.N];
                a = sk.p + (e - sk.off);
                st = 1;
            }
        }
        double x[kLocalAedMax];
#pragma unroll
        for (int r = 0; r < kLocalAedMax; ++r) x[r] = (r < w) ? a[r * st] : 0.0;
        for (int j = 0; j < w; ++j) {
            double acc = 0.0;
#pragma unroll
            for (int r = 0; r < kLocalAedMax; ++r)
                if (r < w) acc += x[r] * Ql[r + j * w];
            a[j * st] = acc;
        }
    }
    __syncthreads();
    PF_ADD(kPfLocal);
    return core;
}

// aed_process_window (schur.cpp:147-248) on the window [e, e+w), in place.
template <int D>
__device__ AedCoreDev aed_dev(Ctx& c, int e, int w, double beta) {
    AedCoreDev core{0, 1, 0, 0, 0.0};
    const int lvl = D / 2;
    // window Frobenius norm (frobenius_norm: scaled two-pass nrm2)
    double mx = 0.0;
    for (int idx = tid(); idx < w * w; idx += NT) mx = fmax(mx, fabs(c.H(e + idx % w, e + idx / w)));
    mx = block_max(mx, c.red);
    double wnorm = 0.0;
    if (mx != 0.0) {
        double acc = 0.0;
        for (int idx = tid(); idx < w * w; idx += NT) {
            const double t = c.H(e + idx % w, e + idx / w) / mx;
            acc += t * t;
        }
        wnorm = mx * sqrt(block_sum(acc, c.red));
    }
    // spike row: Q row 0 at the top level (Q is the window accumulator), a
    // tracked row for nested windows
    double* sp;
    int sps;
    if (D == 0) {
        sp = &c.Q(0, 0);
        sps = c.Q.ld;
    } else {
        sp = c.spkb + lvl * c.N;
        sps = 1;
        for (int i = tid(); i < w; i += NT) sp[i] = (i == 0) ? 1.0 : 0.0;
        c.spk[c.nspk] = Spk{sp, e};
        c.nspk++;
    }
    __syncthreads();
    bool conv;
    if (w <= c.o.small_threshold || D >= 8) conv = small_schur_dev(c, e, w);
    else {
        if constexpr (D < 8) conv = mshift_dev<D + 1>(c, e, w);
        else conv = small_schur_dev(c, e, w);
    }
    core.converged = conv ? 1 : 0;
    if (conv && beta == 0.0) {
        core.deflated = w;
        core.newbeta = 0.0;
        core.spike_eliminated = 1;
    } else if (conv) {
        int ktop = 0, ns = w;
        bool waved = false;
        if (D == 0 && w >= kWaveMinWindow && c.snap && !(c.o.flags & kSchurFlagNoWave)) {
            PF_T0();
            snap_copy(c, true);
            int nsw = w;
            if (deflate_wave(c, e, w, beta, wnorm, sp, sps, nsw)) {
                waved = true;
                ns = nsw;
                ktop = ns;
            } else {
                snap_copy(c, false);  // a rejected swap: rerun in the reference's order
            }
            PF_ADD(kPfSwap);
        }
        while (!waved && ns > ktop) {
            const int bsize = (ns >= 2 && ns - 2 >= ktop && c.H(e + ns - 1, e + ns - 2) != 0.0) ? 2 : 1;
            const int bs = ns - bsize;
            double spike = 0.0, dsum = 0.0;
            for (int r = bs; r < ns; ++r) {
                spike = fmax(spike, fabs(beta * sp[r * sps]));
                dsum += fabs(c.H(e + r, e + r));
            }
            if (deflation_check_dev(spike, dsum, c.o.deflation, wnorm)) {
                ns = bs;
            } else {
                int cur = bs;
                bool stuck = false;
                while (cur > ktop) {
                    const int psize = (cur >= 2 && cur - 2 >= ktop && c.H(e + cur - 1, e + cur - 2) != 0.0) ? 2 : 1;
                    const int ps = cur - psize;
                    PF_T0();
                    const bool sok = swap_dev(c, e + ps, psize, bsize);
                    PF_ADD(kPfSwap);
                    PF_INC(kPfSwapN);
                    if (!sok) {
                        stuck = true;
                        break;
                    }
                    cur = ps;
                }
                if (stuck) {
                    core.swap_rejected = 1;
                    break;
                }
                ktop += bsize;
            }
        }
        core.deflated = w - ns;
        // harvest the shifts of the undeflated part (schur.cpp:206-219)
        __syncthreads();
        if (tid() == 0) {
            double* sh = c.shb + lvl * 2 * c.N;
            int nsh = 0;
            for (int i = 0; i < ns;) {
                if (i + 1 < ns && c.H(e + i + 1, e + i) != 0.0) {
                    const double a = c.H(e + i, e + i), b = c.H(e + i, e + i + 1), cc = c.H(e + i + 1, e + i);
                    const double im = sqrt(fabs(b)) * sqrt(fabs(cc));
                    sh[2 * nsh] = a;
                    sh[2 * nsh + 1] = im;
                    sh[2 * nsh + 2] = a;
                    sh[2 * nsh + 3] = -im;
                    nsh += 2;
                    i += 2;
                } else {
                    sh[2 * nsh] = c.H(e + i, e + i);
                    sh[2 * nsh + 1] = 0.0;
                    nsh += 1;
                    i += 1;
                }
            }
            c.nsh[lvl] = nsh;
        }
        // spike elimination and Hessenberg restore (schur.cpp:222-245)
        if (ns == 0) {
            core.newbeta = 0.0;
        } else if (ns == 1) {
            core.newbeta = beta * sp[0];
        } else {
            PF_T0();
            for (int i = tid(); i < ns; i += NT) c.scr[i] = beta * sp[i * sps];
            make_refl_block(c, ns);
            core.newbeta = c.scr[ns + 1];
            left_apply_n(c, e, ns, e);
            __syncthreads();
            right_apply_n(c, e, ns, e + ns);
            __syncthreads();
            for (int j = 0; j + 2 < ns; ++j) {
                const int len = ns - j - 1;
                for (int i = tid(); i < len; i += NT) c.scr[i] = c.H(e + j + 1 + i, e + j);
                make_refl_block(c, len);
                if (c.scr[len] == 0.0) continue;
                const double hb = c.scr[len + 1];
                left_apply_n(c, e + j + 1, len, e + j + 1);
                for (int i = tid(); i < len; i += NT) c.H(e + j + 1 + i, e + j) = (i == 0) ? hb : 0.0;
                __syncthreads();
                right_apply_n(c, e + j + 1, len, e + ns);
                __syncthreads();
            }
            PF_ADD(kPfSpike);
        }
        core.spike_eliminated = 1;
    }
    __syncthreads();
    if (D != 0) c.nspk--;
    __syncthreads();
    return core;
}

}  // namespace

// ---------------------------------------------------------------------------
// AED / small-solve / 2x2 window kernel (one CTA)
__global__ void __launch_bounds__(NT) aed_window_kernel(double* __restrict__ Hg, long long ldh, int mode, int l,
                                                        int e, int w, SchurDevOpts o, double* __restrict__ qw_out,
                                                        AedDevOut* __restrict__ out, double* __restrict__ shifts_out,
                                                        unsigned long long* __restrict__ prof_out,
                                                        double* __restrict__ snap) {
    extern __shared__ __align__(16) double sm[];
    __shared__ unsigned long long pf[kPfN];
    const long long t_start = clock64();
    if (tid() < kPfN) pf[tid()] = 0ull;
    const int ld = w | 1;
    double* base = sm;
    Ctx c;
    c.H = Mat{base, ld};
    base += (size_t)ld * w;
    c.Q = Mat{base, ld};
    base += (size_t)ld * w;
    c.N = w;
    c.nspk = 0;
    c.red = base;
    base += 32;
    c.scr = base;
    base += w + 40;
    c.shb = base;
    base += (size_t)kMaxSpk * 2 * w;
    c.pkb = base;
    base += (size_t)kMaxSpk * 2 * (w + 4);
    c.spkb = base;
    base += (size_t)kMaxSpk * w;
    c.brf = base;
    base += 64 * 6;
    c.wave_d = base;
    base += kWaveMaxPairs * 32;
    c.loc = base;
    base += kLocalAedDoubles;
    c.snap = snap;
    c.iscr = reinterpret_cast<int*>(base);
    c.nsh = c.iscr + 8;
    c.wave_i = c.iscr + 32;
    c.o = o;
    c.prof = prof_out ? pf : nullptr;
    for (int idx = tid(); idx < w * w; idx += NT) {
        const int j = idx / w, i = idx - j * w;
        c.H(i, j) = Hg[(long long)(e + i) + (long long)(e + j) * ldh];
        c.Q(i, j) = (i == j) ? 1.0 : 0.0;
    }
    const double beta = (e > l) ? Hg[(long long)e + (long long)(e - 1) * ldh] : 0.0;
    __syncthreads();
    AedCoreDev core{0, 1, 0, 0, 0.0};
    if (mode == kSchurModeAed) {
        core = aed_dev<0>(c, 0, w, beta);
    } else if (mode == kSchurModeSmall) {
        core.converged = small_schur_dev(c, 0, w) ? 1 : 0;
    } else {
        std_block_dev(c, 0);
    }
    __syncthreads();
    const bool keep = !(mode == kSchurModeAed && !core.converged);
    for (int idx = tid(); idx < w * w; idx += NT) {
        const int j = idx / w, i = idx - j * w;
        if (keep) Hg[(long long)(e + i) + (long long)(e + j) * ldh] = c.H(i, j);
        qw_out[i + (long long)j * w] = keep ? c.Q(i, j) : (i == j ? 1.0 : 0.0);
    }
    if (tid() == 0) {
        if (mode == kSchurModeAed && core.converged && e > l) Hg[(long long)e + (long long)(e - 1) * ldh] = core.newbeta;
        out->deflated = core.deflated;
        out->converged = core.converged;
        out->swap_rejected = core.swap_rejected;
        out->spike_eliminated = core.spike_eliminated;
        out->newbeta = core.newbeta;
        out->nshifts = (mode == kSchurModeAed && core.converged && beta != 0.0) ? c.nsh[0] : 0;
    }
    if (mode == kSchurModeAed && core.converged && beta != 0.0)
        for (int i = tid(); i < 2 * c.nsh[0]; i += NT) shifts_out[i] = c.shb[i];
    if (prof_out && tid() == 0) {
        pf[kPfTotal] = (unsigned long long)(clock64() - t_start);
        for (int i = 0; i < kPfN; ++i) atomicAdd(prof_out + i, pf[i]);
    }
}

size_t aed_window_smem_bytes(int w) {
    const size_t ld = (size_t)(w | 1);
    const size_t dbl = 2 * ld * w + 32 + w + 40 + kMaxSpk * 2 * w + kMaxSpk * 2 * (w + 4) + kMaxSpk * w + 64 * 6 +
                       kWaveMaxPairs * 32 + kLocalAedDoubles;
    return dbl * sizeof(double) + (32 + 8 + 128 + 128 + 4 * kWaveMaxPairs + 4 + 4 * kWaveMaxPairs) * sizeof(int);
}

cudaError_t launch_aed_window(double* H, long long ldh, int mode, int l, int e, int w, const SchurDevOpts& o,
                              double* qw_out, AedDevOut* out, double* shifts_out, cudaStream_t stream,
                              unsigned long long* prof, double* snap) {
    const size_t smem = aed_window_smem_bytes(w);
    {
        cudaError_t err = ensure_dyn_smem((const void*)aed_window_kernel, aed_window_smem_bytes(kAedMaxWindow));
        if (err != cudaSuccess) return err;
    }
    aed_window_kernel<<<1, NT, smem, stream>>>(H, ldh, mode, l, e, w, o, qw_out, out, shifts_out, prof, snap);
    return cudaGetLastError();
}

}  // namespace teig
