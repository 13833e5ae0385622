// swap_math.cuh -- register-resident scalar arithmetic of one adjacent
// diagonal-block swap (sm_100a device code).
//
// Restates the reference's `kernels::swap_adjacent_blocks`
// (kernels.cpp:510-631) for one thread: the block sizes P (upper, moving
// down) and Q (lower, moving up) are template parameters so every loop is
// unrolled and every small matrix lives in registers (no local memory);
// pivoting decisions are applied with predicated selects.
//
// Output of a successful swap: the (P+Q)x(P+Q) orthogonal M such that the
// window becomes M^T W M (rows/columns outside the block) and the new
// (P+Q)x(P+Q) diagonal block `nb` (standardized, exact zeros below the new
// block profile).  M folds the reference's qd and its restandardization
// rotations (kernels.cpp:616-629) into one matrix; the block values are the
// reference's, and the coupled rows/columns receive the same similarity.
#pragma once
#include <cfloat>
#include <cstdint>

namespace teig {

constexpr double kEpsD = 2.220446049250313e-16;  // 2^-52 (kernels.cpp:16)
constexpr double kSafeMinD = DBL_MIN;            // kernels.cpp:17

__device__ __forceinline__ double sgnd(double x) { return x >= 0.0 ? 1.0 : -1.0; }

// 2x2 standardization (reference kernels.cpp:126-219).  out: cs, sn, a, b, c, d.
__device__ __forceinline__ void std2x2(double a, double b, double c, double d, double out[6]) {
    double cs = 1.0, sn = 0.0;
    const double mx = fmax(fmax(fabs(a), fabs(b)), fmax(fabs(c), fabs(d)));
    int ex = 0;
    if (mx > 0.0 && (mx > 1e150 || mx < 1e-150)) {
        ex = ilogb(mx);
        const double sc = ldexp(1.0, -ex);
        a *= sc; b *= sc; c *= sc; d *= sc;
    }
    if (c == 0.0) {
    } else if (b == 0.0) {
        cs = 0.0;
        sn = 1.0;
        const double ta = a;
        a = d;
        d = ta;
        b = -c;
        c = 0.0;
    } else if ((a - d) == 0.0 && sgnd(b) != sgnd(c)) {
    } else {
        const double p = 0.5 * (a - d);
        const double qq = b + c;
        const double r2 = hypot(2.0 * p, qq);
        const double sig = sgnd(qq);
        const double cos2 = sig * qq / r2;
        const double sin2 = -sig * 2.0 * p / r2;
        cs = sqrt(0.5 * (1.0 + cos2));
        sn = sin2 / (2.0 * cs);
        const double aa = cs * a + sn * c, bb = cs * b + sn * d;
        const double cc = -sn * a + cs * c, dd = -sn * b + cs * d;
        a = aa * cs + bb * sn;
        b = -aa * sn + bb * cs;
        c = cc * cs + dd * sn;
        d = -cc * sn + dd * cs;
        const double m = 0.5 * (a + d);
        a = m;
        d = m;
        if (c == 0.0) {
        } else if (b == 0.0) {
            const double tc = cs;
            cs = -sn;
            sn = tc;
            b = -c;
            c = 0.0;
        } else if (sgnd(b) != sgnd(c)) {
        } else {
            const double sab = sqrt(fabs(b)), sac = sqrt(fabs(c));
            const double pp = sab * sac;
            const double tau = 1.0 / sqrt(fabs(b + c));
            const double cs1 = sab * tau, sn1 = sgnd(c) * sac * tau;
            a = m + pp;
            d = m - pp;
            b = b - c;
            c = 0.0;
            const double tc = cs * cs1 - sn * sn1;
            sn = cs * sn1 + sn * cs1;
            cs = tc;
        }
    }
    const double back = ldexp(1.0, ex);
    out[0] = cs;
    out[1] = sn;
    out[2] = a * back;
    out[3] = b * back;
    out[4] = c * back;
    out[5] = d * back;
}

// Householder reflector of a length-L vector (reference kernels.cpp:24-58).
template <int L>
__device__ __forceinline__ double reflector(const double (&x)[L], double (&v)[L], double& tau) {
    tau = 0.0;
    v[0] = 1.0;
#pragma unroll
    for (int i = 1; i < L; ++i) v[i] = 0.0;
    if (L == 1) return x[0];
    const double alpha = x[0];
    double tl[L > 1 ? L - 1 : 1];
#pragma unroll
    for (int i = 1; i < L; ++i) tl[i - 1] = x[i];
    auto nrm = [&]() {
        double mx = 0.0;
#pragma unroll
        for (int i = 0; i < L - 1; ++i) mx = fmax(mx, fabs(tl[i]));
        if (mx == 0.0) return 0.0;
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < L - 1; ++i) {
            const double t = tl[i] / mx;
            acc += t * t;
        }
        return mx * sqrt(acc);
    };
    const double tail = nrm();
    if (tail == 0.0) return alpha == 0.0 ? 0.0 : alpha;
    double beta = -sgnd(alpha) * hypot(alpha, tail);
    double a = alpha;
    int rescale = 0;
    while (fabs(beta) < kSafeMinD / kEpsD && rescale < 20) {
        const double big = 1.0 / (kSafeMinD / kEpsD);
#pragma unroll
        for (int i = 0; i < L - 1; ++i) tl[i] *= big;
        a *= big;
        beta = -sgnd(a) * hypot(a, nrm());
        ++rescale;
    }
    tau = (beta - a) / beta;
    const double inv = 1.0 / (a - beta);
#pragma unroll
    for (int i = 1; i < L; ++i) v[i] = tl[i - 1] * inv;
    for (int r = 0; r < rescale; ++r) beta *= kSafeMinD / kEpsD;
    return beta;
}

// Householder reflector of a length-L (2 or 3) vector with the reference's
// conventions (beta = -sign(x0)||x||, v[0] = 1, zero tail -> tau = 0;
// kernels.cpp:24-58) in one square root and one division: mathematically the
// same reflector as reflector<L> (the reference's scaled two-pass norm and
// rescale loop are kept for the out-of-range cases only), used on the bulge
// chase critical path.
template <int L>
__device__ __forceinline__ double reflector_fast(const double (&x)[L], double (&v)[L], double& tau) {
    const double alpha = x[0];
    double mx = 0.0;
#pragma unroll
    for (int i = 1; i < L; ++i) mx = fmax(mx, fabs(x[i]));
    const double s = fmax(mx, fabs(alpha));
    if (mx == 0.0 || !(s > 1e-140 && s < 1e140)) return reflector<L>(x, v, tau);
    double ss = alpha * alpha;
#pragma unroll
    for (int i = 1; i < L; ++i) ss = fma(x[i], x[i], ss);
    const double beta = -sgnd(alpha) * sqrt(ss);
    const double u = beta - alpha;           // |u| = |alpha| + ||x|| > 0
    const double r = 1.0 / (beta * u);
    tau = u * u * r;                         // (beta - alpha) / beta
    const double inv = -beta * r;            // 1 / (alpha - beta)
    v[0] = 1.0;
#pragma unroll
    for (int i = 1; i < L; ++i) v[i] = x[i] * inv;
    return beta;
}

// Complete-pivoting LU of a K x K system (reference kernels.cpp:419-464),
// kept so that the refinement solve (kernels.cpp:501-504, which refactors the
// same matrix) replays the identical elimination on the new right-hand side
// instead of factoring twice.  m row-major m[i][j].  Row/column interchanges
// are predicated selects so everything stays in registers.
template <int K>
struct GecpLU {
    double u[K][K];     // upper factor (after interchanges)
    double f[K][K];     // elimination multipliers f[i][s], i > s
    int pi[K], pj[K];   // row / column pivot of step s
    double rcond;
    bool ok;

    __device__ __forceinline__ void factor(const double (&m_in)[K][K]) {
#pragma unroll
        for (int i = 0; i < K; ++i)
#pragma unroll
            for (int j = 0; j < K; ++j) u[i][j] = m_in[i][j];
        double amax = 0.0, smin = 0.0;
        ok = true;
#pragma unroll
        for (int s = 0; s < K; ++s) {
            int bi = s, bj = s;
            double pv = 0.0;
#pragma unroll
            for (int i = s; i < K; ++i)
#pragma unroll
                for (int j = s; j < K; ++j)
                    if (fabs(u[i][j]) > pv) {
                        pv = fabs(u[i][j]);
                        bi = i;
                        bj = j;
                    }
            pi[s] = bi;
            pj[s] = bj;
            if (s == 0) amax = pv;
            smin = pv;
            if (pv == 0.0) ok = false;
#pragma unroll
            for (int i = s + 1; i < K; ++i)
                if (bi == i) {
#pragma unroll
                    for (int j = 0; j < K; ++j) {
                        const double t = u[s][j];
                        u[s][j] = u[i][j];
                        u[i][j] = t;
                    }
                }
#pragma unroll
            for (int j = s + 1; j < K; ++j)
                if (bj == j) {
#pragma unroll
                    for (int i = 0; i < K; ++i) {
                        const double t = u[i][s];
                        u[i][s] = u[i][j];
                        u[i][j] = t;
                    }
                }
#pragma unroll
            for (int i = s + 1; i < K; ++i) {
                const double fm = u[i][s] / u[s][s];
                f[i][s] = fm;
                u[i][s] = 0.0;
#pragma unroll
                for (int j = s + 1; j < K; ++j) u[i][j] -= fm * u[s][j];
            }
        }
        rcond = ok ? ((amax > 0.0) ? smin / amax : 0.0) : 0.0;
    }

    // rhs <- solution, replaying the interchanges and multipliers.  The
    // interchanges are select chains: written as conditional swaps the
    // compiler turned them into dynamically indexed local-memory swaps on the
    // window kernels' critical path (same values either way).
    __device__ __forceinline__ void solve(double (&rhs)[K]) const {
#pragma unroll
        for (int s = 0; s < K; ++s) {
            const int p = pi[s];
            const double xs = rhs[s];
            double xq = xs;
#pragma unroll
            for (int i = s + 1; i < K; ++i) xq = (p == i) ? rhs[i] : xq;
#pragma unroll
            for (int i = s + 1; i < K; ++i) rhs[i] = (p == i) ? xs : rhs[i];
            rhs[s] = xq;
#pragma unroll
            for (int i = s + 1; i < K; ++i) rhs[i] -= f[i][s] * rhs[s];
        }
        double x[K];
#pragma unroll
        for (int kk = K - 1; kk >= 0; --kk) {
            double acc = rhs[kk];
#pragma unroll
            for (int j = kk + 1; j < K; ++j) acc -= u[kk][j] * x[j];
            x[kk] = acc / u[kk][kk];
        }
        // undo the column interchanges: cp = product of the transpositions
        int cp[K];
#pragma unroll
        for (int i = 0; i < K; ++i) cp[i] = i;
#pragma unroll
        for (int s = 0; s < K; ++s) {
            const int p = pj[s], cs = cp[s];
            int cq = cs;
#pragma unroll
            for (int j = s + 1; j < K; ++j) cq = (p == j) ? cp[j] : cq;
#pragma unroll
            for (int j = s + 1; j < K; ++j) cp[j] = (p == j) ? cs : cp[j];
            cp[s] = cq;
        }
#pragma unroll
        for (int t = 0; t < K; ++t) {
            double v = 0.0;
#pragma unroll
            for (int i = 0; i < K; ++i) v = (cp[i] == t) ? x[i] : v;
            rhs[t] = v;
        }
    }
};

// Direct swap of the adjacent P x P (upper) and Q x Q (lower) blocks held in
// blk (row-major, D = P+Q).  On success: M (row-major D x D, window <- M^T W M)
// and nbk, the new block.  Returns false when the reference rejects the swap.
template <int P, int Q>
__device__ __forceinline__ bool direct_swap(const double (&blk)[P + Q][P + Q], double (&M)[P + Q][P + Q],
                                            double (&nbk)[P + Q][P + Q]) {
    constexpr int D = P + Q;
    constexpr int K = P * Q;
    // Kronecker form of A X - X C = B (kernels.cpp:468-487); x index j*P + i
    double Km[K][K], rhs[K];
#pragma unroll
    for (int j = 0; j < Q; ++j)
#pragma unroll
        for (int i = 0; i < P; ++i) {
            const int row = j * P + i;
#pragma unroll
            for (int l = 0; l < Q; ++l)
#pragma unroll
                for (int kk = 0; kk < P; ++kk) {
                    double val = 0.0;
                    if (l == j) val += blk[i][kk];
                    if (kk == i) val -= blk[P + l][P + j];
                    Km[row][l * P + kk] = val;
                }
            rhs[row] = blk[i][P + j];
        }
    GecpLU<K> lu;
    lu.factor(Km);
    if (!lu.ok) return false;
    const double rcond = lu.rcond;
    lu.solve(rhs);
    double x[K];
#pragma unroll
    for (int i = 0; i < K; ++i) x[i] = rhs[i];
    // one refinement pass on r = B - A X + X C (kernels.cpp:494-504)
    double r[K];
#pragma unroll
    for (int j = 0; j < Q; ++j)
#pragma unroll
        for (int i = 0; i < P; ++i) {
            double acc = blk[i][P + j];
#pragma unroll
            for (int kk = 0; kk < P; ++kk) {
                const double sc = -x[j * P + kk];
                if (sc != 0.0) acc += sc * blk[i][kk];
            }
#pragma unroll
            for (int l = 0; l < Q; ++l) {
                const double sc = blk[P + l][P + j];
                if (sc != 0.0) acc += sc * x[l * P + i];
            }
            r[j * P + i] = acc;
        }
    lu.solve(r);  // same matrix: the reference's second factorization is identical
#pragma unroll
    for (int i = 0; i < K; ++i) x[i] += r[i];
    if (rcond < 1.8189894035458565e-12) return false;  // eps^(3/4) = 2^-39 (kernels.cpp:540)

    // Householder QR of Z = [-X; I] (D x Q) (kernels.cpp:542-559)
    double z[D][Q];
#pragma unroll
    for (int j = 0; j < Q; ++j) {
#pragma unroll
        for (int i = 0; i < P; ++i) z[i][j] = -x[j * P + i];
#pragma unroll
        for (int i = 0; i < Q; ++i) z[P + i][j] = (i == j) ? 1.0 : 0.0;
    }
    double v0[D], tau0;
    {
        double col[D];
#pragma unroll
        for (int i = 0; i < D; ++i) col[i] = z[i][0];
        const double beta = reflector<D>(col, v0, tau0);
        z[0][0] = beta;
#pragma unroll
        for (int i = 1; i < D; ++i) z[i][0] = 0.0;
        if (Q > 1 && tau0 != 0.0) {
            double w = 0.0;
#pragma unroll
            for (int i = 0; i < D; ++i) w += v0[i] * z[i][Q - 1];
            w *= tau0;
#pragma unroll
            for (int i = 0; i < D; ++i) z[i][Q - 1] -= w * v0[i];
        }
    }
    double v1[D > 1 ? D - 1 : 1], tau1 = 0.0;
    if (Q == 2) {
        double col[D - 1];
#pragma unroll
        for (int i = 1; i < D; ++i) col[i - 1] = z[i][Q - 1];
        reflector<D - 1>(col, v1, tau1);
    }
    // qd = H0 H1 (apply H1 then H0 to the identity, kernels.cpp:558-559)
    double qd[D][D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) qd[i][j] = (i == j) ? 1.0 : 0.0;
    if (Q == 2 && tau1 != 0.0) {
#pragma unroll
        for (int jj = 0; jj < D; ++jj) {
            double w = 0.0;
#pragma unroll
            for (int i = 0; i < D - 1; ++i) w += v1[i] * qd[1 + i][jj];
            w *= tau1;
#pragma unroll
            for (int i = 0; i < D - 1; ++i) qd[1 + i][jj] -= w * v1[i];
        }
    }
    if (tau0 != 0.0) {
#pragma unroll
        for (int jj = 0; jj < D; ++jj) {
            double w = 0.0;
#pragma unroll
            for (int i = 0; i < D; ++i) w += v0[i] * qd[i][jj];
            w *= tau0;
#pragma unroll
            for (int i = 0; i < D; ++i) qd[i][jj] -= w * v0[i];
        }
    }
    // wn = qd^T W qd (kernels.cpp:565-567, same accumulation order)
    double tmp[D][D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
            double acc = 0.0;
#pragma unroll
            for (int p = 0; p < D; ++p) {
                const double sc = blk[p][j];
                if (sc != 0.0) acc += sc * qd[p][i];
            }
            tmp[i][j] = acc;
        }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
            double acc = 0.0;
#pragma unroll
            for (int p = 0; p < D; ++p) {
                const double sc = qd[p][j];
                if (sc != 0.0) acc += sc * tmp[i][p];
            }
            nbk[i][j] = acc;
        }
    double wnorm = 0.0, offnorm = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
            wnorm = fmax(wnorm, fabs(blk[i][j]));
            if (i >= Q && j < Q && i >= j + 1) offnorm = fmax(offnorm, fabs(nbk[i][j]));
        }
    if (offnorm > 32.0 * kEpsD * fmax(wnorm, kSafeMinD)) return false;  // kernels.cpp:575
#pragma unroll
    for (int j = 0; j < Q; ++j)
#pragma unroll
        for (int i = Q; i < D; ++i) nbk[i][j] = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) M[i][j] = qd[i][j];

    // restandardize the relocated 2x2 blocks (kernels.cpp:615-629): rotate
    // block rows/cols, set the standard values, fold the rotation into M
    auto restd = [&](int bp) {
        double st[6];
        std2x2(nbk[bp][bp], nbk[bp][bp + 1], nbk[bp + 1][bp], nbk[bp + 1][bp + 1], st);
        const double c = st[0], s = st[1];
#pragma unroll
        for (int k = 0; k < D; ++k) {
            if (k >= bp + 2) {  // rows bp, bp+1 right of the 2x2
                const double x0 = nbk[bp][k], y0 = nbk[bp + 1][k];
                nbk[bp][k] = c * x0 + s * y0;
                nbk[bp + 1][k] = -s * x0 + c * y0;
            }
            if (k < bp) {  // columns bp, bp+1 above the 2x2
                const double x0 = nbk[k][bp], y0 = nbk[k][bp + 1];
                nbk[k][bp] = c * x0 + s * y0;
                nbk[k][bp + 1] = -s * x0 + c * y0;
            }
        }
        nbk[bp][bp] = st[2];
        nbk[bp][bp + 1] = st[3];
        nbk[bp + 1][bp] = st[4];
        nbk[bp + 1][bp + 1] = st[5];
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const double x0 = M[k][bp], y0 = M[k][bp + 1];
            M[k][bp] = c * x0 + s * y0;
            M[k][bp + 1] = -s * x0 + c * y0;
        }
    };
    if (Q == 2) restd(0);
    if (P == 2) restd(Q);
    return true;
}

}  // namespace teig
