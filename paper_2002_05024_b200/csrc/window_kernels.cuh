// window_kernels.cuh -- window-local arithmetic for the single-CTA window
// kernels (sm_100a).  One warp owns one diagonal window held in shared
// memory; scalar decisions (rotations, the 2x2 standardization, the direct
// swap's Sylvester/QR/stability test) are evaluated redundantly by all 32
// lanes (warp-uniform control flow, no broadcast round trips), and the
// row/column/accumulator applications are lane-strided.
//
// Storage inside the window (d <= 128):
//   * W: the d x d upper quasi-triangular window in PACKED upper-Hessenberg
//     column storage -- column j keeps rows 0..min(j+1, d-1) at
//     offset j*(j+3)/2.  Entries below the first subdiagonal are exact zeros
//     in the reference's Schur form (verify.cpp:78-102) and are never stored.
//   * ACC: the d x d orthogonal accumulator, column-major, ld = d.
// This halves the window's footprint so that W (66 KB) + ACC (128 KB) of a
// 128-wide window fit the 227 KB per-CTA shared-memory limit.
#pragma once
#include <cfloat>
#include <cstdint>

namespace teig {

constexpr double kEps = 2.220446049250313e-16;  // 2^-52
constexpr double kSafeMin = DBL_MIN;

__device__ __forceinline__ double sgn(double x) { return x >= 0.0 ? 1.0 : -1.0; }

__device__ __forceinline__ int pk(int i, int j) { return j * (j + 3) / 2 + i; }  // i <= j+1

struct WinView {
    double* w;    // packed window
    double* acc;  // d x d, ld d
    int d;
    __device__ __forceinline__ double& W(int i, int j) const { return w[pk(i, j)]; }
    // read with the structural zeros below the subdiagonal
    __device__ __forceinline__ double Wz(int i, int j) const { return (i <= j + 1) ? w[pk(i, j)] : 0.0; }
    __device__ __forceinline__ double& A(int i, int j) const { return acc[i + j * d]; }
};

// make_givens semantics (reference kernels.cpp:86-102): c*a + s*b = r.
__device__ __forceinline__ void make_givens(double a, double b, double& c, double& s) {
    if (b == 0.0) {
        c = 1.0;
        s = 0.0;
    } else if (a == 0.0) {
        c = 0.0;
        s = 1.0;
    } else {
        const double r = hypot(a, b);
        c = a / r;
        s = b / r;
    }
}

// rows (i, i+1), columns [c0, d): [c s; -s c] from the left.
__device__ __forceinline__ void rot_rows(const WinView& v, double c, double s, int i, int c0, int lane) {
    for (int k = c0 + lane; k < v.d; k += 32) {
        double& x = v.W(i, k);
        double& y = v.W(i + 1, k);
        const double xv = x, yv = y;
        x = c * xv + s * yv;
        y = -s * xv + c * yv;
    }
}
// columns (i, i+1), rows [0, r1) of W
__device__ __forceinline__ void rot_cols(const WinView& v, double c, double s, int i, int r1, int lane) {
    for (int k = lane; k < r1; k += 32) {
        double& x = v.W(k, i);
        double& y = v.W(k, i + 1);
        const double xv = x, yv = y;
        x = c * xv + s * yv;
        y = -s * xv + c * yv;
    }
}
// columns (i, i+1) of ACC, all rows
__device__ __forceinline__ void rot_acc(const WinView& v, double c, double s, int i, int lane) {
    double* ci = v.acc + i * v.d;
    double* cj = ci + v.d;
    for (int k = lane; k < v.d; k += 32) {
        const double xv = ci[k], yv = cj[k];
        ci[k] = c * xv + s * yv;
        cj[k] = -s * xv + c * yv;
    }
}

// 2x2 standardization (reference kernels.cpp:126-219).  out: cs, sn, a, b, c, d.
__device__ __forceinline__ void standardize_2x2(double a, double b, double c, double d, double out[6]) {
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
    } else if ((a - d) == 0.0 && sgn(b) != sgn(c)) {
    } else {
        const double p = 0.5 * (a - d);
        const double qq = b + c;
        const double r2 = hypot(2.0 * p, qq);
        const double sig = sgn(qq);
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
        } else if (sgn(b) != sgn(c)) {
        } else {
            const double sab = sqrt(fabs(b)), sac = sqrt(fabs(c));
            const double pp = sab * sac;
            const double tau = 1.0 / sqrt(fabs(b + c));
            const double cs1 = sab * tau, sn1 = sgn(c) * sac * tau;
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

// Householder reflector of a short vector (reference kernels.cpp:24-58).
// len <= 4; v[0] = 1.  Returns beta.
__device__ __forceinline__ double make_reflector4(const double* x, int len, double v[4], double& tau) {
    tau = 0.0;
    v[0] = 1.0;
    v[1] = v[2] = v[3] = 0.0;
    if (len == 1) return x[0];
    const double alpha = x[0];
    double mx = 0.0;
    for (int i = 1; i < len; ++i) mx = fmax(mx, fabs(x[i]));
    double tail = 0.0;
    if (mx != 0.0) {
        double acc = 0.0;
        for (int i = 1; i < len; ++i) {
            const double t = x[i] / mx;
            acc += t * t;
        }
        tail = mx * sqrt(acc);
    }
    if (tail == 0.0) return alpha == 0.0 ? 0.0 : alpha;
    double beta = -sgn(alpha) * hypot(alpha, tail);
    double tl[3] = {len > 1 ? x[1] : 0.0, len > 2 ? x[2] : 0.0, len > 3 ? x[3] : 0.0};
    double a = alpha;
    int rescale = 0;
    while (fabs(beta) < kSafeMin / kEps && rescale < 20) {
        const double big = 1.0 / (kSafeMin / kEps);
        for (int i = 0; i < len - 1; ++i) tl[i] *= big;
        a *= big;
        double m2 = 0.0, t = 0.0;
        for (int i = 0; i < len - 1; ++i) m2 = fmax(m2, fabs(tl[i]));
        if (m2 != 0.0) {
            double acc = 0.0;
            for (int i = 0; i < len - 1; ++i) {
                const double u = tl[i] / m2;
                acc += u * u;
            }
            t = m2 * sqrt(acc);
        }
        beta = -sgn(a) * hypot(a, t);
        ++rescale;
    }
    tau = (beta - a) / beta;
    const double inv = 1.0 / (a - beta);
    for (int i = 1; i < len; ++i) v[i] = tl[i - 1] * inv;
    for (int r = 0; r < rescale; ++r) beta *= kSafeMin / kEps;
    return beta;
}

// Complete-pivoting elimination on a k x k (k <= 4) system; col-major m.
// rhs overwritten by the solution.  Returns false on a zero pivot.
// (reference kernels.cpp:419-464)
__device__ __forceinline__ bool gecp4(const double* m_in, int k, double* rhs, double& rcond) {
    double m[16];
    int cp[4] = {0, 1, 2, 3};
    for (int i = 0; i < k * k; ++i) m[i] = m_in[i];
    double amax = 0.0, smin = 0.0;
    for (int s = 0; s < k; ++s) {
        int pi = s, pj = s;
        double pv = 0.0;
        for (int i = s; i < k; ++i)
            for (int j = s; j < k; ++j)
                if (fabs(m[i + j * k]) > pv) {
                    pv = fabs(m[i + j * k]);
                    pi = i;
                    pj = j;
                }
        if (s == 0) amax = pv;
        smin = pv;
        if (pv == 0.0) {
            rcond = 0.0;
            return false;
        }
        if (pi != s) {
            for (int j = 0; j < k; ++j) {
                const double t = m[s + j * k];
                m[s + j * k] = m[pi + j * k];
                m[pi + j * k] = t;
            }
            const double t = rhs[s];
            rhs[s] = rhs[pi];
            rhs[pi] = t;
        }
        if (pj != s) {
            for (int i = 0; i < k; ++i) {
                const double t = m[i + s * k];
                m[i + s * k] = m[i + pj * k];
                m[i + pj * k] = t;
            }
            const int t = cp[s];
            cp[s] = cp[pj];
            cp[pj] = t;
        }
        for (int i = s + 1; i < k; ++i) {
            const double f = m[i + s * k] / m[s + s * k];
            m[i + s * k] = 0.0;
            for (int j = s + 1; j < k; ++j) m[i + j * k] -= f * m[s + j * k];
            rhs[i] -= f * rhs[s];
        }
    }
    double x[4];
    for (int kk = k - 1; kk >= 0; --kk) {
        double acc = rhs[kk];
        for (int j = kk + 1; j < k; ++j) acc -= m[kk + j * k] * x[j];
        x[kk] = acc / m[kk + kk * k];
    }
    for (int i = 0; i < k; ++i) rhs[cp[i]] = x[i];
    rcond = (amax > 0.0) ? smin / amax : 0.0;
    return true;
}

// Evaluates the direct swap of the adjacent p x p and q x q blocks whose
// (p+q)-sized diagonal window is blk (col-major, ld 4).  On success returns
// true, fills qd (the (p+q)x(p+q) orthogonal factor, ld 4) and wn (the
// swapped block, lower-left zeroed).  (reference kernels.cpp:529-578)
__device__ __forceinline__ bool direct_swap_eval(const double* blk, int p, int q, double qd[16], double wn[16]) {
    const int d = p + q;
    double a[4], c[4], b[4], x[4];
    for (int j = 0; j < p; ++j)
        for (int i = 0; i < p; ++i) a[i + j * p] = blk[i + j * 4];
    for (int j = 0; j < q; ++j)
        for (int i = 0; i < q; ++i) c[i + j * q] = blk[(p + i) + (p + j) * 4];
    for (int j = 0; j < q; ++j)
        for (int i = 0; i < p; ++i) b[i + j * p] = blk[i + (p + j) * 4];
    // Kronecker form of A X - X C = B (kernels.cpp:468-487)
    const int kd = p * q;
    double K[16], rhs[4];
    for (int j = 0; j < q; ++j)
        for (int i = 0; i < p; ++i) {
            const int row = j * p + i;
            for (int l = 0; l < q; ++l)
                for (int kk = 0; kk < p; ++kk) {
                    double val = 0.0;
                    if (l == j) val += a[i + kk * p];
                    if (kk == i) val -= c[l + j * q];
                    K[row + (l * p + kk) * kd] = val;
                }
        }
    for (int j = 0; j < q; ++j)
        for (int i = 0; i < p; ++i) rhs[j * p + i] = b[i + j * p];
    double rcond;
    if (!gecp4(K, kd, rhs, rcond)) return false;
    for (int i = 0; i < kd; ++i) x[i] = rhs[i];
    // one refinement pass on r = B - A X + X C (kernels.cpp:494-504)
    double r[4];
    for (int j = 0; j < q; ++j)
        for (int i = 0; i < p; ++i) {
            double acc = b[i + j * p];
            for (int kk = 0; kk < p; ++kk) {
                const double sc = -x[kk + j * p];
                if (sc != 0.0) acc += sc * a[i + kk * p];
            }
            r[i + j * p] = acc;
        }
    for (int j = 0; j < q; ++j)
        for (int i = 0; i < p; ++i) {
            double acc = r[i + j * p];
            for (int l = 0; l < q; ++l) {
                const double sc = c[l + j * q];
                if (sc != 0.0) acc += sc * x[i + l * p];
            }
            r[i + j * p] = acc;
        }
    double rc2;
    if (gecp4(K, kd, r, rc2))
        for (int i = 0; i < kd; ++i) x[i] += r[i];
    if (rcond < 1.8189894035458565e-12) return false;  // eps^(3/4) = 2^-39, kernels.cpp:540

    // Householder QR of [-X; I] (kernels.cpp:542-559)
    double z[16];
    for (int i = 0; i < 16; ++i) z[i] = 0.0;
    for (int j = 0; j < q; ++j) {
        for (int i = 0; i < p; ++i) z[i + j * 4] = -x[i + j * p];
        z[(p + j) + j * 4] = 1.0;
    }
    double v[2][4], tau[2];
    for (int j = 0; j < q; ++j) {
        double col[4];
        for (int i = j; i < d; ++i) col[i - j] = z[i + j * 4];
        const double beta = make_reflector4(col, d - j, v[j], tau[j]);
        z[j + j * 4] = beta;
        for (int i = j + 1; i < d; ++i) z[i + j * 4] = 0.0;
        if (tau[j] != 0.0)
            for (int jj = j + 1; jj < q; ++jj) {
                double w = 0.0;
                for (int i = 0; i < d - j; ++i) w += v[j][i] * z[(j + i) + jj * 4];
                w *= tau[j];
                for (int i = 0; i < d - j; ++i) z[(j + i) + jj * 4] -= w * v[j][i];
            }
    }
    for (int i = 0; i < 16; ++i) qd[i] = 0.0;
    for (int i = 0; i < d; ++i) qd[i + i * 4] = 1.0;
    for (int j = q - 1; j >= 0; --j) {
        if (tau[j] == 0.0) continue;
        for (int jj = 0; jj < d; ++jj) {
            double w = 0.0;
            for (int i = 0; i < d - j; ++i) w += v[j][i] * qd[(j + i) + jj * 4];
            w *= tau[j];
            for (int i = 0; i < d - j; ++i) qd[(j + i) + jj * 4] -= w * v[j][i];
        }
    }
    // wn = qd^T W qd with the reference's accumulation order (kernels.cpp:565-567)
    double tmp[16];
    for (int j = 0; j < d; ++j)
        for (int i = 0; i < d; ++i) {
            double acc = 0.0;
            for (int pp = 0; pp < d; ++pp) {
                const double sc = blk[pp + j * 4];
                if (sc != 0.0) acc += sc * qd[pp + i * 4];
            }
            tmp[i + j * 4] = acc;
        }
    for (int j = 0; j < d; ++j)
        for (int i = 0; i < d; ++i) {
            double acc = 0.0;
            for (int pp = 0; pp < d; ++pp) {
                const double sc = qd[pp + j * 4];
                if (sc != 0.0) acc += sc * tmp[i + pp * 4];
            }
            wn[i + j * 4] = acc;
        }
    double wnorm = 0.0, offnorm = 0.0;
    for (int j = 0; j < d; ++j)
        for (int i = 0; i < d; ++i) {
            wnorm = fmax(wnorm, fabs(blk[i + j * 4]));
            if (i >= q && j < q && i >= j + 1) offnorm = fmax(offnorm, fabs(wn[i + j * 4]));
        }
    if (offnorm > 32.0 * kEps * fmax(wnorm, kSafeMin)) return false;  // kernels.cpp:575
    for (int j = 0; j < q; ++j)
        for (int i = q; i < d; ++i) wn[i + j * 4] = 0.0;
    return true;
}

// Standardizes the 2x2 block at bp and folds the rotation into ACC
// (kernels.cpp:616-627).  Warp-collective; ends with __syncwarp.
__device__ __forceinline__ void restandardize(const WinView& v, int bp, int lane) {
    double st[6];
    standardize_2x2(v.W(bp, bp), v.W(bp, bp + 1), v.W(bp + 1, bp), v.W(bp + 1, bp + 1), st);
    __syncwarp();
    rot_rows(v, st[0], st[1], bp, bp + 2, lane);
    rot_cols(v, st[0], st[1], bp, bp, lane);
    rot_acc(v, st[0], st[1], bp, lane);
    if (lane == 0) {
        v.W(bp, bp) = st[2];
        v.W(bp, bp + 1) = st[3];
        v.W(bp + 1, bp) = st[4];
        v.W(bp + 1, bp + 1) = st[5];
    }
    __syncwarp();
}

// swap_adjacent_blocks (reference kernels.cpp:510-631) inside the window.
// Warp-collective.  Returns true on success, false when rejected (window
// unchanged).
__device__ __forceinline__ bool swap_adjacent(const WinView& v, int pos, int p, int q, int lane) {
    if (p == 1 && q == 1) {
        const double t11 = v.W(pos, pos), t12 = v.W(pos, pos + 1), t22 = v.W(pos + 1, pos + 1);
        double c, s;
        make_givens(t12, t22 - t11, c, s);
        if (t12 == 0.0 && t22 - t11 == 0.0) return true;
        __syncwarp();
        rot_rows(v, c, s, pos, pos + 2, lane);
        rot_cols(v, c, s, pos, pos, lane);
        rot_acc(v, c, s, pos, lane);
        if (lane == 0) {
            v.W(pos, pos) = t22;
            v.W(pos + 1, pos + 1) = t11;
            v.W(pos + 1, pos) = 0.0;
        }
        __syncwarp();
        return true;
    }
    const int d = p + q;
    double blk[16], qd[16], wn[16];
    for (int j = 0; j < 4; ++j)
        for (int i = 0; i < 4; ++i) blk[i + j * 4] = (i < d && j < d) ? v.Wz(pos + i, pos + j) : 0.0;
    if (!direct_swap_eval(blk, p, q, qd, wn)) return false;
    __syncwarp();
    // commit the block (only the packed, upper-Hessenberg part is stored)
    if (lane < d * d) {
        const int i = lane % d, j = lane / d;
        if (i <= j + 1) v.W(pos + i, pos + j) = wn[i + j * 4];
    }
    // rows above: W[0:pos, pos:pos+d] <- W[0:pos, pos:pos+d] qd
    for (int r = lane; r < pos; r += 32) {
        double t[4];
        for (int j = 0; j < d; ++j) t[j] = v.W(r, pos + j);
        for (int j = 0; j < d; ++j) {
            double acc = 0.0;
            for (int pp = 0; pp < d; ++pp) {
                const double sc = qd[pp + j * 4];
                if (sc != 0.0) acc += sc * t[pp];
            }
            v.W(r, pos + j) = acc;
        }
    }
    // columns right: W[pos:pos+d, c] <- qd^T W[pos:pos+d, c]
    for (int cc = pos + d + lane; cc < v.d; cc += 32) {
        double t[4];
        for (int i = 0; i < d; ++i) t[i] = v.W(pos + i, cc);
        double o[4];
        for (int i = 0; i < d; ++i) o[i] = 0.0;
        for (int pp = 0; pp < d; ++pp) {
            const double sc = t[pp];
            if (sc == 0.0) continue;
            for (int i = 0; i < d; ++i) o[i] += sc * qd[pp + i * 4];
        }
        for (int i = 0; i < d; ++i) v.W(pos + i, cc) = o[i];
    }
    // accumulator columns [pos, pos+d)
    for (int r = lane; r < v.d; r += 32) {
        double t[4];
        for (int j = 0; j < d; ++j) t[j] = v.A(r, pos + j);
        for (int j = 0; j < d; ++j) {
            double acc = 0.0;
            for (int pp = 0; pp < d; ++pp) {
                const double sc = qd[pp + j * 4];
                if (sc != 0.0) acc += sc * t[pp];
            }
            v.A(r, pos + j) = acc;
        }
    }
    __syncwarp();
    if (q == 2) restandardize(v, pos, lane);
    if (p == 2) restandardize(v, pos + q, lane);
    return true;
}

}  // namespace teig
