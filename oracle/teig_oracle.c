/*
 * oracle/teig_oracle.c -- TEST INFRASTRUCTURE ONLY (see teig_oracle.h).
 *
 * A plain-C restatement of the reference's reorder path.  Every function
 * cites the reference file:line it restates; the arithmetic is performed in
 * the same order as the reference so that, compiled with the same flags
 * (oracle/Makefile), results agree BIT-FOR-BIT with oracle/_ref
 * (tests/test_oracle.py).  Never used by the product path.
 */
#include "teig_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define EPS 2.220446049250313e-16 /* 2^-52, kernels.cpp:16 */
#define SAFMIN DBL_MIN            /* kernels.cpp:17 */
#define A_(m, i, j, ld) ((m)[(size_t)(i) + (size_t)(j) * (size_t)(ld)])

static double sgn(double x) { return x >= 0.0 ? 1.0 : -1.0; } /* kernels.cpp:19 */

/* ======================================================================= */
/* Philox4x32-10, philox.hpp:18-84                                          */

void teo_philox_round10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n1 = (uint32_t)p1;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        const uint32_t n3 = (uint32_t)p0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

void teo_philox_init(teo_philox* p, uint64_t seed) {
    p->key[0] = (uint32_t)seed;
    p->key[1] = (uint32_t)(seed >> 32);
    p->counter = 0;
    p->have = 0;
}

uint64_t teo_philox_next_u64(teo_philox* p) {
    if (p->have == 0) {
        const uint32_t ctr[4] = {(uint32_t)p->counter, (uint32_t)(p->counter >> 32), 0u, 0u};
        teo_philox_round10(ctr, p->key, p->buf);
        p->counter++;
        p->have = 2;
    }
    const int i = 2 - p->have;
    p->have--;
    return ((uint64_t)p->buf[2 * i + 1] << 32) | p->buf[2 * i];
}

double teo_philox_uniform_sym(teo_philox* p) {
    const uint64_t u = teo_philox_next_u64(p) >> 11;
    return (double)u * (2.0 / 9007199254740992.0) - 1.0;
}

double teo_philox_uniform01(teo_philox* p) {
    const uint64_t u = teo_philox_next_u64(p) >> 11;
    return (double)u * (1.0 / 9007199254740992.0);
}

uint64_t teo_philox_bounded(teo_philox* p, uint64_t n) { return teo_philox_next_u64(p) % n; }

/* ======================================================================= */
/* generators, generate.cpp                                                 */

void teo_default_spectrum(size_t n, double* re, double* im) {
    /* generate.cpp:68-91: n - 2*floor(n/4) reals on [-10,10], then floor(n/4)
     * conjugate pairs, re on [-9.7,9.7], im cycling 1,3,5 */
    const size_t npairs = n / 4, nreal = n - 2 * npairs;
    size_t k = 0;
    for (size_t i = 0; i < nreal; ++i, ++k) {
        re[k] = (nreal == 1) ? 1.0 : -10.0 + 20.0 * (double)i / (double)(nreal - 1);
        im[k] = 0.0;
    }
    for (size_t i = 0; i < npairs; ++i) {
        const double r = (npairs == 1) ? 0.5 : -9.7 + 19.4 * (double)i / (double)(npairs - 1);
        const double m = 1.0 + 2.0 * (double)(i % 3);
        re[k] = r; im[k] = m; ++k;
        re[k] = r; im[k] = -m; ++k;
    }
}

uint64_t teo_known_spectrum_seed(uint64_t seed) {
    /* generate.cpp:184 with ProblemKind::known_spectrum == 1 */
    return seed * 0x9E3779B97F4A7C15ull + 1ull;
}

void teo_schur_input(size_t n, uint64_t fill_seed, double* s, size_t ld) {
    /* generate.cpp:115-150.  The default spectrum lists reals first and then
     * pairs, so the layout is nreal 1x1 blocks followed by 2x2 blocks
     * [[a, b], [-b, a]] (b = |im|); the strictly upper part outside the
     * blocks is filled row by row from the Philox stream. */
    double* re = (double*)malloc(n * sizeof(double));
    double* im = (double*)malloc(n * sizeof(double));
    teo_default_spectrum(n, re, im);
    for (size_t j = 0; j < n; ++j) memset(&A_(s, 0, j, ld), 0, n * sizeof(double));
    size_t pos = 0;
    for (size_t i = 0; i < n;) {
        if (im[i] == 0.0) {
            A_(s, pos, pos, ld) = re[i];
            pos += 1;
            i += 1;
        } else { /* default spectrum stores the conjugate right after */
            const double a = re[i], b = fabs(im[i]);
            A_(s, pos, pos, ld) = a;
            A_(s, pos, pos + 1, ld) = b;
            A_(s, pos + 1, pos, ld) = -b;
            A_(s, pos + 1, pos + 1, ld) = a;
            pos += 2;
            i += 2;
        }
    }
    teo_philox rng;
    teo_philox_init(&rng, fill_seed);
    for (size_t i = 0; i < n; ++i)
        for (size_t j = i + 1; j < n; ++j) {
            const int in_block = (j == i + 1) && (A_(s, i + 1, i, ld) != 0.0);
            if (!in_block && A_(s, i, j, ld) == 0.0) A_(s, i, j, ld) = teo_philox_uniform_sym(&rng);
        }
    free(re);
    free(im);
}

void teo_hessenberg_random(size_t n, uint64_t seed, double* h, size_t ld) {
    /* generate.cpp:184 (kind hessenberg_random == 4) and :192-198, row-major
     * draw order */
    teo_philox rng;
    teo_philox_init(&rng, seed * 0x9E3779B97F4A7C15ull + 4ull);
    for (size_t j = 0; j < n; ++j) memset(&A_(h, 0, j, ld), 0, n * sizeof(double));
    for (size_t i = 0; i < n; ++i)
        for (size_t j = (i == 0 ? 0 : i - 1); j < n; ++j) A_(h, i, j, ld) = teo_philox_uniform_sym(&rng);
}

/* ======================================================================= */
/* selection, reorder.cpp:21-43, 80-97                                      */

size_t teo_scan_blocks(size_t n, const double* s, size_t ld, uint8_t* sizes) {
    size_t nb = 0;
    for (size_t i = 0; i < n;) {
        if (i + 1 < n && A_(s, i + 1, i, ld) != 0.0) {
            sizes[nb++] = 2;
            i += 2;
        } else {
            sizes[nb++] = 1;
            i += 1;
        }
    }
    return nb;
}

void teo_select_fraction(size_t nb, double fraction, uint64_t seed, uint8_t* flags) {
    const size_t want = (size_t)(fraction * (double)nb);
    size_t* idx = (size_t*)malloc((nb ? nb : 1) * sizeof(size_t));
    for (size_t i = 0; i < nb; ++i) idx[i] = i;
    teo_philox rng;
    teo_philox_init(&rng, seed ^ 0x5e1ec7u);
    for (size_t i = 0; i < want && i + 1 < nb; ++i) {
        const size_t j = i + (size_t)teo_philox_bounded(&rng, nb - i);
        const size_t t = idx[i];
        idx[i] = idx[j];
        idx[j] = t;
    }
    memset(flags, 0, nb);
    for (size_t i = 0; i < want; ++i) flags[idx[i]] = 1;
    free(idx);
}

/* ======================================================================= */
/* dense helpers, dense.hpp:64-82, :145-156                                 */

void teo_gemm(int ta, int tb, size_t m, size_t n, size_t k, double alpha, const double* a,
              size_t lda, const double* b, size_t ldb, double* c, size_t ldc) {
    if (m == 0 || n == 0) return;
    for (size_t j = 0; j < n; ++j) {
        double* cj = c + j * ldc;
        for (size_t p = 0; p < k; ++p) {
            const double sc = alpha * (tb ? b[p * ldb + j] : b[j * ldb + p]);
            if (sc == 0.0) continue;
            if (!ta) {
                const double* ap = a + p * lda;
                for (size_t i = 0; i < m; ++i) cj[i] += sc * ap[i];
            } else {
                for (size_t i = 0; i < m; ++i) cj[i] += sc * a[i * lda + p];
            }
        }
    }
}

static double nrm2(size_t n, const double* x) {
    double mx = 0.0;
    for (size_t i = 0; i < n; ++i) mx = fmax(mx, fabs(x[i]));
    if (mx == 0.0) return 0.0;
    double acc = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double t = x[i] / mx;
        acc += t * t;
    }
    return mx * sqrt(acc);
}

/* ======================================================================= */
/* reflectors and rotations, kernels.cpp:24-120                             */

typedef struct {
    size_t len;
    double v[8];
    double tau;
} refl8; /* reflectors inside the swap kernel have length <= 4 */

/* make_reflector, kernels.cpp:24-58; len <= 8; returns beta */
static double make_refl(const double* x, size_t len, refl8* h) {
    h->len = len;
    h->tau = 0.0;
    for (size_t i = 0; i < len; ++i) h->v[i] = 0.0;
    if (len == 0) return 0.0;
    h->v[0] = 1.0;
    if (len == 1) return x[0];
    const double alpha = x[0];
    const double tail = nrm2(len - 1, x + 1);
    if (tail == 0.0) return alpha == 0.0 ? 0.0 : alpha;
    double beta = -sgn(alpha) * hypot(alpha, tail);
    double tl[8];
    for (size_t i = 1; i < len; ++i) tl[i - 1] = x[i];
    double a = alpha, t;
    int rescale = 0;
    while (fabs(beta) < SAFMIN / EPS && rescale < 20) {
        const double big = 1.0 / (SAFMIN / EPS);
        for (size_t i = 0; i + 1 < len; ++i) tl[i] *= big;
        a *= big;
        t = nrm2(len - 1, tl);
        beta = -sgn(a) * hypot(a, t);
        ++rescale;
    }
    h->tau = (beta - a) / beta;
    const double inv = 1.0 / (a - beta);
    for (size_t i = 1; i < len; ++i) h->v[i] = tl[i - 1] * inv;
    for (int r = 0; r < rescale; ++r) beta *= SAFMIN / EPS;
    return beta;
}

/* apply_reflector_left, kernels.cpp:60-70 */
static void refl_left(double* a, size_t ld, const refl8* h, size_t r0, size_t c0, size_t c1) {
    if (h->tau == 0.0) return;
    for (size_t j = c0; j < c1; ++j) {
        double w = 0.0;
        for (size_t i = 0; i < h->len; ++i) w += h->v[i] * A_(a, r0 + i, j, ld);
        w *= h->tau;
        for (size_t i = 0; i < h->len; ++i) A_(a, r0 + i, j, ld) -= w * h->v[i];
    }
}

/* apply_reflector_right, kernels.cpp:72-82 (kept for the Schur restatement) */
static void refl_right(double* a, size_t ld, const refl8* h, size_t c0, size_t r0, size_t r1)
    __attribute__((unused));
static void refl_right(double* a, size_t ld, const refl8* h, size_t c0, size_t r0, size_t r1) {
    if (h->tau == 0.0) return;
    for (size_t i = r0; i < r1; ++i) {
        double w = 0.0;
        for (size_t j = 0; j < h->len; ++j) w += A_(a, i, c0 + j, ld) * h->v[j];
        w *= h->tau;
        for (size_t j = 0; j < h->len; ++j) A_(a, i, c0 + j, ld) -= w * h->v[j];
    }
}

void teo_make_givens(double a, double b, double* c, double* s) {
    if (b == 0.0) {
        *c = 1.0;
        *s = 0.0;
    } else if (a == 0.0) {
        *c = 0.0;
        *s = 1.0;
    } else {
        const double r = hypot(a, b);
        *c = a / r;
        *s = b / r;
    }
}

/* apply_givens_left on rows (i, j), columns [c0, c1): kernels.cpp:104-111 */
static void rot_rows(double* a, size_t ld, double c, double s, size_t i, size_t j, size_t c0,
                     size_t c1) {
    for (size_t k = c0; k < c1; ++k) {
        const double x = A_(a, i, k, ld), y = A_(a, j, k, ld);
        A_(a, i, k, ld) = c * x + s * y;
        A_(a, j, k, ld) = -s * x + c * y;
    }
}

/* apply_givens_right on columns (i, j), rows [r0, r1): kernels.cpp:113-120 */
static void rot_cols(double* a, size_t ld, double c, double s, size_t i, size_t j, size_t r0,
                     size_t r1) {
    for (size_t k = r0; k < r1; ++k) {
        const double x = A_(a, k, i, ld), y = A_(a, k, j, ld);
        A_(a, k, i, ld) = c * x + s * y;
        A_(a, k, j, ld) = -s * x + c * y;
    }
}

/* ======================================================================= */
/* 2x2 standardization, kernels.cpp:126-219                                 */

void teo_standardize_2x2(double a, double b, double c, double d, double out[10]) {
    double cs = 1.0, sn = 0.0;
    const double mx = fmax(fmax(fabs(a), fabs(b)), fmax(fabs(c), fabs(d)));
    int ex = 0;
    if (mx > 0.0 && (mx > 1e150 || mx < 1e-150)) { /* power-of-two prescale */
        ex = ilogb(mx);
        const double sc = ldexp(1.0, -ex);
        a *= sc; b *= sc; c *= sc; d *= sc;
    }
    if (c == 0.0) {
        /* triangular already */
    } else if (b == 0.0) {
        cs = 0.0;
        sn = 1.0;
        const double ta = a;
        a = d;
        d = ta;
        b = -c;
        c = 0.0;
    } else if ((a - d) == 0.0 && sgn(b) != sgn(c)) {
        /* standard complex pair already */
    } else {
        const double p = 0.5 * (a - d);
        const double qq = b + c;
        const double r2 = hypot(2.0 * p, qq);
        const double sig = sgn(qq);
        const double cos2 = sig * qq / r2;
        const double sin2 = -sig * 2.0 * p / r2;
        cs = sqrt(0.5 * (1.0 + cos2));
        sn = sin2 / (2.0 * cs);
        {
            const double aa = cs * a + sn * c, bb = cs * b + sn * d;
            const double cc = -sn * a + cs * c, dd = -sn * b + cs * d;
            a = aa * cs + bb * sn;
            b = -aa * sn + bb * cs;
            c = cc * cs + dd * sn;
            d = -cc * sn + dd * cs;
        }
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
        } else { /* real pair: rotate onto the eigenvector basis */
            const double sab = sqrt(fabs(b));
            const double sac = sqrt(fabs(c));
            const double pp = sab * sac;
            const double tau = 1.0 / sqrt(fabs(b + c));
            const double cs1 = sab * tau;
            const double sn1 = sgn(c) * sac * tau;
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
    if (c == 0.0) {
        out[6] = out[2]; out[7] = 0.0;
        out[8] = out[5]; out[9] = 0.0;
    } else {
        const double beta = sqrt(fabs(b)) * sqrt(fabs(c)) * back;
        out[6] = out[2]; out[7] = beta;
        out[8] = out[2]; out[9] = -beta;
    }
}

/* ======================================================================= */
/* adjacent block swap, kernels.cpp:419-631                                 */

/* complete-pivoting elimination on a d x d (d <= 4) system, kernels.cpp:419-464.
 * m is taken by value (copied), rhs overwritten by the solution. */
static int gecp_solve(const double* m_in, size_t d, double* rhs, double* rcond) {
    double m[16];
    size_t colperm[4];
    memcpy(m, m_in, d * d * sizeof(double));
    for (size_t i = 0; i < d; ++i) colperm[i] = i;
    double amax = 0.0, smin = 0.0;
    for (size_t k = 0; k < d; ++k) {
        size_t pi = k, pj = k;
        double pv = 0.0;
        for (size_t i = k; i < d; ++i)
            for (size_t j = k; j < d; ++j)
                if (fabs(A_(m, i, j, d)) > pv) {
                    pv = fabs(A_(m, i, j, d));
                    pi = i;
                    pj = j;
                }
        if (k == 0) amax = pv;
        smin = pv;
        if (pv == 0.0) {
            *rcond = 0.0;
            return 0;
        }
        if (pi != k) {
            for (size_t j = 0; j < d; ++j) {
                const double t = A_(m, k, j, d);
                A_(m, k, j, d) = A_(m, pi, j, d);
                A_(m, pi, j, d) = t;
            }
            const double t = rhs[k];
            rhs[k] = rhs[pi];
            rhs[pi] = t;
        }
        if (pj != k) {
            for (size_t i = 0; i < d; ++i) {
                const double t = A_(m, i, k, d);
                A_(m, i, k, d) = A_(m, i, pj, d);
                A_(m, i, pj, d) = t;
            }
            const size_t t = colperm[k];
            colperm[k] = colperm[pj];
            colperm[pj] = t;
        }
        for (size_t i = k + 1; i < d; ++i) {
            const double f = A_(m, i, k, d) / A_(m, k, k, d);
            A_(m, i, k, d) = 0.0;
            for (size_t j = k + 1; j < d; ++j) A_(m, i, j, d) -= f * A_(m, k, j, d);
            rhs[i] -= f * rhs[k];
        }
    }
    double x[4];
    for (size_t kk = d; kk-- > 0;) {
        double acc = rhs[kk];
        for (size_t j = kk + 1; j < d; ++j) acc -= A_(m, kk, j, d) * x[j];
        x[kk] = acc / A_(m, kk, kk, d);
    }
    for (size_t i = 0; i < d; ++i) rhs[colperm[i]] = x[i];
    *rcond = (amax > 0.0) ? smin / amax : 0.0;
    return 1;
}

/* A X - X C = B, Kronecker form + one refinement, kernels.cpp:468-506.
 * a p x p, c q x q, b p x q, x p x q, all col-major with ld = rows. */
static int small_sylvester(size_t p, size_t q, const double* a, const double* c,
                           const double* b, double* x, double* rcond) {
    const size_t d = p * q;
    double k[16], rhs[4];
    for (size_t j = 0; j < q; ++j)
        for (size_t i = 0; i < p; ++i) {
            const size_t row = j * p + i;
            for (size_t l = 0; l < q; ++l)
                for (size_t kk = 0; kk < p; ++kk) {
                    double val = 0.0;
                    if (l == j) val += A_(a, i, kk, p);
                    if (kk == i) val -= A_(c, l, j, q);
                    A_(k, row, l * p + kk, d) = val;
                }
        }
    for (size_t j = 0; j < q; ++j)
        for (size_t i = 0; i < p; ++i) rhs[j * p + i] = A_(b, i, j, p);
    if (!gecp_solve(k, d, rhs, rcond)) return 0;
    for (size_t j = 0; j < q; ++j)
        for (size_t i = 0; i < p; ++i) A_(x, i, j, p) = rhs[j * p + i];
    double r[4], dr[4], rc2;
    memcpy(r, b, p * q * sizeof(double));
    teo_gemm(0, 0, p, q, p, -1.0, a, p, x, p, r, p);
    teo_gemm(0, 0, p, q, q, 1.0, x, p, c, q, r, p);
    for (size_t j = 0; j < q; ++j)
        for (size_t i = 0; i < p; ++i) dr[j * p + i] = A_(r, i, j, p);
    if (gecp_solve(k, d, dr, &rc2))
        for (size_t j = 0; j < q; ++j)
            for (size_t i = 0; i < p; ++i) A_(x, i, j, p) += dr[j * p + i];
    return 1;
}

/* standardize the 2x2 block at bp of an m x m s and fold the rotation into
 * acc, kernels.cpp:616-627 */
static void restandardize(size_t m, double* s, size_t ar, double* acc, size_t bp) {
    double st[10];
    teo_standardize_2x2(A_(s, bp, bp, m), A_(s, bp, bp + 1, m), A_(s, bp + 1, bp, m),
                        A_(s, bp + 1, bp + 1, m), st);
    rot_rows(s, m, st[0], st[1], bp, bp + 1, bp + 2, m);
    rot_cols(s, m, st[0], st[1], bp, bp + 1, 0, bp);
    A_(s, bp, bp, m) = st[2];
    A_(s, bp, bp + 1, m) = st[3];
    A_(s, bp + 1, bp, m) = st[4];
    A_(s, bp + 1, bp + 1, m) = st[5];
    rot_cols(acc, ar, st[0], st[1], bp, bp + 1, 0, ar);
}

int teo_swap_adjacent_blocks(size_t m, double* s, size_t ar, double* acc, size_t pos,
                             size_t p, size_t q) {
    const size_t d = p + q;
    if (p == 1 && q == 1) { /* kernels.cpp:515-527 */
        const double t11 = A_(s, pos, pos, m), t12 = A_(s, pos, pos + 1, m);
        const double t22 = A_(s, pos + 1, pos + 1, m);
        double c, sn;
        teo_make_givens(t12, t22 - t11, &c, &sn);
        if (t12 == 0.0 && t22 - t11 == 0.0) return 0;
        rot_rows(s, m, c, sn, pos, pos + 1, pos + 2, m);
        rot_cols(s, m, c, sn, pos, pos + 1, 0, pos);
        A_(s, pos, pos, m) = t22;
        A_(s, pos + 1, pos + 1, m) = t11;
        A_(s, pos + 1, pos, m) = 0.0;
        rot_cols(acc, ar, c, sn, pos, pos + 1, 0, ar);
        return 0;
    }
    double a[4], c[4], b[4], x[4];
    for (size_t j = 0; j < p; ++j)
        for (size_t i = 0; i < p; ++i) A_(a, i, j, p) = A_(s, pos + i, pos + j, m);
    for (size_t j = 0; j < q; ++j)
        for (size_t i = 0; i < q; ++i) A_(c, i, j, q) = A_(s, pos + p + i, pos + p + j, m);
    for (size_t j = 0; j < q; ++j)
        for (size_t i = 0; i < p; ++i) A_(b, i, j, p) = A_(s, pos + i, pos + p + j, m);
    double rcond = 0.0;
    if (!small_sylvester(p, q, a, c, b, x, &rcond)) return 1;
    if (rcond < pow(EPS, 0.75)) return 1; /* kernels.cpp:540 */

    /* Householder QR of [-X; I] (d x q), kernels.cpp:542-559 */
    double z[16];
    memset(z, 0, sizeof z);
    for (size_t j = 0; j < q; ++j) {
        for (size_t i = 0; i < p; ++i) A_(z, i, j, d) = -A_(x, i, j, p);
        A_(z, p + j, j, d) = 1.0;
    }
    refl8 rf[2];
    for (size_t j = 0; j < q; ++j) {
        double col[4];
        for (size_t i = j; i < d; ++i) col[i - j] = A_(z, i, j, d);
        const double beta = make_refl(col, d - j, &rf[j]);
        A_(z, j, j, d) = beta;
        for (size_t i = j + 1; i < d; ++i) A_(z, i, j, d) = 0.0;
        refl_left(z, d, &rf[j], j, j + 1, q);
    }
    double qd[16];
    memset(qd, 0, sizeof qd);
    for (size_t i = 0; i < d; ++i) A_(qd, i, i, d) = 1.0;
    for (size_t j = q; j-- > 0;) refl_left(qd, d, &rf[j], j, 0, d);

    /* wnew = qd^T W qd and the stability test, kernels.cpp:561-575 */
    double w[16], tmp[16], wn[16];
    for (size_t j = 0; j < d; ++j)
        for (size_t i = 0; i < d; ++i) A_(w, i, j, d) = A_(s, pos + i, pos + j, m);
    memset(tmp, 0, sizeof tmp);
    memset(wn, 0, sizeof wn);
    teo_gemm(1, 0, d, d, d, 1.0, qd, d, w, d, tmp, d);
    teo_gemm(0, 0, d, d, d, 1.0, tmp, d, qd, d, wn, d);
    double wnorm = 0.0, offnorm = 0.0;
    for (size_t j = 0; j < d; ++j)
        for (size_t i = 0; i < d; ++i) {
            wnorm = fmax(wnorm, fabs(A_(w, i, j, d)));
            if (i >= q && j < q && i >= j + 1) offnorm = fmax(offnorm, fabs(A_(wn, i, j, d)));
        }
    if (offnorm > 32.0 * EPS * fmax(wnorm, SAFMIN)) return 1;
    for (size_t j = 0; j < q; ++j)
        for (size_t i = q; i < d; ++i) A_(wn, i, j, d) = 0.0;

    /* commit, kernels.cpp:577-613 */
    for (size_t j = 0; j < d; ++j)
        for (size_t i = 0; i < d; ++i) A_(s, pos + i, pos + j, m) = A_(wn, i, j, d);
    if (pos > 0) {
        double* top = (double*)malloc(pos * d * sizeof(double));
        double* topn = (double*)calloc(pos * d, sizeof(double));
        for (size_t j = 0; j < d; ++j)
            for (size_t i = 0; i < pos; ++i) top[i + j * pos] = A_(s, i, pos + j, m);
        teo_gemm(0, 0, pos, d, d, 1.0, top, pos, qd, d, topn, pos);
        for (size_t j = 0; j < d; ++j)
            for (size_t i = 0; i < pos; ++i) A_(s, i, pos + j, m) = topn[i + j * pos];
        free(top);
        free(topn);
    }
    if (pos + d < m) {
        const size_t rw = m - pos - d;
        double* rg = (double*)malloc(d * rw * sizeof(double));
        double* rgn = (double*)calloc(d * rw, sizeof(double));
        for (size_t j = 0; j < rw; ++j)
            for (size_t i = 0; i < d; ++i) rg[i + j * d] = A_(s, pos + i, pos + d + j, m);
        teo_gemm(1, 0, d, rw, d, 1.0, qd, d, rg, d, rgn, d);
        for (size_t j = 0; j < rw; ++j)
            for (size_t i = 0; i < d; ++i) A_(s, pos + i, pos + d + j, m) = rgn[i + j * d];
        free(rg);
        free(rgn);
    }
    {
        double* av = (double*)malloc(ar * d * sizeof(double));
        double* avn = (double*)calloc(ar * d, sizeof(double));
        for (size_t j = 0; j < d; ++j)
            for (size_t i = 0; i < ar; ++i) av[i + j * ar] = A_(acc, i, pos + j, ar);
        teo_gemm(0, 0, ar, d, d, 1.0, av, ar, qd, d, avn, ar);
        for (size_t j = 0; j < d; ++j)
            for (size_t i = 0; i < ar; ++i) A_(acc, i, pos + j, ar) = avn[i + j * ar];
        free(av);
        free(avn);
    }
    if (q == 2) restandardize(m, s, ar, acc, pos);
    if (p == 2) restandardize(m, s, ar, acc, pos + q);
    return 0;
}

/* ======================================================================= */
/* window_reorder, reorder.cpp:124-194                                      */

int teo_window_reorder(size_t d, double* w, size_t nb, const uint8_t* sizes,
                       const uint8_t* sel, double* acc, uint32_t* order, uint8_t* stuck) {
    for (size_t j = 0; j < d; ++j)
        for (size_t i = 0; i < d; ++i) A_(acc, i, j, d) = (i == j) ? 1.0 : 0.0;
    { /* layout check against the exact-zero subdiagonal, :132-154 */
        size_t row = 0;
        for (size_t k = 0; k < nb; ++k) {
            const size_t sz = sizes[k];
            if (row + sz > d) return 0;
            if (sz == 2 && A_(w, row + 1, row, d) == 0.0) return 0;
            if (row + sz < d && A_(w, row + sz, row + sz - 1, d) != 0.0) return 0;
            row += sz;
        }
        if (row != d) return 0;
    }
    uint32_t* arr = order; /* arrangement[slot] = original local block */
    for (size_t i = 0; i < nb; ++i) {
        arr[i] = (uint32_t)i;
        stuck[i] = 0;
    }
    size_t dest = 0;
    for (size_t blk = 0; blk < nb; ++blk) {
        if (!sel[blk]) continue;
        size_t slot = 0;
        while (arr[slot] != blk) ++slot;
        int st = 0;
        while (slot > dest) {
            const uint32_t pred = arr[slot - 1];
            size_t row = 0;
            for (size_t i = 0; i + 1 < slot; ++i) row += sizes[arr[i]];
            if (teo_swap_adjacent_blocks(d, w, d, acc, row, sizes[pred], sizes[blk])) {
                st = 1;
                break;
            }
            arr[slot - 1] = (uint32_t)blk;
            arr[slot] = pred;
            --slot;
        }
        if (st) stuck[blk] = 1;
        dest = slot + 1;
    }
    return 1;
}

/* ======================================================================= */
/* reorder planner, reorder.cpp:241-324 (iterated assuming success)         */

typedef struct {
    uint8_t size, selected;
    uint32_t orig;
} blockst;

static int plan_push(teo_plan* pl, size_t wtop, size_t wbot, size_t first, size_t count,
                     size_t group, const blockst* bl) {
    if (pl->n_windows == pl->cap_windows) {
        pl->cap_windows = pl->cap_windows ? 2 * pl->cap_windows : 64;
        pl->windows = (teo_window*)realloc(pl->windows, pl->cap_windows * sizeof(teo_window));
        if (!pl->windows) return -1;
    }
    while (pl->n_entries + count > pl->cap_entries) {
        pl->cap_entries = pl->cap_entries ? 2 * pl->cap_entries : 1024;
        pl->sizes = (uint8_t*)realloc(pl->sizes, pl->cap_entries);
        pl->sel = (uint8_t*)realloc(pl->sel, pl->cap_entries);
        if (!pl->sizes || !pl->sel) return -1;
    }
    teo_window* w = &pl->windows[pl->n_windows++];
    w->wtop = wtop;
    w->wbot = wbot;
    w->first_block = first;
    w->count = count;
    w->group = group;
    w->sizes_off = pl->n_entries;
    for (size_t i = 0; i < count; ++i) {
        pl->sizes[pl->n_entries + i] = bl[first + i].size;
        pl->sel[pl->n_entries + i] = bl[first + i].selected;
    }
    pl->n_entries += count;
    return 0;
}

/* Plans one group's chain on state bl/starts (mutated as if every window
 * succeeded).  target/fs/group as in reorder.cpp:243-267. */
static int plan_chain(blockst* bl, size_t* starts, size_t nbk, size_t target, size_t fs,
                      size_t gcount, size_t glast0, size_t ws, size_t gid, teo_plan* pl,
                      long* first_window) {
    size_t gfirst = fs, glast = glast0;
    *first_window = (long)pl->n_windows;
    blockst tmp[4096];
    (void)nbk;
    for (;;) {
        if (gfirst == target) break;
        const size_t gbot = starts[glast + 1];
        size_t wtop = gbot > ws ? gbot - ws : 0;
        if (wtop < starts[target]) wtop = starts[target];
        /* snap up to a block boundary (first block starting at/after wtop) */
        size_t bfirst = gfirst;
        while (bfirst > target && starts[bfirst - 1] >= wtop) --bfirst;
        wtop = starts[bfirst];
        const size_t count = glast - bfirst + 1;
        if (plan_push(pl, wtop, gbot, bfirst, count, gid, bl)) return -1;
        /* pack: selected to the top in order, then the rest in order */
        size_t k = 0;
        for (size_t i = bfirst; i <= glast; ++i)
            if (bl[i].selected) tmp[k++] = bl[i];
        for (size_t i = bfirst; i <= glast; ++i)
            if (!bl[i].selected) tmp[k++] = bl[i];
        for (size_t i = 0; i < count; ++i) {
            bl[bfirst + i] = tmp[i];
            starts[bfirst + i + 1] = starts[bfirst + i] + tmp[i].size;
        }
        gfirst = bfirst;
        glast = bfirst + gcount - 1;
        if (wtop == starts[target]) break;
    }
    return 0;
}

int teo_plan_reorder(size_t nb, const uint8_t* sizes, const uint8_t* flags, size_t ws,
                     teo_plan* pl) {
    memset(pl, 0, sizeof *pl);
    if (ws < 8) ws = 8;
    blockst* bl = (blockst*)malloc((nb + 1) * sizeof(blockst));
    size_t* starts = (size_t*)malloc((nb + 1) * sizeof(size_t));
    starts[0] = 0;
    for (size_t i = 0; i < nb; ++i) {
        bl[i].size = sizes[i];
        bl[i].selected = flags[i] ? 1 : 0;
        bl[i].orig = (uint32_t)i;
        starts[i + 1] = starts[i] + sizes[i];
    }
    size_t target = 0, gid = 0;
    int rc = 0;
    for (;;) {
        while (target < nb && bl[target].selected) ++target;
        size_t fs = target;
        while (fs < nb && !bl[fs].selected) ++fs;
        if (fs == nb) break;
        size_t grows = bl[fs].size, gcount = 1, glast = fs;
        for (size_t g = fs + 1; g < nb; ++g) {
            if (!bl[g].selected) continue;
            const size_t span = starts[g + 1] - starts[fs];
            if (grows + bl[g].size > ws / 2 || span > ws) break;
            grows += bl[g].size;
            ++gcount;
            glast = g;
        }
        long fw;
        if (plan_chain(bl, starts, nb, target, fs, gcount, glast, ws, gid, pl, &fw)) {
            rc = -1;
            break;
        }
        ++gid;
        /* after a successful chain the group's blocks lead at `target`, so
         * the next iteration's prefix skip moves past them */
    }
    pl->n_groups = gid;
    free(bl);
    free(starts);
    return rc;
}

void teo_plan_free(teo_plan* pl) {
    free(pl->windows);
    free(pl->sizes);
    free(pl->sel);
    memset(pl, 0, sizeof *pl);
}

double teo_plan_flops(const teo_plan* pl, size_t n, int with_q) {
    double f = 0.0;
    for (size_t i = 0; i < pl->n_windows; ++i) {
        const double d = (double)(pl->windows[i].wbot - pl->windows[i].wtop);
        const double a = (double)pl->windows[i].wtop, b = (double)pl->windows[i].wbot;
        f += 2.0 * d * d * ((double)n - b) + 2.0 * d * d * a + (with_q ? 2.0 * d * d * (double)n : 0.0);
    }
    return f;
}

/* ======================================================================= */
/* serial reorder_schur, reorder.cpp:215-404                                */

/* left / right panel updates with the window accumulator, window_tasks.cpp:12-30,
 * applied to the whole panel at once (per element identical to the per-tile
 * tasks: the k = d accumulation runs in the same order). */
static void update_left(size_t n, double* s, size_t lds, size_t a, size_t b, const double* acc,
                        double* scratch) {
    const size_t d = b - a, m = n - b;
    if (!m) return;
    double* g = scratch;
    double* gn = scratch + d * m;
    for (size_t j = 0; j < m; ++j)
        for (size_t i = 0; i < d; ++i) g[i + j * d] = A_(s, a + i, b + j, lds);
    memset(gn, 0, d * m * sizeof(double));
    teo_gemm(1, 0, d, m, d, 1.0, acc, d, g, d, gn, d);
    for (size_t j = 0; j < m; ++j)
        for (size_t i = 0; i < d; ++i) A_(s, a + i, b + j, lds) = gn[i + j * d];
}

static void update_right(size_t rows, double* s, size_t lds, size_t a, size_t b,
                         const double* acc, double* scratch) {
    const size_t d = b - a;
    if (!rows) return;
    double* g = scratch;
    double* gn = scratch + d * rows;
    for (size_t j = 0; j < d; ++j)
        for (size_t i = 0; i < rows; ++i) g[i + j * rows] = A_(s, i, a + j, lds);
    memset(gn, 0, d * rows * sizeof(double));
    teo_gemm(0, 0, rows, d, d, 1.0, g, rows, acc, d, gn, rows);
    for (size_t j = 0; j < d; ++j)
        for (size_t i = 0; i < rows; ++i) A_(s, i, a + j, lds) = gn[i + j * rows];
}

long teo_reorder_schur(size_t n, double* s, size_t lds, double* q, size_t ldq, size_t nb,
                       const uint8_t* sizes, const uint8_t* flags, size_t ws, size_t* perm,
                       size_t* rejected, size_t* n_rejected, size_t* plan_out, size_t plan_cap,
                       size_t* n_plan, int* clean, long max_windows) {
    if (ws == 0) ws = n >= 1000 ? 128 : ((n / 8 > 32 ? n / 8 : 32) + 7) / 8 * 8; /* tile */
    if (ws < 8) ws = 8;
    blockst* bl = (blockst*)malloc((nb + 1) * sizeof(blockst));
    size_t* starts = (size_t*)malloc((nb + 1) * sizeof(size_t));
    {
        size_t row = 0;
        for (size_t i = 0; i < nb; ++i) {
            bl[i].size = sizes[i];
            bl[i].selected = flags[i] ? 1 : 0;
            bl[i].orig = (uint32_t)i;
            row += sizes[i];
        }
        if (row != n) {
            free(bl);
            free(starts);
            return -1;
        }
    }
    *n_rejected = 0;
    *n_plan = 0;
    *clean = 1;
    long executed = 0;
    double* win = (double*)malloc(ws * ws * sizeof(double));
    double* acc = (double*)malloc(ws * ws * sizeof(double));
    double* scratch = (double*)malloc(2 * ws * n * sizeof(double) + 16);
    uint32_t* order = (uint32_t*)malloc(ws * sizeof(uint32_t));
    uint8_t* stuck = (uint8_t*)malloc(ws);
    blockst* slice = (blockst*)malloc(ws * sizeof(blockst));
    size_t target = 0;
    teo_plan pl;
    memset(&pl, 0, sizeof pl);
    for (;;) {
        if (max_windows > 0 && executed >= max_windows) break;
        while (target < nb && bl[target].selected) ++target;
        size_t fs = target;
        while (fs < nb && !bl[fs].selected) ++fs;
        if (fs == nb) break;
        starts[0] = 0;
        for (size_t i = 0; i < nb; ++i) starts[i + 1] = starts[i] + bl[i].size;
        size_t grows = bl[fs].size, gcount = 1, glast = fs;
        for (size_t g = fs + 1; g < nb; ++g) {
            if (!bl[g].selected) continue;
            const size_t span = starts[g + 1] - starts[fs];
            if (grows + bl[g].size > ws / 2 || span > ws) break;
            grows += bl[g].size;
            ++gcount;
            glast = g;
        }
        /* plan the chain on a simulated copy (reorder.cpp:277-324) */
        blockst* sim = (blockst*)malloc((nb + 1) * sizeof(blockst));
        size_t* sst = (size_t*)malloc((nb + 1) * sizeof(size_t));
        memcpy(sim, bl, nb * sizeof(blockst));
        memcpy(sst, starts, (nb + 1) * sizeof(size_t));
        pl.n_windows = 0;
        pl.n_entries = 0;
        long fw;
        plan_chain(sim, sst, nb, target, fs, gcount, glast, ws, 0, &pl, &fw);
        free(sim);
        free(sst);
        if (pl.n_windows == 0) continue;
        /* execute every planned window of the chain, in order (the task
         * graph's serial semantics, runtime.hpp:79-82) */
        typedef struct {
            int executed;
            uint32_t order[256];
            uint8_t stuck[256];
        } outcome;
        outcome* oc = (outcome*)malloc(pl.n_windows * sizeof(outcome));
        for (size_t wi = 0; wi < pl.n_windows; ++wi) {
            const teo_window* w = &pl.windows[wi];
            const size_t a = w->wtop, b = w->wbot, d = b - a;
            for (size_t j = 0; j < d; ++j)
                for (size_t i = 0; i < d; ++i) win[i + j * d] = A_(s, a + i, a + j, lds);
            oc[wi].executed = teo_window_reorder(d, win, w->count, pl.sizes + w->sizes_off,
                                                 pl.sel + w->sizes_off, acc, oc[wi].order,
                                                 oc[wi].stuck);
            if (oc[wi].executed)
                for (size_t j = 0; j < d; ++j)
                    for (size_t i = 0; i < d; ++i) A_(s, a + i, a + j, lds) = win[i + j * d];
            update_left(n, s, lds, a, b, acc, scratch);
            update_right(a, s, lds, a, b, acc, scratch);
            if (q) update_right(n, q, ldq, a, b, acc, scratch);
            ++executed;
        }
        /* fold outcomes, reorder.cpp:366-397 */
        for (size_t wi = 0; wi < pl.n_windows; ++wi) {
            const teo_window* w = &pl.windows[wi];
            if (*n_plan < plan_cap) {
                plan_out[3 * *n_plan] = w->wtop;
                plan_out[3 * *n_plan + 1] = w->wbot - w->wtop;
                plan_out[3 * *n_plan + 2] = w->count;
            }
            ++*n_plan;
            if (!oc[wi].executed) break;
            memcpy(slice, bl + w->first_block, w->count * sizeof(blockst));
            for (size_t i = 0; i < w->count; ++i) bl[w->first_block + i] = slice[oc[wi].order[i]];
            int any = 0;
            for (size_t i = 0; i < w->count; ++i)
                if (oc[wi].stuck[i]) {
                    any = 1;
                    rejected[(*n_rejected)++] = slice[i].orig;
                    *clean = 0;
                    for (size_t k = 0; k < nb; ++k)
                        if (bl[k].orig == slice[i].orig) bl[k].selected = 0;
                }
            if (any) break;
        }
        free(oc);
    }
    for (size_t i = 0; i < nb; ++i) perm[bl[i].orig] = i;
    teo_plan_free(&pl);
    free(bl);
    free(starts);
    free(win);
    free(acc);
    free(scratch);
    free(order);
    free(stuck);
    free(slice);
    return executed;
}

/* ======================================================================= */
/* verification, verify.cpp:17-130                                         */

static double frob(size_t n, const double* a) { return nrm2(n * n, a); }

double teo_similarity_residual(size_t n, const double* a, size_t lda, const double* q,
                               size_t ldq, const double* s, size_t lds) {
    /* ||A - Q S Q^T||_F / ||A||_F  (verify.cpp:39-57) */
    double* qs = (double*)calloc(n * n, sizeof(double));
    double* r = (double*)malloc(n * n * sizeof(double));
    double* ad = (double*)malloc(n * n * sizeof(double));
    for (size_t j = 0; j < n; ++j)
        for (size_t i = 0; i < n; ++i) ad[i + j * n] = r[i + j * n] = A_(a, i, j, lda);
    for (size_t k = 0; k < n; ++k)
        for (size_t j = 0; j < n; ++j) {
            const double skj = A_(s, k, j, lds);
            if (skj == 0.0) continue;
            for (size_t i = 0; i < n; ++i) qs[i + j * n] += A_(q, i, k, ldq) * skj;
        }
    for (size_t k = 0; k < n; ++k)
        for (size_t j = 0; j < n; ++j) {
            const double qjk = A_(q, j, k, ldq);
            if (qjk == 0.0) continue;
            for (size_t i = 0; i < n; ++i) r[i + j * n] -= qs[i + k * n] * qjk;
        }
    const double na = frob(n, ad);
    const double res = frob(n, r) / (na > 0.0 ? na : 1.0);
    free(qs);
    free(r);
    free(ad);
    return res;
}

double teo_orthogonality_defect(size_t n, const double* q, size_t ldq) {
    /* ||Q^T Q - I||_F  (verify.cpp:59-69) */
    double* g = (double*)calloc(n * n, sizeof(double));
    for (size_t j = 0; j < n; ++j)
        for (size_t i = 0; i <= j; ++i) {
            double acc = 0.0;
            for (size_t k = 0; k < n; ++k) acc += A_(q, k, i, ldq) * A_(q, k, j, ldq);
            g[i + j * n] = g[j + i * n] = acc;
        }
    for (size_t i = 0; i < n; ++i) g[i + i * n] -= 1.0;
    const double r = frob(n, g);
    free(g);
    return r;
}

int teo_is_standardized(size_t n, const double* s, size_t ld) {
    /* verify.cpp:78-102 */
    for (size_t j = 0; j < n; ++j)
        for (size_t i = j + 2; i < n; ++i)
            if (A_(s, i, j, ld) != 0.0) return 0;
    for (size_t i = 0; i < n;) {
        if (i + 1 < n && A_(s, i + 1, i, ld) != 0.0) {
            if (A_(s, i, i, ld) != A_(s, i + 1, i + 1, ld)) return 0;
            if (!(A_(s, i, i + 1, ld) * A_(s, i + 1, i, ld) < 0.0)) return 0;
            if (i + 2 < n && A_(s, i + 2, i + 1, ld) != 0.0) return 0;
            i += 2;
        } else {
            i += 1;
        }
    }
    return 1;
}

void teo_read_eigenvalues(size_t n, const double* s, size_t ld, double* re, double* im) {
    for (size_t i = 0; i < n;) {
        if (i + 1 < n && A_(s, i + 1, i, ld) != 0.0) {
            const double a = A_(s, i, i, ld), b = A_(s, i, i + 1, ld);
            const double c = A_(s, i + 1, i, ld), d = A_(s, i + 1, i + 1, ld);
            const double m = 0.5 * (a + d), p = 0.5 * (a - d);
            const double disc = p * p + b * c;
            if (disc < 0.0) {
                re[i] = m; im[i] = sqrt(-disc);
                re[i + 1] = m; im[i + 1] = -sqrt(-disc);
            } else {
                const double r = sqrt(disc);
                re[i] = m + r; im[i] = 0.0;
                re[i + 1] = m - r; im[i + 1] = 0.0;
            }
            i += 2;
        } else {
            re[i] = A_(s, i, i, ld);
            im[i] = 0.0;
            i += 1;
        }
    }
}

/* ======================================================================= */
/* Schur reduction path: small_schur (kernels.cpp:223-381), multishift QR   */
/* with AED (schur.cpp:29-399), the tiled driver (schur.cpp:406-906).       */
/* The reference's task graphs have serial semantics (runtime.hpp:79-82):   */
/* every window op is followed by its L/R/Q updates in insertion order,     */
/* which is what the serial restatement below executes.                     */

/* general-length make_reflector (kernels.cpp:24-58); v[len], returns beta */
static double make_refl_n(const double* x, size_t len, double* v, double* tau) {
    *tau = 0.0;
    for (size_t i = 0; i < len; ++i) v[i] = 0.0;
    if (len == 0) return 0.0;
    v[0] = 1.0;
    if (len == 1) return x[0];
    const double alpha = x[0];
    const double tail = nrm2(len - 1, x + 1);
    if (tail == 0.0) return alpha == 0.0 ? 0.0 : alpha;
    double beta = -sgn(alpha) * hypot(alpha, tail);
    double* tl = (double*)malloc((len - 1) * sizeof(double));
    for (size_t i = 1; i < len; ++i) tl[i - 1] = x[i];
    double a = alpha, t;
    int rescale = 0;
    while (fabs(beta) < SAFMIN / EPS && rescale < 20) {
        const double big = 1.0 / (SAFMIN / EPS);
        for (size_t i = 0; i + 1 < len; ++i) tl[i] *= big;
        a *= big;
        t = nrm2(len - 1, tl);
        beta = -sgn(a) * hypot(a, t);
        ++rescale;
    }
    *tau = (beta - a) / beta;
    const double inv = 1.0 / (a - beta);
    for (size_t i = 1; i < len; ++i) v[i] = tl[i - 1] * inv;
    for (int r = 0; r < rescale; ++r) beta *= SAFMIN / EPS;
    free(tl);
    return beta;
}

/* apply_reflector_left / _right (kernels.cpp:60-82) for general length */
static void rl_n(double* a, size_t ld, const double* v, double tau, size_t len, size_t r0,
                 size_t c0, size_t c1) {
    if (tau == 0.0) return;
    for (size_t j = c0; j < c1; ++j) {
        double w = 0.0;
        for (size_t i = 0; i < len; ++i) w += v[i] * A_(a, r0 + i, j, ld);
        w *= tau;
        for (size_t i = 0; i < len; ++i) A_(a, r0 + i, j, ld) -= w * v[i];
    }
}
static void rr_n(double* a, size_t ld, const double* v, double tau, size_t len, size_t c0,
                 size_t r0, size_t r1) {
    if (tau == 0.0) return;
    for (size_t i = r0; i < r1; ++i) {
        double w = 0.0;
        for (size_t j = 0; j < len; ++j) w += A_(a, i, c0 + j, ld) * v[j];
        w *= tau;
        for (size_t j = 0; j < len; ++j) A_(a, i, c0 + j, ld) -= w * v[j];
    }
}

static void set_identity(size_t n, double* q, size_t ld) {
    for (size_t j = 0; j < n; ++j)
        for (size_t i = 0; i < n; ++i) A_(q, i, j, ld) = (i == j) ? 1.0 : 0.0;
}

/* standardize_block_at (kernels.cpp:245-256) == standardize_block_dense
 * (schur.cpp:82-94): h n x n (ld), q qr x n (ld ldq) */
static void std_block(size_t n, double* h, size_t ld, size_t qr, double* q, size_t ldq,
                      size_t p) {
    double st[10];
    teo_standardize_2x2(A_(h, p, p, ld), A_(h, p, p + 1, ld), A_(h, p + 1, p, ld),
                        A_(h, p + 1, p + 1, ld), st);
    rot_rows(h, ld, st[0], st[1], p, p + 1, p + 2, n);
    rot_cols(h, ld, st[0], st[1], p, p + 1, 0, p);
    A_(h, p, p, ld) = st[2];
    A_(h, p, p + 1, ld) = st[3];
    A_(h, p + 1, p, ld) = st[4];
    A_(h, p + 1, p + 1, ld) = st[5];
    rot_cols(q, ldq, st[0], st[1], p, p + 1, 0, qr);
}

static size_t scan_active(size_t n, double* h, size_t ld, size_t ihi, double hnorm) {
    const double smlnum = SAFMIN * ((double)n / EPS);
    size_t l = ihi - 1;
    while (l > 0) {
        double tst = fabs(A_(h, l - 1, l - 1, ld)) + fabs(A_(h, l, l, ld));
        if (tst == 0.0) tst = hnorm;
        if (fabs(A_(h, l, l - 1, ld)) <= fmax(EPS * tst, smlnum)) {
            A_(h, l, l - 1, ld) = 0.0;
            break;
        }
        --l;
    }
    return l;
}

static double hess_norm(size_t n, const double* h, size_t ld) {
    double hn = 0.0;
    for (size_t j = 0; j < n; ++j)
        for (size_t i = 0; i <= (j + 1 < n - 1 ? j + 1 : n - 1); ++i) hn = fmax(hn, fabs(A_(h, i, j, ld)));
    return hn;
}

int teo_small_schur(size_t n, double* h, double* q, size_t* sweeps_out) {
    set_identity(n, q, n);
    size_t sweeps = 0;
    if (sweeps_out) *sweeps_out = 0;
    if (n <= 1) return 1;
    const double hnorm = hess_norm(n, h, n);
    if (hnorm == 0.0) return 1;
    const size_t max_sweeps = 30 * n;
    size_t ihi = n, its = 0;
    while (ihi > 0) {
        if (ihi == 1) {
            ihi = 0;
            its = 0;
            continue;
        }
        const size_t l = scan_active(n, h, n, ihi, hnorm);
        if (l == ihi - 1) {
            ihi = l;
            its = 0;
            continue;
        }
        if (l == ihi - 2) {
            std_block(n, h, n, n, q, n, l);
            ihi = l;
            its = 0;
            continue;
        }
        ++its;
        ++sweeps;
        if (sweeps_out) *sweeps_out = sweeps;
        if (sweeps > max_sweeps) return 0;
        double s11, s12, s21, s22;
        if (its % 10 == 0) {
            const double sp = fabs(A_(h, ihi - 1, ihi - 2, n)) +
                              ((ihi >= l + 3) ? fabs(A_(h, ihi - 2, ihi - 3, n)) : 0.0);
            s11 = 0.75 * sp + A_(h, ihi - 1, ihi - 1, n);
            s12 = -0.4375 * sp;
            s21 = sp;
            s22 = s11;
        } else {
            s11 = A_(h, ihi - 2, ihi - 2, n);
            s12 = A_(h, ihi - 2, ihi - 1, n);
            s21 = A_(h, ihi - 1, ihi - 2, n);
            s22 = A_(h, ihi - 1, ihi - 1, n);
        }
        const double ssum = s11 + s22, sprod = s11 * s22 - s12 * s21;
        double v[3];
        {
            const double a11 = A_(h, l, l, n), a12 = A_(h, l, l + 1, n);
            const double a21 = A_(h, l + 1, l, n), a22 = A_(h, l + 1, l + 1, n);
            const double a32 = A_(h, l + 2, l + 1, n);
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
        for (size_t i = l; i + 3 <= ihi; ++i) {
            double w[3], rv[3], tau;
            if (i == l) {
                w[0] = v[0];
                w[1] = v[1];
                w[2] = v[2];
            } else {
                w[0] = A_(h, i, i - 1, n);
                w[1] = A_(h, i + 1, i - 1, n);
                w[2] = A_(h, i + 2, i - 1, n);
            }
            const double beta = make_refl_n(w, 3, rv, &tau);
            if (i > l) {
                A_(h, i, i - 1, n) = beta;
                A_(h, i + 1, i - 1, n) = 0.0;
                A_(h, i + 2, i - 1, n) = 0.0;
            }
            rl_n(h, n, rv, tau, 3, i, i, n);
            rr_n(h, n, rv, tau, 3, i, 0, (i + 4 < ihi ? i + 4 : ihi));
            rr_n(q, n, rv, tau, 3, i, 0, n);
        }
        {
            const size_t i = ihi - 2;
            double w[2] = {A_(h, i, i - 1, n), A_(h, i + 1, i - 1, n)}, rv[2], tau;
            const double beta = make_refl_n(w, 2, rv, &tau);
            A_(h, i, i - 1, n) = beta;
            A_(h, i + 1, i - 1, n) = 0.0;
            rl_n(h, n, rv, tau, 2, i, i, n);
            rr_n(h, n, rv, tau, 2, i, 0, ihi);
            rr_n(q, n, rv, tau, 2, i, 0, n);
        }
    }
    return 1;
}

/* shift_vector (schur.cpp:29-43) on the window whose (0,0) is h(o,o) */
static void shift_vec(const double* w, size_t ld, size_t rows, size_t o, double ssum, double sprod,
                      double v[3]) {
    const double a11 = A_(w, o, o, ld), a12 = A_(w, o, o + 1, ld);
    const double a21 = A_(w, o + 1, o, ld), a22 = A_(w, o + 1, o + 1, ld);
    const double a32 = (rows > 2) ? A_(w, o + 2, o + 1, ld) : 0.0;
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

/* chase_one_step (schur.cpp:48-63): w d x d (ld d) spans [a, b); acc d x d */
static size_t chase_step(double* w, double* acc, size_t a, size_t b, size_t ihi, size_t r) {
    const size_t d = b - a;
    const size_t len = (ihi - r < 3) ? ihi - r : 3;
    if (len < 2 || r + 1 >= ihi) return ihi - 1;
    const size_t ri = r - a;
    double col[3], v[3], tau;
    for (size_t i = 0; i < len; ++i) col[i] = A_(w, ri + i, ri - 1, d);
    const double beta = make_refl_n(col, len, v, &tau);
    A_(w, ri, ri - 1, d) = beta;
    for (size_t i = 1; i < len; ++i) A_(w, ri + i, ri - 1, d) = 0.0;
    rl_n(w, d, v, tau, len, ri, ri, d);
    rr_n(w, d, v, tau, len, ri, 0, (ri + len + 1 < d ? ri + len + 1 : d));
    rr_n(acc, d, v, tau, len, ri, 0, d);
    return r + 1;
}

/* introduce_one_bulge (schur.cpp:67-78) */
static void intro_bulge(double* w, double* acc, size_t d, double ssum, double sprod) {
    double sv[3], v[3], tau;
    shift_vec(w, d, d, 0, ssum, sprod, sv);
    const size_t len = d < 3 ? d : 3;
    (void)make_refl_n(sv, len, v, &tau);
    rl_n(w, d, v, tau, len, 0, 0, d);
    rr_n(w, d, v, tau, len, 0, 0, (len + 1 < d ? len + 1 : d));
    rr_n(acc, d, v, tau, len, 0, 0, d);
}

static size_t default_shift_count(size_t active) { /* schur.cpp:119-129 */
    size_t m = (active / 16) & ~(size_t)1;
    if (m < 4) m = 4;
    if (m > 64) m = 64;
    if (3 * (m / 2) + 2 > active) {
        const size_t nb = (active >= 6) ? (active - 2) / 3 : 1;
        m = 2 * nb;
        if (m < 2) m = 2;
        if (m > 64) m = 64;
    }
    return m;
}

/* pick_shifts (schur.cpp:97-117); sh/out: (re, im) pairs */
static size_t pick_shifts(const double* sh, size_t nh, size_t m_max, double* out) {
    size_t no = 0, nr = 0;
    double* reals = (double*)malloc((nh + 1) * sizeof(double));
    for (size_t i = 0; i < nh && no + 1 < m_max + 1; ++i) {
        const double re = sh[2 * i], im = sh[2 * i + 1];
        if (im > 0.0) {
            if (no + 2 <= m_max) {
                out[2 * no] = re;
                out[2 * no + 1] = im;
                out[2 * no + 2] = re;
                out[2 * no + 3] = -im;
                no += 2;
            }
        } else if (im == 0.0) {
            reals[nr++] = re;
        }
    }
    for (size_t i = 0; i + 1 < nr && no + 2 <= m_max; i += 2) {
        out[2 * no] = reals[i];
        out[2 * no + 1] = 0.0;
        out[2 * no + 2] = reals[i + 1];
        out[2 * no + 3] = 0.0;
        no += 2;
    }
    free(reals);
    return no;
}

int teo_deflation_check(double spike, double diag_sum, int norm_stable, double wnorm) {
    if (!norm_stable) return spike <= fmax(EPS * diag_sum, SAFMIN); /* schur.cpp:406-411 */
    return spike <= EPS * wnorm;
}

/* apply_similarity_dense (schur.cpp:252-282): h n x n, q n x n (or NULL) */
static void similarity_dense(size_t n, double* h, size_t ldh, size_t qr, double* q, size_t ldq,
                             size_t a, size_t b, const double* acc) {
    const size_t d = b - a;
    double* scratch = (double*)malloc(2 * d * (n > qr ? n : qr) * sizeof(double) + 16);
    if (b < n) update_left(n, h, ldh, a, b, acc, scratch);
    if (a > 0) update_right(a, h, ldh, a, b, acc, scratch);
    if (q) update_right(qr, q, ldq, a, b, acc, scratch);
    free(scratch);
}

static int mshift_dense(size_t n, double* h, double* q, const teo_schur_opts* o, int depth);

/* aed_process_window (schur.cpp:147-248): s (w x w, ld w) is transformed in
 * place; qw (w x w) receives the window similarity. */
static void aed_core(size_t w, double* s, double* qw, double beta, const teo_schur_opts* o,
                     int depth, teo_aed_out* r, double* shifts) {
    memset(r, 0, sizeof *r);
    r->converged = 1;
    const double wnorm = nrm2(w * w, s);
    if (w <= o->small_threshold || depth >= 8) {
        size_t sw;
        r->converged = teo_small_schur(w, s, qw, &sw);
    } else {
        set_identity(w, qw, w);
        r->converged = mshift_dense(w, s, qw, o, depth + 1);
    }
    if (!r->converged) return;
    if (beta == 0.0) {
        r->deflated = w;
        r->newbeta = 0.0;
        r->spike_eliminated = 1;
        return;
    }
    size_t ktop = 0, ns = w;
    while (ns > ktop) {
        const size_t bsize = (ns >= 2 && ns - 2 >= ktop && A_(s, ns - 1, ns - 2, w) != 0.0) ? 2 : 1;
        const size_t bs = ns - bsize;
        double spike = 0.0, dsum = 0.0;
        for (size_t rr = bs; rr < ns; ++rr) {
            spike = fmax(spike, fabs(beta * A_(qw, 0, rr, w)));
            dsum += fabs(A_(s, rr, rr, w));
        }
        if (teo_deflation_check(spike, dsum, o->deflation, wnorm)) {
            ns = bs;
        } else {
            size_t cur = bs;
            int stuck = 0;
            while (cur > ktop) {
                const size_t psize =
                    (cur >= 2 && cur - 2 >= ktop && A_(s, cur - 1, cur - 2, w) != 0.0) ? 2 : 1;
                const size_t ps = cur - psize;
                if (teo_swap_adjacent_blocks(w, s, w, qw, ps, psize, bsize)) {
                    stuck = 1;
                    break;
                }
                cur = ps;
            }
            if (stuck) {
                r->swap_rejected = 1;
                break;
            }
            ktop += bsize;
        }
    }
    r->deflated = w - ns;
    size_t nsh = 0;
    for (size_t i = 0; i < ns;) {
        if (i + 1 < ns && A_(s, i + 1, i, w) != 0.0) {
            const double a = A_(s, i, i, w), b = A_(s, i, i + 1, w), c = A_(s, i + 1, i, w);
            const double im = sqrt(fabs(b)) * sqrt(fabs(c));
            shifts[2 * nsh] = a;
            shifts[2 * nsh + 1] = im;
            shifts[2 * nsh + 2] = a;
            shifts[2 * nsh + 3] = -im;
            nsh += 2;
            i += 2;
        } else {
            shifts[2 * nsh] = A_(s, i, i, w);
            shifts[2 * nsh + 1] = 0.0;
            nsh += 1;
            i += 1;
        }
    }
    r->nshifts = nsh;
    if (ns == 0) {
        r->newbeta = 0.0;
    } else if (ns == 1) {
        r->newbeta = beta * A_(qw, 0, 0, w);
    } else {
        double* spk = (double*)malloc(ns * sizeof(double));
        double* v = (double*)malloc(ns * sizeof(double));
        double tau;
        for (size_t i = 0; i < ns; ++i) spk[i] = beta * A_(qw, 0, i, w);
        r->newbeta = make_refl_n(spk, ns, v, &tau);
        rl_n(s, w, v, tau, ns, 0, 0, w);
        rr_n(s, w, v, tau, ns, 0, 0, ns);
        rr_n(qw, w, v, tau, ns, 0, 0, w);
        for (size_t j = 0; j + 2 < ns; ++j) {
            const size_t len = ns - j - 1;
            double hb;
            for (size_t i = j + 1; i < ns; ++i) spk[i - j - 1] = A_(s, i, j, w);
            hb = make_refl_n(spk, len, v, &tau);
            if (tau == 0.0) continue;
            A_(s, j + 1, j, w) = hb;
            for (size_t i = j + 2; i < ns; ++i) A_(s, i, j, w) = 0.0;
            rl_n(s, w, v, tau, len, j + 1, j + 1, w);
            rr_n(s, w, v, tau, len, j + 1, 0, ns);
            rr_n(qw, w, v, tau, len, j + 1, 0, w);
        }
        free(spk);
        free(v);
    }
    r->spike_eliminated = 1;
}

static void gather(const double* h, size_t ld, size_t r0, size_t c0, size_t m, double* w) {
    for (size_t j = 0; j < m; ++j)
        for (size_t i = 0; i < m; ++i) A_(w, i, j, m) = A_(h, r0 + i, c0 + j, ld);
}
static void scatter(double* h, size_t ld, size_t r0, size_t c0, size_t m, const double* w) {
    for (size_t j = 0; j < m; ++j)
        for (size_t i = 0; i < m; ++i) A_(h, r0 + i, c0 + j, ld) = A_(w, i, j, m);
}

/* multishift_schur_dense (schur.cpp:304-399): h, q n x n (ld n) */
static int mshift_dense(size_t n, double* h, double* q, const teo_schur_opts* o, int depth) {
    if (n <= 1) return 1;
    const double hnorm = hess_norm(n, h, n);
    const size_t limit = 30 * n;
    size_t sweeps = 0, stagnation = 0, ihi = n;
    int ok = 1;
    double* win = (double*)malloc(n * n * sizeof(double));
    double* qw = (double*)malloc(n * n * sizeof(double));
    double* sh = (double*)malloc(2 * (n + 2) * sizeof(double));
    double* picked = (double*)malloc(2 * (n + 70) * sizeof(double));
    while (ihi > 0) {
        if (ihi == 1) {
            ihi = 0;
            continue;
        }
        const size_t l = scan_active(n, h, n, ihi, hnorm);
        const size_t active = ihi - l;
        if (active == 1) {
            ihi = l;
            continue;
        }
        if (active == 2) {
            std_block(n, h, n, n, q, n, l);
            ihi = l;
            continue;
        }
        if (active <= o->small_threshold || depth >= 8) {
            gather(h, n, l, l, active, win);
            if (!teo_small_schur(active, win, qw, NULL)) {
                ok = 0;
                break;
            }
            scatter(h, n, l, l, active, win);
            similarity_dense(n, h, n, n, q, n, l, ihi, qw);
            ihi = l;
            continue;
        }
        const size_t m = o->shift_count ? o->shift_count : default_shift_count(active);
        size_t w = o->aed_window ? o->aed_window : (3 * m) / 2;
        if (w < 4) w = 4;
        if (w > active) w = active;
        const size_t e = ihi - w;
        gather(h, n, e, e, w, win);
        const double beta = (e > l) ? A_(h, e, e - 1, n) : 0.0;
        teo_aed_out core;
        aed_core(w, win, qw, beta, o, depth + 1, &core, sh);
        if (!core.converged) {
            ok = 0;
            break;
        }
        scatter(h, n, e, e, w, win);
        if (e > l) A_(h, e, e - 1, n) = core.newbeta;
        similarity_dense(n, h, n, n, q, n, e, ihi, qw);
        stagnation = (core.deflated == 0) ? stagnation + 1 : 0;
        ihi -= core.deflated;
        if (core.deflated > 0 && 100 * core.deflated >= 14 * w) continue;
        if (ihi - l < 4) continue;
        size_t np = pick_shifts(sh, core.nshifts, m, picked);
        if (stagnation >= 6 || np < 2) {
            const double sp = fabs(A_(h, ihi - 1, ihi - 2, n)) +
                              ((ihi >= l + 3) ? fabs(A_(h, ihi - 2, ihi - 3, n)) : 0.0);
            const double h11 = 0.75 * sp + A_(h, ihi - 1, ihi - 1, n);
            double st[10];
            teo_standardize_2x2(h11, -0.4375 * sp, sp, h11, st);
            picked[0] = st[6];
            picked[1] = st[7];
            picked[2] = st[8];
            picked[3] = st[9];
            np = 2;
            stagnation = 0;
        }
        if (++sweeps > limit) {
            ok = 0;
            break;
        }
        const size_t nb = (np / 2 < (ihi - l - 2) / 3) ? np / 2 : (ihi - l - 2) / 3;
        if (nb == 0) continue;
        const size_t aw = ihi - l;
        gather(h, n, l, l, aw, win);
        set_identity(aw, qw, aw);
        size_t* pos = (size_t*)malloc(nb * sizeof(size_t));
        for (size_t j = 0; j < nb; ++j) {
            /* (s1 + s2).real(), (s1 * s2).real() */
            const double ssum = picked[4 * j] + picked[4 * j + 2];
            const double sprod = picked[4 * j] * picked[4 * j + 2] - picked[4 * j + 1] * picked[4 * j + 3];
            intro_bulge(win, qw, aw, ssum, sprod);
            size_t r = l + 1;
            const size_t target = l + 1 + 3 * (nb - 1 - j);
            while (r < target) r = chase_step(win, qw, l, ihi, ihi, r);
            pos[j] = target;
        }
        for (size_t j = 0; j < nb; ++j) {
            size_t r = pos[j];
            while (r < ihi - 1) r = chase_step(win, qw, l, ihi, ihi, r);
        }
        free(pos);
        scatter(h, n, l, l, aw, win);
        similarity_dense(n, h, n, n, q, n, l, ihi, qw);
    }
    free(win);
    free(qw);
    free(sh);
    free(picked);
    return ok;
}

/* ---- tiled driver, serial semantics ------------------------------------ */

typedef struct {
    size_t n;
    double* h;
    size_t ldh;
    double* q;
    size_t ldq;
    double* scratch;
} teo_mat;

/* apply_window_updates (window_tasks.cpp:89-102) */
static void win_updates(teo_mat* M, size_t a, size_t b, const double* acc) {
    if (b < M->n) update_left(M->n, M->h, M->ldh, a, b, acc, M->scratch);
    if (a > 0) update_right(a, M->h, M->ldh, a, b, acc, M->scratch);
    if (M->q) update_right(M->n, M->q, M->ldq, a, b, acc, M->scratch);
}

/* insert_aed_tasks' window task + updates (schur.cpp:421-459) */
static void aed_round(teo_mat* M, size_t l, size_t ihi, size_t w, const teo_schur_opts* o,
                      teo_aed_out* r, double* shifts) {
    const size_t e = ihi - w;
    double* win = (double*)malloc(w * w * sizeof(double));
    double* qw = (double*)malloc(w * w * sizeof(double));
    gather(M->h, M->ldh, e, e, w, win);
    const double beta = (e > l) ? A_(M->h, e, e - 1, M->ldh) : 0.0;
    aed_core(w, win, qw, beta, o, 0, r, shifts);
    r->window = w;
    if (!r->converged) {
        set_identity(w, qw, w);
    } else {
        scatter(M->h, M->ldh, e, e, w, win);
        if (e > l) A_(M->h, e, e - 1, M->ldh) = r->newbeta;
    }
    win_updates(M, e, ihi, qw);
    free(win);
    free(qw);
}

int teo_aed_step(size_t n, double* h, size_t ldh, double* q, size_t ldq, size_t l, size_t ihi,
                 size_t window, const teo_schur_opts* o, teo_aed_out* r, double* shifts) {
    if (window < 4 || ihi > n || l >= ihi) return -1;
    if (window > ihi - l) window = ihi - l;
    teo_mat M = {n, h, ldh, q, ldq, (double*)malloc(2 * window * n * sizeof(double) + 16)};
    aed_round(&M, l, ihi, window, o, r, shifts);
    free(M.scratch);
    return 0;
}

/* plan_chase + run_chase_window (schur.cpp:484-523), executed in order */
static int chase_chain(teo_mat* M, size_t* positions, size_t npos, size_t ihi, size_t cw) {
    double* w = (double*)malloc(cw * cw * sizeof(double));
    double* acc = (double*)malloc(cw * cw * sizeof(double));
    while (npos) {
        const size_t p_top = positions[npos - 1], p_bot = positions[0];
        const size_t a = p_top - 1;
        const size_t b = (a + cw < ihi) ? a + cw : ihi;
        const int final = (b == ihi);
        size_t hop = 0;
        if (!final) {
            hop = (b >= p_bot + 4) ? (b - 4 - p_bot) : 0;
            if (hop == 0) {
                free(w);
                free(acc);
                return -1;
            }
        }
        const size_t d = b - a;
        gather(M->h, M->ldh, a, a, d, w);
        set_identity(d, acc, d);
        for (size_t j = 0; j < npos; ++j) {
            size_t r = positions[j];
            if (final) {
                while (r < ihi - 1) r = chase_step(w, acc, a, b, ihi, r);
            } else {
                for (size_t s = 0; s < hop; ++s) r = chase_step(w, acc, a, b, ihi, r);
            }
        }
        scatter(M->h, M->ldh, a, a, d, w);
        win_updates(M, a, b, acc);
        if (final) npos = 0;
        else
            for (size_t j = 0; j < npos; ++j) positions[j] += hop;
    }
    free(w);
    free(acc);
    return 0;
}

/* introduce_bulges' window (schur.cpp:628-647 / 851-866); positions out,
 * bottom first */
static void intro_window(teo_mat* M, size_t l, size_t ihi, size_t nb, const double* sh,
                         size_t* positions) {
    const size_t wi = (l + 3 * nb + 2 < ihi) ? l + 3 * nb + 2 : ihi;
    const size_t d = wi - l;
    double* w = (double*)malloc(d * d * sizeof(double));
    double* acc = (double*)malloc(d * d * sizeof(double));
    gather(M->h, M->ldh, l, l, d, w);
    set_identity(d, acc, d);
    for (size_t j = 0; j < nb; ++j) {
        const double ssum = sh[4 * j] + sh[4 * j + 2];
        const double sprod = sh[4 * j] * sh[4 * j + 2] - sh[4 * j + 1] * sh[4 * j + 3];
        intro_bulge(w, acc, d, ssum, sprod);
        size_t r = l + 1;
        const size_t target = l + 1 + 3 * (nb - 1 - j);
        while (r < target) r = chase_step(w, acc, l, wi, ihi, r);
        positions[j] = target; /* decreasing in j: already bottom first */
    }
    scatter(M->h, M->ldh, l, l, d, w);
    win_updates(M, l, wi, acc);
    free(w);
    free(acc);
}

int teo_sweep(size_t n, double* h, size_t ldh, double* q, size_t ldq, size_t l, size_t ihi,
              size_t nshifts, const double* shifts, size_t window_size) {
    if (nshifts < 2 || nshifts % 2 || l + 3 * (nshifts / 2) + 2 > ihi || ihi > n) return -1;
    const size_t nb = nshifts / 2;
    size_t cw = window_size > 3 * nb + 6 ? window_size : 3 * nb + 6;
    teo_mat M = {n, h, ldh, q, ldq, (double*)malloc(2 * cw * n * sizeof(double) + 16)};
    size_t* pos = (size_t*)malloc(nb * sizeof(size_t));
    intro_window(&M, l, ihi, nb, shifts, pos);
    const int rc = chase_chain(&M, pos, nb, ihi, cw);
    free(pos);
    free(M.scratch);
    return rc;
}

/* schur_reduce (schur.cpp:671-906), serial semantics */
int teo_schur_reduce(size_t n, double* h, size_t ldh, double* q, size_t ldq, size_t tile,
                     const teo_schur_opts* o, double* eig, teo_schur_info* info) {
    memset(info, 0, sizeof *info);
    if (!tile) tile = n >= 1000 ? 128 : ((n / 8 > 32 ? n / 8 : 32) + 7) / 8 * 8;
    const size_t limit = o->iteration_limit ? o->iteration_limit : 30 * n;
    const double hnorm = hess_norm(n, h, ldh);
    const size_t cwmax = tile > 3 * 32 + 6 ? tile : 3 * 32 + 6;
    size_t smax = cwmax > 256 ? cwmax : 256;
    teo_mat M = {n, h, ldh, q, ldq, (double*)malloc(2 * smax * n * sizeof(double) + 16)};
    double* shifts = (double*)malloc(2 * 512 * sizeof(double));
    double* picked = (double*)malloc(2 * 520 * sizeof(double));
    size_t* pos = (size_t*)malloc(64 * sizeof(size_t));
    size_t ihi = n, stagnation = 0;
    int have_pending = 0, hard_fail = 0;
    teo_aed_out pend;
    memset(&pend, 0, sizeof pend);
    while (ihi > 0 && !hard_fail) {
        teo_aed_out res;
        int have_aed = 0;
        size_t l = 0;
        memset(&res, 0, sizeof res);
        if (have_pending) {
            res = pend;
            have_pending = 0;
            have_aed = 1;
            if (!res.converged) {
                const size_t w2 = res.window / 2 > 4 ? res.window / 2 : 4;
                l = scan_active(n, h, ldh, ihi, hnorm);
                if (w2 < res.window && ihi - l >= w2) aed_round(&M, l, ihi, w2, o, &res, shifts);
                if (!res.converged) {
                    hard_fail = 1;
                    break;
                }
            }
            ihi -= res.deflated;
            stagnation = (res.deflated == 0) ? stagnation + 1 : 0;
            if (ihi == 0) break;
        }
        l = scan_active(n, h, ldh, ihi, hnorm);
        size_t active = ihi - l;
        if (active == 1) {
            ihi = l;
            have_pending = 0;
            continue;
        }
        if (active == 2) {
            double w[4], qw[4];
            gather(h, ldh, l, l, 2, w);
            set_identity(2, qw, 2);
            std_block(2, w, 2, 2, qw, 2, 0);
            scatter(h, ldh, l, l, 2, w);
            win_updates(&M, l, ihi, qw);
            info->rounds++;
            ihi = l;
            continue;
        }
        if (active <= o->small_threshold) {
            double* w = (double*)malloc(active * active * sizeof(double));
            double* qw = (double*)malloc(active * active * sizeof(double));
            gather(h, ldh, l, l, active, w);
            const int ok = teo_small_schur(active, w, qw, NULL);
            scatter(h, ldh, l, l, active, w);
            win_updates(&M, l, ihi, qw);
            free(w);
            free(qw);
            info->rounds++;
            if (!ok) {
                hard_fail = 1;
                break;
            }
            ihi = l;
            continue;
        }
        if (!have_aed) {
            const size_t m = o->shift_count ? o->shift_count : default_shift_count(active);
            size_t w = o->aed_window ? o->aed_window : (3 * m) / 2;
            if (w < 4) w = 4;
            if (w > active) w = active;
            aed_round(&M, l, ihi, w, o, &res, shifts);
            info->rounds++;
            if (!res.converged) {
                const size_t w2 = w / 2 > 4 ? w / 2 : 4;
                if (w2 < w) aed_round(&M, l, ihi, w2 < ihi - l ? w2 : ihi - l, o, &res, shifts);
                if (!res.converged) {
                    hard_fail = 1;
                    break;
                }
            }
            ihi -= res.deflated;
            stagnation = (res.deflated == 0) ? stagnation + 1 : 0;
            if (ihi == 0) break;
            l = scan_active(n, h, ldh, ihi, hnorm);
            active = ihi - l;
            if (active < 4) continue;
        }
        if (res.deflated > 0 && 100 * res.deflated >= 14 * res.window) continue;
        if (active <= o->small_threshold) continue;
        if (info->sweeps >= limit) {
            hard_fail = 1;
            break;
        }
        info->sweeps++;
        const size_t m_want = o->shift_count ? o->shift_count : default_shift_count(active);
        size_t np = pick_shifts(shifts, res.nshifts, m_want, picked);
        if (stagnation >= 6 || np < 2) {
            const double sp = fabs(A_(h, ihi - 1, ihi - 2, ldh)) +
                              ((ihi >= l + 3) ? fabs(A_(h, ihi - 2, ihi - 3, ldh)) : 0.0);
            const double h11 = 0.75 * sp + A_(h, ihi - 1, ihi - 1, ldh);
            double st[10];
            teo_standardize_2x2(h11, -0.4375 * sp, sp, h11, st);
            picked[0] = st[6];
            picked[1] = st[7];
            picked[2] = st[8];
            picked[3] = st[9];
            np = 2;
            stagnation = 0;
        }
        size_t nb = np / 2 < (active - 2) / 3 ? np / 2 : (active - 2) / 3;
        if (nb == 0) continue;
        info->rounds++;
        intro_window(&M, l, ihi, nb, picked, pos);
        const size_t cw = tile > 3 * nb + 6 ? tile : 3 * nb + 6;
        if (chase_chain(&M, pos, nb, ihi, cw)) {
            hard_fail = 1;
            break;
        }
        {
            const size_t m2 = o->shift_count ? o->shift_count : default_shift_count(active);
            size_t w2 = o->aed_window ? o->aed_window : (3 * m2) / 2;
            if (w2 < 4) w2 = 4;
            if (w2 > active) w2 = active;
            aed_round(&M, l, ihi, w2, o, &pend, shifts);
            have_pending = 1;
        }
    }
    info->converged = !hard_fail;
    info->converged_trailing = n - ihi;
    if (!hard_fail && eig) { /* eigenvalue read-off, schur.cpp:888-904 */
        for (size_t i = 0; i < n;) {
            if (i + 1 < n && A_(h, i + 1, i, ldh) != 0.0) {
                const double a = A_(h, i, i, ldh), b = A_(h, i, i + 1, ldh), c = A_(h, i + 1, i, ldh);
                const double im = sqrt(fabs(b)) * sqrt(fabs(c));
                eig[i] = a;
                eig[n + i] = im;
                eig[i + 1] = a;
                eig[n + i + 1] = -im;
                i += 2;
            } else {
                eig[i] = A_(h, i, i, ldh);
                eig[n + i] = 0.0;
                i += 1;
            }
        }
    }
    free(M.scratch);
    free(shifts);
    free(picked);
    free(pos);
    return 0;
}

/* ======================================================================= */
/* C5 input T (generalized pair; no reference generator exists -- the      */
/* library's gen_pair_t_kernel, restated): upper triangular on the          */
/* synthetic S's block pattern, diagonal 1 + U[0,1) (shared inside a 2x2    */
/* block, in-block T(p, p+1) = 0), strictly upper uniform [-1, 1]; entry    */
/* (i, j) uses the (i*n + j)-th draw of Philox(seed).                       */

static uint64_t philox_u64_at(uint64_t seed, uint64_t k) {
    const uint64_t blk = k >> 1;
    const uint32_t ctr[4] = {(uint32_t)blk, (uint32_t)(blk >> 32), 0u, 0u};
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t out[4];
    teo_philox_round10(ctr, key, out);
    const int i = (int)(k & 1);
    return ((uint64_t)out[2 * i + 1] << 32) | out[2 * i];
}

void teo_pair_t(size_t n, uint64_t seed, double* t, size_t ld) {
    const size_t npairs = n / 4, nreal = n - 2 * npairs;
    for (size_t j = 0; j < n; ++j)
        for (size_t i = 0; i < n; ++i) {
            double v = 0.0;
            const int pair_first_i = i >= nreal && ((i - nreal) & 1) == 0;
            if (i == j) {
                const int second = j >= nreal && ((j - nreal) & 1) == 1;
                const size_t r = second ? i - 1 : i;
                v = 1.0 + (double)(philox_u64_at(seed, (uint64_t)(r * n + r)) >> 11) * (1.0 / 9007199254740992.0);
            } else if (j > i && !(pair_first_i && j == i + 1)) {
                v = 2.0 * ((double)(philox_u64_at(seed, (uint64_t)(i * n + j)) >> 11) * (1.0 / 9007199254740992.0)) - 1.0;
            }
            A_(t, i, j, ld) = v;
        }
}
