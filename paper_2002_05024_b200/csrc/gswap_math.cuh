// gswap_math.cuh -- register-resident arithmetic of one adjacent block swap
// in a generalized real Schur pair (S, T) (sm_100a device code).
//
// SURVEY.md 8a row a16 (config C5): the reference has no generalized path;
// the semantics follow LAPACK DTGEX2 (Kagstrom's direct swapping method):
// for the pencil block
//     (A, B) = ([A11 A12; 0 A22], [B11 B12; 0 B22]),  A11/B11 P x P, A22/B22 Q x Q,
// solve the generalized Sylvester equation
//     A11 R - L A22 = A12,   B11 R - L B22 = B12          (2PQ unknowns)
// by complete-pivoting Gaussian elimination on its Kronecker form (one
// refinement step); then (A, B) = [I -L; 0 I] diag(A11, A22; B11, B22) [I R; 0 I],
// so the deflating subspaces of (A22, B22) are span[-R; I] (right) and
// span[-L; I] (left).  Z (Q) = the orthogonal factor of the QR factorization
// of [-R; I_Q] ([-L; I_Q]); (A, B) <- Q^T (A, B) Z moves (A22, B22) to the
// top.  The swap is rejected when the system is ill conditioned (rcond <
// eps^(3/4)) or when the new lower-left blocks exceed 32 eps max|(A, B)|
// (DTGEX2's weak stability test); otherwise they are set to zero and the new
// 2x2 diagonal blocks of B are made upper triangular by a Givens rotation
// from the left, folded into Q.  Output: Qm, Zm (row-major D x D) and the
// new blocks An, Bn.
#pragma once
#include "swap_math.cuh"

namespace teig {

// full orthogonal D x D factor of the Householder QR of [-X; I_Q] (D x Q),
// X P x Q (row-major) -- the first Q columns span range([-X; I])
template <int P, int Q>
__device__ __forceinline__ void qr_basis(const double (&X)[P][Q], double (&O)[P + Q][P + Q]) {
    constexpr int D = P + Q;
    double z[D][Q];
#pragma unroll
    for (int j = 0; j < Q; ++j) {
#pragma unroll
        for (int i = 0; i < P; ++i) z[i][j] = -X[i][j];
#pragma unroll
        for (int i = 0; i < Q; ++i) z[P + i][j] = (i == j) ? 1.0 : 0.0;
    }
    double v0[D], tau0;
    {
        double col[D];
#pragma unroll
        for (int i = 0; i < D; ++i) col[i] = z[i][0];
        reflector<D>(col, v0, tau0);
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
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) O[i][j] = (i == j) ? 1.0 : 0.0;
    if (Q == 2 && tau1 != 0.0) {  // O = H0 H1: apply H1 then H0 to I
#pragma unroll
        for (int jj = 0; jj < D; ++jj) {
            double w = 0.0;
#pragma unroll
            for (int i = 0; i < D - 1; ++i) w += v1[i] * O[1 + i][jj];
            w *= tau1;
#pragma unroll
            for (int i = 0; i < D - 1; ++i) O[1 + i][jj] -= w * v1[i];
        }
    }
    if (tau0 != 0.0) {
#pragma unroll
        for (int jj = 0; jj < D; ++jj) {
            double w = 0.0;
#pragma unroll
            for (int i = 0; i < D; ++i) w += v0[i] * O[i][jj];
            w *= tau0;
#pragma unroll
            for (int i = 0; i < D; ++i) O[i][jj] -= w * v0[i];
        }
    }
}

// C = U^T M V (D x D, row-major)
template <int D>
__device__ __forceinline__ void sandwich(const double (&U)[D][D], const double (&M)[D][D], const double (&V)[D][D],
                                         double (&C)[D][D]) {
    double tmp[D][D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
            double acc = 0.0;
#pragma unroll
            for (int p = 0; p < D; ++p) acc += U[p][i] * M[p][j];
            tmp[i][j] = acc;
        }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
            double acc = 0.0;
#pragma unroll
            for (int p = 0; p < D; ++p) acc += tmp[i][p] * V[p][j];
            C[i][j] = acc;
        }
}

// make the 2x2 diagonal block of Bn at r upper triangular with a rotation of
// rows r, r+1 (An and Bn, all columns), folded into the columns of Qm
template <int D>
__device__ __forceinline__ void tri_block(int r, double (&An)[D][D], double (&Bn)[D][D], double (&Qm)[D][D]) {
    const double a = Bn[r][r], b = Bn[r + 1][r];
    if (b == 0.0) return;
    const double h = hypot(a, b);
    const double c = a / h, s = b / h;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        const double x = An[r][j], y = An[r + 1][j];
        An[r][j] = c * x + s * y;
        An[r + 1][j] = -s * x + c * y;
        const double u = Bn[r][j], w = Bn[r + 1][j];
        Bn[r][j] = c * u + s * w;
        Bn[r + 1][j] = -s * u + c * w;
    }
    Bn[r + 1][r] = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        const double x = Qm[i][r], y = Qm[i][r + 1];
        Qm[i][r] = c * x + s * y;
        Qm[i][r + 1] = -s * x + c * y;
    }
}

template <int P, int Q>
__device__ __forceinline__ bool gswap(const double (&A)[P + Q][P + Q], const double (&B)[P + Q][P + Q],
                                      double (&Qm)[P + Q][P + Q], double (&Zm)[P + Q][P + Q],
                                      double (&An)[P + Q][P + Q], double (&Bn)[P + Q][P + Q]) {
    constexpr int D = P + Q;
    constexpr int PQ = P * Q;
    constexpr int K = 2 * PQ;
    double Km[K][K], rhs[K];
#pragma unroll
    for (int r = 0; r < K; ++r)
#pragma unroll
        for (int c = 0; c < K; ++c) Km[r][c] = 0.0;
#pragma unroll
    for (int j = 0; j < Q; ++j)
#pragma unroll
        for (int i = 0; i < P; ++i) {
            const int r1 = j * P + i, r2 = PQ + j * P + i;
#pragma unroll
            for (int k = 0; k < P; ++k) {  // A11 R, B11 R
                Km[r1][j * P + k] = A[i][k];
                Km[r2][j * P + k] = B[i][k];
            }
#pragma unroll
            for (int k = 0; k < Q; ++k) {  // - L A22, - L B22
                Km[r1][PQ + k * P + i] = -A[P + k][P + j];
                Km[r2][PQ + k * P + i] = -B[P + k][P + j];
            }
            rhs[r1] = A[i][P + j];
            rhs[r2] = B[i][P + j];
        }
    GecpLU<K> lu;
    lu.factor(Km);
    if (!lu.ok || lu.rcond < 1.8189894035458565e-12) return false;  // eps^(3/4)
    double x[K];
#pragma unroll
    for (int i = 0; i < K; ++i) x[i] = rhs[i];
    lu.solve(x);
    {  // one refinement step on the residual
        double res[K];
#pragma unroll
        for (int r = 0; r < K; ++r) {
            double acc = rhs[r];
#pragma unroll
            for (int c = 0; c < K; ++c) acc -= Km[r][c] * x[c];
            res[r] = acc;
        }
        lu.solve(res);
#pragma unroll
        for (int i = 0; i < K; ++i) x[i] += res[i];
    }
    double R[P][Q], L[P][Q];
#pragma unroll
    for (int j = 0; j < Q; ++j)
#pragma unroll
        for (int i = 0; i < P; ++i) {
            R[i][j] = x[j * P + i];
            L[i][j] = x[PQ + j * P + i];
        }
    qr_basis<P, Q>(R, Zm);
    qr_basis<P, Q>(L, Qm);
    sandwich<D>(Qm, A, Zm, An);
    sandwich<D>(Qm, B, Zm, Bn);
    double nrm = 0.0, off = 0.0;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
            nrm = fmax(nrm, fmax(fabs(A[i][j]), fabs(B[i][j])));
            if (i >= Q && j < Q) off = fmax(off, fmax(fabs(An[i][j]), fabs(Bn[i][j])));
        }
    if (off > 32.0 * kEpsD * fmax(nrm, kSafeMinD)) return false;
#pragma unroll
    for (int i = Q; i < D; ++i)
#pragma unroll
        for (int j = 0; j < Q; ++j) {
            An[i][j] = 0.0;
            Bn[i][j] = 0.0;
        }
    // 1x1 blocks keep a zero subdiagonal coupling; B's 2x2 blocks triangular
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j)
            if (i > j + 1) An[i][j] = 0.0;
    if (Q == 2) tri_block<D>(0, An, Bn, Qm);
    if (P == 2) tri_block<D>(Q, An, Bn, Qm);
    if (Q == 1 && P == 2) An[1][0] = 0.0;  // the new upper 1x1 block is decoupled
    if (Q == 2 && P == 1) An[2][1] = 0.0;
    if (Q == 1 && P == 1) An[1][0] = 0.0;
    return true;
}

}  // namespace teig
