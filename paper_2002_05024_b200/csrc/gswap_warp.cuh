// gswap_warp.cuh -- one adjacent block swap of a generalized Schur pair
// (S, T), decided by a whole warp (sm_100a device code).
//
// Same arithmetic as gswap<P, Q> (gswap_math.cuh: DTGEX2 semantics, the
// generalized Sylvester equation in Kronecker form by complete-pivoting
// Gaussian elimination plus one refinement step, QR of the deflating-subspace
// bases, the weak stability test, triangularisation of B's 2x2 blocks), with
// every element-wise stage spread over the lanes instead of one thread:
//   * the K x K elimination (K = 2PQ <= 8): one entry per lane and step, the
//     pivot by a warp max and a ballot (the first entry of maximal modulus
//     in row-major order, the serial scan's choice), interchanges and the
//     rank-1 update in parallel;
// Every value sees the single-thread code's operations in its order: the
// outputs are bitwise those of gswap<P, Q> (tools/microbench/gswap_check.cu).
// 1x1|1x1 pairs (K = 2) run the single-thread code in lane 0, which is
// faster there than the warp's synchronisation.
//   * the triangular solves (dependent chains) redundantly in every lane,
//     from broadcast reads of the factors, each lane keeping one component;
//     the refinement residual one row per lane;
//   * the two QR bases (Z from R, Q from L) in lanes 0 and 1 at once;
//   * U^T M V for (A, B) by lanes 0-15 / 16-31, one output element each.
// The single-thread version's latency (a 255-register frame with local
// spills, ~40k cycles for a 2x2|2x2 pair) was the generalized window
// kernel's critical path; this one runs in a few thousand cycles, and since
// every pair now takes one warp, the pairs of a step spread over all warps.
#pragma once
#include "gswap_math.cuh"

namespace teig {

struct GSwapScratch {
    double A[16], B[16];  // the pair's D x D diagonal blocks (row-major)
    double K0[64];        // Kronecker matrix as built (residual of the refinement)
    double U[64];         // elimination in progress (row-major K x K)
    double F[64];         // multipliers F[i][s]
    double T[2][16];      // U^T M temporaries (A, B)
    double X[8];          // the Sylvester solution (R then L)
};

template <int P, int Q>
__device__ __forceinline__ bool wgswap(const double* Sw, const double* Tw, int ld, int pos, GSwapScratch& w, int lane,
                                       double* Qo, double* Zo, double* Ao, double* Bo) {
    constexpr int D = P + Q, PQ = P * Q, K = 2 * PQ, KK = K * K;
    constexpr unsigned kFull = 0xffffffffu;
    if constexpr (P == 1 && Q == 1) {
        int ok = 0;
        if (lane == 0) {
            double A[2][2], B[2][2], Qm[2][2], Zm[2][2], An[2][2], Bn[2][2];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    A[i][j] = Sw[(pos + i) + (pos + j) * ld];
                    B[i][j] = Tw[(pos + i) + (pos + j) * ld];
                }
            ok = gswap<1, 1>(A, B, Qm, Zm, An, Bn) ? 1 : 0;
            if (ok)
#pragma unroll
                for (int i = 0; i < 2; ++i)
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        Qo[i * 2 + j] = Qm[i][j];
                        Zo[i * 2 + j] = Zm[i][j];
                        Ao[i * 2 + j] = An[i][j];
                        Bo[i * 2 + j] = Bn[i][j];
                    }
        }
        ok = __shfl_sync(kFull, ok, 0);
        return ok != 0;
    }
    __syncwarp();  // the previous pair's reads of the scratch are done
    if (lane < D * D) {
        const int i = lane / D, j = lane % D;
        w.A[lane] = Sw[(pos + i) + (pos + j) * ld];
        w.B[lane] = Tw[(pos + i) + (pos + j) * ld];
    }
    __syncwarp();
    // Kronecker form: row j*P+i of the A (then B) equation;
    // unknowns R (j*P+k) then L (PQ + k*P+i), as in gswap
    for (int e = lane; e < KK; e += 32) {
        const int r = e / K, c = e % K;
        const bool second = r >= PQ;
        const int rr = second ? r - PQ : r;
        const int j = rr / P, i = rr % P;
        const double* M = second ? w.B : w.A;
        double v = 0.0;
        if (c < PQ) {
            if (c / P == j) v = M[i * D + c % P];
        } else {
            const int cc = c - PQ;
            if (cc % P == i) v = -M[(P + cc / P) * D + P + j];
        }
        w.K0[e] = v;
        w.U[e] = v;
    }
    __syncwarp();
    // complete-pivoting elimination (GecpLU::factor's operations per entry)
    double amax = 0.0, smin = 0.0;
    bool ok = true;
    int piv_r[K], piv_c[K];
#pragma unroll
    for (int s = 0; s < K; ++s) {
        // pivot: the first entry (row-major) of maximal modulus in U[s:, s:]
        // -- the serial scan's choice: warp max, then a ballot for the lowest
        // index attaining it (NaN never wins; an all-zero block keeps (s, s))
        double v0 = -1.0, v1 = -1.0;
        if (lane < KK && (lane / K) >= s && (lane % K) >= s) v0 = fabs(w.U[lane]);
        if (KK > 32 && lane + 32 < KK && ((lane + 32) / K) >= s && ((lane + 32) % K) >= s) v1 = fabs(w.U[lane + 32]);
        double mx = fmax(v0, v1);  // fmax drops a NaN operand
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(kFull, mx, o));
        const unsigned b0 = __ballot_sync(kFull, v0 == mx), b1 = __ballot_sync(kFull, v1 == mx);
        int bidx = b0 ? __ffs(b0) - 1 : 32 + __ffs(b1) - 1;
        if (!(mx > 0.0)) bidx = s * K + s;
        const double bv = mx > 0.0 ? mx : 0.0;
        __syncwarp();  // the search's reads before the interchanges' writes
        const int bi = bidx / K, bj = bidx % K;
        piv_r[s] = bi;
        piv_c[s] = bj;
        if (s == 0) amax = bv;
        smin = bv;
        if (bv == 0.0) ok = false;
        if (bi != s && lane < K) {
            const double t = w.U[s * K + lane];
            w.U[s * K + lane] = w.U[bi * K + lane];
            w.U[bi * K + lane] = t;
        }
        __syncwarp();
        if (bj != s && lane < K) {
            const double t = w.U[lane * K + s];
            w.U[lane * K + s] = w.U[lane * K + bj];
            w.U[lane * K + bj] = t;
        }
        __syncwarp();
        double nv[(KK + 31) / 32];
#pragma unroll
        for (int t = 0; t < (KK + 31) / 32; ++t) {
            const int e = lane + 32 * t;
            const int r = e / K, c = e % K;
            nv[t] = 0.0;
            if (e < KK && r > s && c >= s) {
                const double fm = w.U[r * K + s] / w.U[s * K + s];
                if (c == s) w.F[r * K + s] = fm;
                else nv[t] = w.U[e] - fm * w.U[s * K + c];
            }
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < (KK + 31) / 32; ++t) {
            const int e = lane + 32 * t;
            const int r = e / K, c = e % K;
            if (e < KK && r > s && c >= s) w.U[e] = nv[t];
        }
        __syncwarp();
    }
    const double rcond = ok ? ((amax > 0.0) ? smin / amax : 0.0) : 0.0;
    if (!ok || rcond < 1.8189894035458565e-12) return false;  // eps^(3/4), warp-uniform
    // the column interchanges undone (GecpLU::solve's cp): lane t takes
    // component src of the back-substituted vector
    int src = 0;
    {
        int cp[K];
#pragma unroll
        for (int i = 0; i < K; ++i) cp[i] = i;
        // (interchanges as select chains: written as conditional swaps the
        // compiler turned them into dynamically indexed local-memory swaps)
#pragma unroll
        for (int s = 0; s < K; ++s) {
            const int p = piv_c[s], cs = cp[s];
            int cq = cs;
#pragma unroll
            for (int j = s + 1; j < K; ++j) cq = (p == j) ? cp[j] : cq;
#pragma unroll
            for (int j = s + 1; j < K; ++j) cp[j] = (p == j) ? cs : cp[j];
            cp[s] = cq;
        }
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (cp[i] == lane) src = i;
    }
    // GecpLU::solve's operations, every lane on the whole vector (broadcast
    // reads of the factors), each lane keeping its own component
    // (everything by value -- the pivots and the vector stay in registers;
    // a by-reference capture put them in local memory)
    struct Vec {
        double v[K];
    };
    auto solve = [=, &w](Vec xv) -> double {
        double (&x)[K] = xv.v;
#pragma unroll
        for (int s = 0; s < K; ++s) {
            const int p = piv_r[s];
            const double xs = x[s];
            double xq = xs;
#pragma unroll
            for (int i = s + 1; i < K; ++i) xq = (p == i) ? x[i] : xq;
#pragma unroll
            for (int i = s + 1; i < K; ++i) x[i] = (p == i) ? xs : x[i];
            x[s] = xq;
#pragma unroll
            for (int i = s + 1; i < K; ++i) x[i] -= w.F[i * K + s] * x[s];
        }
        double y[K];
#pragma unroll
        for (int kk = K - 1; kk >= 0; --kk) {
            double acc = x[kk];
#pragma unroll
            for (int j = kk + 1; j < K; ++j) acc -= w.U[kk * K + j] * y[j];
            y[kk] = acc / w.U[kk * K + kk];
        }
        // y[src] by a tree of selects on src's bits (a linear select chain
        // was turned back into an indexed local-memory load)
        double t2[K];
#pragma unroll
        for (int i = 0; i < K; ++i) t2[i] = y[i];
#pragma unroll
        for (int w2 = K / 2, bit = 0; w2 >= 1; w2 >>= 1, ++bit) {
            const bool hi = (src >> bit) & 1;
#pragma unroll
            for (int i = 0; i < w2; ++i) t2[i] = hi ? t2[2 * i + 1] : t2[2 * i];
        }
        return t2[0];
    };
    double rhs[K];
#pragma unroll
    for (int j = 0; j < Q; ++j)
#pragma unroll
        for (int i = 0; i < P; ++i) {
            rhs[j * P + i] = w.A[i * D + P + j];
            rhs[PQ + j * P + i] = w.B[i * D + P + j];
        }
    double x;
    {
        Vec t;
#pragma unroll
        for (int i = 0; i < K; ++i) t.v[i] = rhs[i];
        x = solve(t);  // lane t < K: x_t
    }
    {  // one refinement step: residual row per lane (serial order), gathered
        double res = 0.0;
#pragma unroll
        for (int r = 0; r < K; ++r)
            if (lane == r) res = rhs[r];
#pragma unroll
        for (int c = 0; c < K; ++c) {
            const double xc = __shfl_sync(kFull, x, c);
            if (lane < K) res -= w.K0[lane * K + c] * xc;
        }
        Vec t;
#pragma unroll
        for (int i = 0; i < K; ++i) t.v[i] = __shfl_sync(kFull, res, i);
        x += solve(t);
    }
    if (lane < K) w.X[lane] = x;
    __syncwarp();
    // orthogonal bases: lane 0 Z (from R), lane 1 Q (from L)
    if (lane < 2) {
        double X[P][Q], O[D][D];
#pragma unroll
        for (int j = 0; j < Q; ++j)
#pragma unroll
            for (int i = 0; i < P; ++i) X[i][j] = w.X[(lane ? PQ : 0) + j * P + i];
        qr_basis<P, Q>(X, O);
        double* dst = lane ? Qo : Zo;
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) dst[i * D + j] = O[i][j];
    }
    __syncwarp();
    // (An, Bn) = Q^T (A, B) Z: lanes 0-15 A, 16-31 B, one element each
    const int half = lane >> 4, idx = lane & 15;
    const int ei = idx / D, ej = idx % D;
    const bool own = idx < D * D;
    const double* M = half ? w.B : w.A;
    if (own) {
        double acc = 0.0;
#pragma unroll
        for (int p = 0; p < D; ++p) acc += Qo[p * D + ei] * M[p * D + ej];
        w.T[half][idx] = acc;
    }
    __syncwarp();
    double cv = 0.0;
    if (own) {
#pragma unroll
        for (int p = 0; p < D; ++p) cv += w.T[half][ei * D + p] * Zo[p * D + ej];
    }
    // weak stability test: new lower-left blocks vs 32 eps max|(A, B)|
    double nrm = own ? fabs(M[idx]) : 0.0;
    double off = (own && ei >= Q && ej < Q) ? fabs(cv) : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        nrm = fmax(nrm, __shfl_xor_sync(kFull, nrm, o));
        off = fmax(off, __shfl_xor_sync(kFull, off, o));
    }
    if (off > 32.0 * kEpsD * fmax(nrm, kSafeMinD)) return false;
    if (ei >= Q && ej < Q) cv = 0.0;
    if (!half && ei > ej + 1) cv = 0.0;
    if (own) (half ? Bo : Ao)[idx] = cv;
    __syncwarp();
    // B's 2x2 diagonal blocks upper triangular: rotations of rows r, r+1
    // (An, Bn, all columns) folded into columns r, r+1 of Q (tri_block)
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const int r = (t == 0) ? 0 : Q;
        if (t == 0 ? Q != 2 : P != 2) continue;
        const double a = Bo[r * D + r], b = Bo[(r + 1) * D + r];
        if (b == 0.0) continue;  // warp-uniform
        const double h = hypot(a, b);
        const double c = a / h, s = b / h;
        if (lane < D) {
            const int j = lane;
            const double xa = Ao[r * D + j], ya = Ao[(r + 1) * D + j];
            Ao[r * D + j] = c * xa + s * ya;
            Ao[(r + 1) * D + j] = -s * xa + c * ya;
            const double u = Bo[r * D + j], v = Bo[(r + 1) * D + j];
            Bo[r * D + j] = c * u + s * v;
            Bo[(r + 1) * D + j] = -s * u + c * v;
        } else if (lane < 2 * D) {
            const int i = lane - D;
            const double xq = Qo[i * D + r], yq = Qo[i * D + r + 1];
            Qo[i * D + r] = c * xq + s * yq;
            Qo[i * D + r + 1] = -s * xq + c * yq;
        }
        __syncwarp();
        if (lane == 0) Bo[(r + 1) * D + r] = 0.0;
        __syncwarp();
    }
    if (lane == 0) {  // 1x1 blocks keep a zero subdiagonal coupling
        if (Q == 1 && P == 2) Ao[1 * D + 0] = 0.0;
        if (Q == 2 && P == 1) Ao[2 * D + 1] = 0.0;
        if (Q == 1 && P == 1) Ao[1 * D + 0] = 0.0;
    }
    __syncwarp();
    return true;
}

}  // namespace teig
