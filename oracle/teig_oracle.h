/*
 * oracle/teig_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C CPU restatement of the reference (taskeig, /root/reference/proj)
 * for the window-based off-diagonal update path.  Used exclusively as the
 * checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * reference legs.  The product (paper_2002_05024_b200/) never links it.
 *
 * Parity is PINNED: tests/test_oracle.py checks this restatement bit-for-bit
 * against the unmodified reference compiled from its own sources
 * (oracle/_ref/libtaskeig_ref.so, see oracle/Makefile), against the Philox
 * known-answer vectors of tests/test_generators.cpp:12-21, and against the
 * committed golden fixtures in tests/golden/.
 *
 * Storage: all matrices are COLUMN-MAJOR with an explicit leading dimension
 * (element (i,j) at a[i + j*ld]), the orientation of the reference's tiles
 * and DenseMatrix (tiled_matrix.hpp:27-35, dense.hpp:33-36).
 */
#ifndef TEIG_ORACLE_H
#define TEIG_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- Philox4x32-10 (philox.hpp:18-84) ---------------------------------- */
typedef struct {
    uint32_t key[2];
    uint64_t counter;
    uint32_t buf[4];
    int have;
} teo_philox;

void teo_philox_round10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
void teo_philox_init(teo_philox* p, uint64_t seed);
uint64_t teo_philox_next_u64(teo_philox* p);
double teo_philox_uniform_sym(teo_philox* p);
double teo_philox_uniform01(teo_philox* p);
uint64_t teo_philox_bounded(teo_philox* p, uint64_t n);

/* ---- generators (generate.cpp) ----------------------------------------- */
/* default_spectrum (generate.cpp:68-91): re[n], im[n]. */
void teo_default_spectrum(size_t n, double* re, double* im);
/* build_quasi_triangular (generate.cpp:115-150) on the default spectrum with
 * the upper fill drawn from Philox(fill_seed); writes col-major s (ld). */
void teo_schur_input(size_t n, uint64_t fill_seed, double* s, size_t ld);
/* the fill seed generate() would use for known_spectrum (generate.cpp:184) */
uint64_t teo_known_spectrum_seed(uint64_t seed);
/* generate(hessenberg_random) (generate.cpp:192-198), col-major out. */
void teo_hessenberg_random(size_t n, uint64_t seed, double* h, size_t ld);

/* ---- selection (reorder.cpp:21-43, 80-97) ------------------------------ */
/* exact-zero subdiagonal block scan; sizes[] (1/2) out, returns #blocks */
size_t teo_scan_blocks(size_t n, const double* s, size_t ld, uint8_t* sizes);
void teo_select_fraction(size_t nb, double fraction, uint64_t seed, uint8_t* flags);

/* ---- window-local kernels (kernels.cpp) -------------------------------- */
/* make_givens (kernels.cpp:86-102) */
void teo_make_givens(double a, double b, double* c, double* s);
/* standardize_2x2 (kernels.cpp:126-219).  out = {cs, sn, a, b, c, d, l1re,
 * l1im, l2re, l2im} */
void teo_standardize_2x2(double a, double b, double c, double d, double out[10]);
/* swap_adjacent_blocks (kernels.cpp:510-631): m x m window s (ld m), acc
 * ar x m (ld ar).  0 ok, 1 rejected. */
int teo_swap_adjacent_blocks(size_t m, double* s, size_t ar, double* acc, size_t pos,
                             size_t p, size_t q);
/* window_reorder (reorder.cpp:124-194); acc (d x d) is overwritten.
 * Returns 1 executed, 0 layout mismatch (acc = I). */
int teo_window_reorder(size_t d, double* w, size_t nb, const uint8_t* sizes,
                       const uint8_t* sel, double* acc, uint32_t* order, uint8_t* stuck);

/* ---- reorder planner + serial driver (reorder.cpp:215-404) ------------- */
typedef struct {
    size_t wtop, wbot;        /* rows [wtop, wbot) */
    size_t first_block, count;/* block slots covered, in planning state */
    size_t group;             /* index of the group (chain) the window belongs to */
    size_t sizes_off;         /* offset into the plan's sizes/sel arrays */
} teo_window;

typedef struct {
    size_t n_windows, cap_windows;
    teo_window* windows;
    size_t n_entries, cap_entries;
    uint8_t* sizes;           /* per window: count block sizes */
    uint8_t* sel;             /* per window: count selection flags */
    size_t n_groups;
} teo_plan;

/* Full plan assuming every swap succeeds (the reference's per-group chain
 * simulation, reorder.cpp:241-324, iterated over all groups). */
int teo_plan_reorder(size_t nb, const uint8_t* sizes, const uint8_t* flags, size_t ws,
                     teo_plan* plan);
void teo_plan_free(teo_plan* plan);
/* sum over windows of 2d^2(n-b) + 2d^2 a + 2d^2 n */
double teo_plan_flops(const teo_plan* plan, size_t n, int with_q);

/* Serial CPU reorder_schur.  s (ld lds), q (ld ldq or NULL).  perm[nb],
 * rejected[nb] out.  plan_out: 3 size_t per window (position, extent,
 * moved_blocks) up to plan_cap.  max_windows > 0 stops after that many
 * executed windows (bounded CPU-baseline samples); returns the number of
 * windows executed, or -1 on bad arguments. */
long teo_reorder_schur(size_t n, double* s, size_t lds, double* q, size_t ldq, size_t nb,
                       const uint8_t* sizes, const uint8_t* flags, size_t ws, size_t* perm,
                       size_t* rejected, size_t* n_rejected, size_t* plan_out, size_t plan_cap,
                       size_t* n_plan, int* clean, long max_windows);

/* C(m x n) += alpha op(A) op(B), k ascending, zero alpha*b terms skipped
 * (dense.hpp:64-82). */
void teo_gemm(int ta, int tb, size_t m, size_t n, size_t k, double alpha, const double* a,
              size_t lda, const double* b, size_t ldb, double* c, size_t ldc);


/* ---- Schur reduction path (schur.cpp, kernels.cpp:223-381) ------------- */
typedef struct {
    int deflation;          /* 0 classic, 1 norm-stable (SchurOptions, schur.hpp:20-29) */
    size_t shift_count;     /* 0: default_shift_count */
    size_t aed_window;      /* 0: 3m/2 */
    size_t iteration_limit; /* 0: 30 n */
    size_t small_threshold; /* 64 */
} teo_schur_opts;

typedef struct { /* AedResult (schur.hpp:32-39) + the window's new spike */
    size_t window, deflated, nshifts;
    int spike_eliminated, converged, swap_rejected;
    double newbeta;
} teo_aed_out;

typedef struct {
    size_t sweeps, rounds, converged_trailing;
    int converged;
} teo_schur_info;

/* small_schur (kernels.cpp:260-381): h k x k (ld k) in place, q (k x k) out.
 * Returns 1 converged. */
int teo_small_schur(size_t k, double* h, double* q, size_t* sweeps);
int teo_deflation_check(double spike, double diag_sum, int norm_stable, double wnorm);
/* aed_step (schur.cpp:599-609); shifts: 2*window doubles (re, im) out */
int teo_aed_step(size_t n, double* h, size_t ldh, double* q, size_t ldq, size_t l, size_t ihi,
                 size_t window, const teo_schur_opts* o, teo_aed_out* r, double* shifts);
/* introduce_bulges + chase_bulges (schur.cpp:611-669); shifts: (re, im) */
int teo_sweep(size_t n, double* h, size_t ldh, double* q, size_t ldq, size_t l, size_t ihi,
              size_t nshifts, const double* shifts, size_t window_size);
/* schur_reduce (schur.cpp:671-906), serial semantics; tile 0: default_tile_size(n).
 * eig: re[n] then im[n] (or NULL). */
int teo_schur_reduce(size_t n, double* h, size_t ldh, double* q, size_t ldq, size_t tile,
                     const teo_schur_opts* o, double* eig, teo_schur_info* info);

/* ---- C5 (generalized pair) input T, the library generator restated ----- */
void teo_pair_t(size_t n, uint64_t seed, double* t, size_t ld);

/* ---- verification (verify.cpp) ----------------------------------------- */
double teo_similarity_residual(size_t n, const double* a, size_t lda, const double* q,
                               size_t ldq, const double* s, size_t lds);
double teo_orthogonality_defect(size_t n, const double* q, size_t ldq);
int teo_is_standardized(size_t n, const double* s, size_t ld);
/* read_eigenvalues (verify.cpp:104-130) */
void teo_read_eigenvalues(size_t n, const double* s, size_t ld, double* re, double* im);

#ifdef __cplusplus
}
#endif
#endif
