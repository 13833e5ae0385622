/*
 * taskeig_b200.h -- C ABI of the B200-native (sm_100a) window-based
 * off-diagonal update path of StarNEig / taskeig.
 *
 * This is the thin, stream-ordered CUDA layer underneath the C++ drop-in
 * (include/taskeig/ headers, namespace taskeig).  It takes plain pointers and
 * sizes -- no C++ or torch types -- so any FFI (ctypes, cgo, JNI) can bind it.
 *
 * Conventions:
 *   * matrices are COLUMN-MAJOR fp64 with an explicit leading dimension
 *     (element (i,j) at p[i + j*ld]), the orientation of the reference's tiles
 *     and DenseMatrix (tiled_matrix.hpp:27-35, dense.hpp:33-36), so a
 *     TiledMatrix <-> device conversion is a tile-wise copy, no transpose;
 *   * `*_device` entry points take DEVICE pointers and a cudaStream_t (passed
 *     as void*, NULL = legacy default stream) and are ordered on that stream;
 *     they return after their host-side bookkeeping completed (the reorder
 *     driver synchronizes once per planning pass to fold window outcomes);
 *   * `*_host` entry points take HOST pointers and include the host<->device
 *     copies;
 *   * return value: 0 ok; < 0 invalid argument -i (LAPACK `info` style) or an
 *     internal error (TEIG_ERR_*); > 0 a count of rejected swaps /
 *     non-converged windows where documented.  teig_last_error() describes
 *     the last failure of the calling thread.
 *
 * Every entry point cites the reference interface it replaces.
 */
#ifndef TASKEIG_B200_H
#define TASKEIG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TEIG_OK 0
#define TEIG_ERR_CUDA (-1000)
#define TEIG_ERR_UNSUPPORTED (-1001)
#define TEIG_ERR_STRICT (-1002)    /* rejected swap in strict mode (reorder.cpp:383-385) */
#define TEIG_ERR_INTERNAL (-1003)
#define TEIG_ERR_NONFINITE (-1004)  /* a non-finite result (the reference's assert_finite) */
#define TEIG_ERR_IO (-1005)         /* file IO / format error (the reference's std::runtime_error) */

const char* teig_last_error(void);
int teig_version(void);

/* ------------------------------------------------------------------------ */
/* Reordering (replaces taskeig::reorder_schur, reorder.hpp:88-89 /           */
/* reorder.cpp:215-404).                                                     */

typedef struct teig_reorder_opts {
    int64_t window_size; /* 0: default_tile_size(n) (reorder.cpp:221-222); values above 128
                            (one CTA's shared memory) run at 128: same result, other plan */
    int32_t strict;      /* !=0: fail with TEIG_ERR_STRICT on a rejected swap */
    int32_t overlap_factor; /* !=0 (default 1 via teig_reorder_opts_default): run the
                               Q-factor updates on a second stream, overlapped */
    int32_t profile;     /* !=0: bracket every launch with CUDA events and report
                            per-kernel-class device time in teig_reorder_info */
    int32_t full_factor; /* !=0: update the factor(s) over all rows (no skipping of the
                            exactly-zero rows; same bits, the reference's flop count) */
} teig_reorder_opts;

typedef struct teig_reorder_info {
    int64_t n_windows;     /* windows that ran or deviated = entries of `plan` (all passes;
                              windows skipped after a deviation are replanned, not counted) */
    int64_t n_levels;      /* wavefronts (all passes) */
    int64_t n_passes;      /* planning passes (1 for a clean run) */
    int64_t n_groups;      /* chains planned in the first pass */
    int64_t n_rejected;    /* blocks whose swap was rejected */
    int32_t clean;         /* no rejection, selection fully leading (reorder.hpp:80) */
    int32_t pad;
    double update_flops;   /* sum over executed windows of 2d^2(n-b) + 2d^2 a (+ 2d^2 n) */
    double update_bytes;   /* algorithmic panel bytes: 16 d ((n-b) + a (+ n)) per window */
    double plan_ms;        /* host planning + scheduling time */
    int64_t n_launches;    /* kernels launched by the call */
    double ms_window;      /* profile only: summed device time of the window kernels */
    double ms_left;        /*   ... of the left (row-panel) update kernels */
    double ms_right;       /*   ... of the right (column-panel) update kernels */
    double ms_factor;      /*   ... of the Q-factor update kernels */
    double flops_left, flops_right, flops_factor; /* update flops per kernel class (the
                                     reference's count: factor updates over all n rows) */
    double flops_factor_exec;  /* factor-update flops actually executed: rows outside the
                                  tracked support of Q's columns are exact zeros and skipped
                                  (Q_in = I: about half; TEIG_NO_Q_SUPPORT=1 disables) */
    double flops_dmma;         /* profile only: flops of the DMMA instructions the update
                                  kernels issued (512 per m8n8k4; Q_w's all-zero fragments are
                                  skipped by the bulk kernels), from device counters */
} teig_reorder_info;

void teig_reorder_opts_default(teig_reorder_opts* o);

/* dS: n x n standardized quasi-triangular Schur form (device, ld lds), updated
 * in place to the reordered form.  dQ: n x n (device, ld ldq) or NULL; updated
 * to Q * Q3.  sizes/flags: host arrays of nb diagonal-block sizes (1/2) and
 * selection flags (a Selection: reorder.hpp:22-32).  perm (host, nb): original
 * block -> final slot; rejected (host, nb): original indices of rejected
 * blocks, count in info->n_rejected.  plan (host, 3*plan_cap or NULL):
 * (position, extent, moved_blocks) per executed window, like
 * ReorderResult::plan.  Returns 0, or < 0 on error. */
int teig_reorder_schur_device(int64_t n, double* dS, int64_t lds, double* dQ, int64_t ldq,
                              int64_t nb, const uint8_t* sizes, const uint8_t* flags,
                              const teig_reorder_opts* opts, int64_t* perm, int64_t* rejected,
                              int64_t* plan, int64_t plan_cap, teig_reorder_info* info,
                              void* stream);

/* Same on HOST buffers (column-major, ld); includes H2D/D2H. */
int teig_reorder_schur_host(int64_t n, double* S, int64_t lds, double* Q, int64_t ldq, int64_t nb,
                            const uint8_t* sizes, const uint8_t* flags,
                            const teig_reorder_opts* opts, int64_t* perm, int64_t* rejected,
                            int64_t* plan, int64_t plan_cap, teig_reorder_info* info,
                            void* stream);

/* Execution trace (the reference's ExecutionReport, runtime.hpp:50-60, and
 * SchurOptions::keep_reports): with tracing on, every reorder / Schur call
 * made on this thread records one task per kernel launch -- {"label":
 * "reorder:<W|L|R|Q>:p<pass>:l<level>" or "schur:<A|C|L|R|Q>:r<round>",
 * "worker": stream (0 critical path, 1 second stream), "start_ns",
 * "end_ns"} from CUDA events relative to the call's start -- and, for
 * reorder, one record per planned window {"pass", "level", "position",
 * "extent", "blocks", "group", "status"}.  teig_trace_json writes the last
 * call's trace as JSON into buf when cap exceeds its length and returns the
 * length; teig_trace_task reads task i.  Tracing brackets every launch with
 * events. */
void teig_trace_enable(int32_t on);
int64_t teig_trace_json(char* buf, int64_t cap);
int64_t teig_trace_task_count(void);
int teig_trace_task(int64_t i, char* label, int64_t cap, int32_t* worker, int64_t* start_ns, int64_t* end_ns);

/* Device memory policy (not part of the reference interface: the reference
 * has no device memory).  Every per-call device buffer comes from a private
 * stream-ordered pool per device.  Retention off (the default; TEIG_RETAIN=1
 * in the environment turns it on at load): the pool returns its memory at
 * every synchronisation and the host entry points allocate their device
 * staging (2 n^2 doubles) per call.  On: both are kept between calls, so a
 * process that calls repeatedly does not remap gigabytes every time.
 * teig_release_memory() returns all of it (staging + pools, every device);
 * teig_release_host_staging() only the staging. */
void teig_set_memory_retention(int32_t on);
int32_t teig_memory_retention(void);
void teig_release_memory(void);
void teig_release_host_staging(void);

/* Bytes the calling thread's last teig_reorder_schur_host call moved host ->
 * device and device -> host (S's upper Hessenberg part, Q's row hulls, the
 * drained and final copies).  Both 0 before any such call. */
void teig_host_transfer_bytes(int64_t* h2d, int64_t* d2h);

/* Diagonal-block scan by exact-zero subdiagonal (reorder.cpp:21-43) on a
 * device matrix.  sizes: host array of capacity n.  Returns nb (>= 0). */
int64_t teig_scan_blocks_device(int64_t n, const double* dS, int64_t lds, uint8_t* sizes,
                                void* stream);

/* select_fraction (reorder.cpp:80-97): exactly floor(fraction*nb) blocks by a
 * Philox(seed ^ 0x5e1ec7) Fisher-Yates shuffle.  flags: host, nb. */
int teig_select_fraction(int64_t nb, double fraction, uint64_t seed, uint8_t* flags);

/* Planner only (host, no device work): the windows reorder_schur would run
 * on a clean pass -- the reference's per-group chains (reorder.cpp:241-324)
 * -- with their wavefront levels.  win (host, 5*cap int64 or NULL):
 * (wtop, wbot, count, group, level) per window.  Returns the window count;
 * *n_levels, *n_groups, *flops (update flops with Q) when non-NULL. */
int64_t teig_plan_reorder(int64_t n, int64_t nb, const uint8_t* sizes, const uint8_t* flags,
                          int64_t window_size, int64_t* win, int64_t cap, int64_t* n_levels,
                          int64_t* n_groups, double* flops);

/* ------------------------------------------------------------------------ */
/* Window-level kernels (device buffers; synchronous on `stream`).           */

/* window_reorder (reorder.hpp:62-65 / reorder.cpp:124-194) on a d x d window
 * (d <= 128) at dW (ld ldw, updated in place); dAcc (d x d, ld d) receives the
 * accumulated orthogonal factor (identity on a layout mismatch).  order /
 * stuck: host, nb.  *executed = 0 on a layout mismatch. */
int teig_window_reorder_device(int64_t d, double* dW, int64_t ldw, int64_t nb,
                               const uint8_t* sizes, const uint8_t* sel, double* dAcc,
                               uint32_t* order, uint8_t* stuck, int32_t* executed, void* stream);

/* apply_window_updates (window_tasks.hpp:36-38 / window_tasks.cpp:89-102):
 * S[a:b, b:n] <- Qw^T S[a:b, b:n];  S[0:a, a:b] <- S[0:a, a:b] Qw;
 * Q[0:n, a:b] <- Q[0:n, a:b] Qw (dQ may be NULL).  dQw: d x d, ld d. */
int teig_apply_window_updates_device(int64_t n, double* dS, int64_t lds, double* dQ, int64_t ldq,
                                     int64_t a, int64_t d, const double* dQw, void* stream);

/* One panel of apply_window_updates on an explicit index range (the unit the
 * distributed driver runs on a slab; window_tasks.cpp:40-86 per tile):
 *   side 0 (L):  M[a:a+d, i0:i1] <- Qw^T M[a:a+d, i0:i1]
 *   side 1 (R):  M[i0:i1, a:a+d] <- M[i0:i1, a:a+d] Qw
 *   side 2 (Q):  as side 1, the factor-update kernel variant.
 * dM is a base such that absolute (i, j) lives at dM[i + j*ldm] for
 * i < rows, j < cols (a slab's base may point before its allocation).
 * Synchronous on `stream`. */
int teig_update_panel_device(int32_t side, int64_t d, const double* dQw, int64_t a, double* dM,
                             int64_t ldm, int64_t rows, int64_t cols, int64_t i0, int64_t i1,
                             void* stream);

/* ------------------------------------------------------------------------ */
/* Schur reduction: multishift QR with aggressive early deflation           */
/* (replaces taskeig::schur_reduce, schur.hpp:94-95 / schur.cpp:671-906,     */
/* and the per-step ops aed_step, introduce_bulges, chase_bulges,            */
/* deflation_check, kernels::small_schur: schur.hpp:63-89, kernels.hpp:93).  */

typedef struct teig_schur_opts {  /* SchurOptions, schur.hpp:20-29 */
    int32_t deflation;        /* 0 classic, 1 norm-stable (default) */
    int32_t shift_count;      /* 0: max(4, round-to-even(active/16)), cap 64; explicit values above 64 run at 64 */
    int32_t aed_window;       /* 0: 3m/2; above 104 (one CTA's shared memory) runs at 104 */
    int32_t small_threshold;  /* direct small_schur at or below (default 64; above 104 runs at 104) */
    int64_t iteration_limit;  /* 0: 30 n sweeps */
    int64_t tile_size;        /* chase window: 0 = default_tile_size(n) (128 for n >= 1000); above 128 runs at 128 */
    int32_t profile;          /* !=0: CUDA-event time per kernel class in teig_schur_info */
    int32_t pad;
} teig_schur_opts;

typedef struct teig_schur_info {  /* SchurDecomposition's scalars, schur.hpp:50-58 */
    int64_t sweeps;
    int64_t rounds;             /* executed rounds (one readback each) */
    int64_t aed_windows;
    int64_t chase_windows;      /* intro + chase windows */
    int64_t converged_trailing; /* meaningful when !converged */
    int64_t n_launches;
    int32_t converged;
    int32_t pad;
    double update_flops;        /* sum over windows of 2d^2(n-b) + 2d^2 a (+ 2d^2 n) */
    double ms_window;           /* profile only: device time of window kernels */
    double ms_update;           /* profile only: device time of update kernels (both streams) */
    double ms_total_host;       /* host wall time of the call */
} teig_schur_info;

typedef struct teig_aed_result {  /* AedResult, schur.hpp:32-39 */
    int64_t window, deflated, nshifts;
    int32_t spike_eliminated, converged, swap_rejected, pad;
} teig_aed_result;

void teig_schur_opts_default(teig_schur_opts* o);

/* schur_reduce: dH (n x n upper Hessenberg, device, ld ldh) -> standardized
 * real Schur form in place; dQ (device, ld ldq) or NULL: Q <- Q * Z.
 * eig_re/eig_im (host, n, or NULL): eigenvalues read off the diagonal as the
 * reference does (schur.cpp:888-904).  Returns 0 (check info->converged), < 0
 * on bad arguments, TEIG_ERR_* otherwise. */
int teig_schur_reduce_device(int64_t n, double* dH, int64_t ldh, double* dQ, int64_t ldq,
                             const teig_schur_opts* opts, double* eig_re, double* eig_im,
                             teig_schur_info* info, void* stream);
/* Same on HOST buffers (column-major, ld); includes H2D/D2H. */
int teig_schur_reduce_host(int64_t n, double* H, int64_t ldh, double* Q, int64_t ldq,
                           const teig_schur_opts* opts, double* eig_re, double* eig_im,
                           teig_schur_info* info, void* stream);

/* aed_step (schur.hpp:68-69): one AED window of the active range [l, ihi)
 * with its off-window updates.  shifts (host, 2*window doubles): (re, im). */
int teig_aed_step_device(int64_t n, double* dH, int64_t ldh, double* dQ, int64_t ldq, int64_t l,
                         int64_t ihi, int64_t window, const teig_schur_opts* opts,
                         teig_aed_result* result, double* shifts, void* stream);

/* introduce_bulges (schur.hpp:73-75): shifts (host) as nshifts (re, im)
 * pairs; positions (host, nshifts/2) receives the bulge rows, bottom first. */
int teig_introduce_bulges_device(int64_t n, double* dH, int64_t ldh, double* dQ, int64_t ldq,
                                 int64_t l, int64_t ihi, int64_t nshifts, const double* shifts,
                                 int64_t* positions, void* stream);

/* chase_bulges (schur.hpp:87-89): chases the chain (positions bottom first,
 * as returned by teig_introduce_bulges_device) off the bottom of [., chain_end)
 * with windows of max(window_size, 3nb+6) rows. */
int teig_chase_bulges_device(int64_t n, double* dH, int64_t ldh, double* dQ, int64_t ldq,
                             int64_t chain_end, int64_t nb, const int64_t* positions,
                             int64_t window_size, int64_t* n_windows, void* stream);

/* plan_chase (schur.cpp:484-505), host only: the windows chase_bulges runs
 * for the chain (positions bottom first), as (a, d, mode) triples (mode 0 hop,
 * 1 final) in win (3*cap int64 or NULL).  Returns the window count or < 0. */
int64_t teig_plan_chase(int64_t nb, const int64_t* positions, int64_t chain_end, int64_t window_size,
                        int64_t* win, int64_t cap);

/* kernels::small_schur (kernels.hpp:93): dH k x k (ld ldh) in place, dQ
 * (k x k, ld k) receives the similarity.  k <= 104. */
int teig_small_schur_device(int64_t k, double* dH, int64_t ldh, double* dQ, int32_t* converged,
                            void* stream);

/* deflation_check (schur.hpp:63-64); host only. */
int teig_deflation_check(double spike, double diag_sum, int32_t deflation, double wnorm);

/* ------------------------------------------------------------------------ */
/* Hessenberg reduction (replaces taskeig::hessenberg_reduce,                 */
/* hessenberg.hpp / hessenberg.cpp:185-280): dA (n x n, column-major, device) */
/* is reduced in place to upper Hessenberg H = Q1^T A Q1 by the reference's   */
/* blocked compact-WY algorithm (panels of panel_width columns; 0: min(tile,  */
/* 64) as the reference, larger values run at 64); dQ (device, or NULL)       */
/* receives Q1.  Entries below the subdiagonal are exact zeros.  Synchronous. */
typedef struct teig_hessenberg_info {
    int64_t panels;
    int64_t launches;
    double flops;
    int64_t panel_width;
} teig_hessenberg_info;
int teig_hessenberg_reduce_device(int64_t n, double* dA, int64_t lda, double* dQ, int64_t ldq,
                                  int64_t panel_width, teig_hessenberg_info* info, void* stream);

/* ------------------------------------------------------------------------ */
/* Eigenvector back-transformation (replaces taskeig::backtransform,          */
/* eigvec.hpp:88-89 / eigvec.cpp:448-516): X = Q Y on the FP64 tensor pipe   */
/* with the device-resident Q of a reorder / Schur call, then every real      */
/* column and every complex pair renormalised to unit max-norm with a         */
/* positive lead entry.  dQ n x n, dY / dX n x k (column-major, device; X    */
/* must not alias Y).  col_kind (host, k; NULL: no renormalisation): 0 real,  */
/* 1 real part of a pair (next column = imaginary part), 2 imaginary part.    */
/* Returns 0, < 0 on bad arguments, TEIG_ERR_NONFINITE on Inf/NaN in X.       */
int teig_backtransform_device(int64_t n, int64_t k, const double* dQ, int64_t ldq, const double* dY,
                              int64_t ldy, double* dX, int64_t ldx, const int8_t* col_kind, void* stream);

/* ------------------------------------------------------------------------ */
/* Matrix files (replaces taskeig::write_matrix_file / read_matrix_file,      */
/* io.hpp / io.cpp:37-121), byte-compatible with the reference.  format:      */
/* "teig" (binary: "TEIG", uint32 1, uint64 rows, uint64 cols, row-major     */
/* float64) or "matrixmarket" ("array real general", column by column, 17    */
/* digits).  Buffers are ROW-major (the reference's DenseBuffer).  Read: pass */
/* a_rm = NULL to get the shape only; cap = capacity of a_rm in doubles.      */
int teig_write_matrix_file(const char* path, const char* format, int64_t rows, int64_t cols,
                           const double* a_rm);
int teig_read_matrix_file(const char* path, const char* format, int64_t* rows, int64_t* cols,
                          double* a_rm, int64_t cap);

/* ------------------------------------------------------------------------ */
/* Synthetic inputs directly in HBM (bit-identical to the      */
/* reference generators).                                                    */

/* default_spectrum + build_quasi_triangular (generate.cpp:68-91, 115-150)
 * with the strictly-upper fill drawn from Philox(fill_seed). */
int teig_gen_schur_input_device(int64_t n, double* dS, int64_t lds, uint64_t fill_seed, void* stream);
/* generate(hessenberg_random, n, seed) (generate.cpp:192-198) */
int teig_gen_hessenberg_device(int64_t n, double* dH, int64_t ldh, uint64_t seed, void* stream);
int teig_set_identity_device(int64_t n, double* dQ, int64_t ldq, void* stream);


/* ------------------------------------------------------------------------ */
/* Multi-GPU reordering: S in column slabs, Q in   */
/* row slabs, the owners' Q_w broadcast (NCCL) per wavefront, halo           */
/* transfers for windows straddling a slab boundary.  Same result, bit for   */
/* bit, as teig_reorder_schur_device (replaces the reference's distributed   */
/* execution of reorder_schur's window tasks, reorder.cpp:330-364 /          */
/* window_tasks.cpp:31-87, which StarNEig runs over MPI+StarPU).             */

/* Balanced slab boundaries (world+1 each): column slabs with equal left +
 * right update flops (from the planner), >= 256 columns each; equal Q row
 * slabs. */
int teig_dist_balance(int64_t n, int64_t nb, const uint8_t* sizes, const uint8_t* flags,
                      int64_t window_size, int32_t world, int64_t* col_bounds, int64_t* row_bounds);

/* Host-side communication schedule of the first pass (no device work): per
 * transfer 8 int64 (level, phase, src, dst, r0, r1, c0, c1); phase 0 window
 * halo in, 1 panel halo in, 2 halo back.  Returns the transfer count. */
int64_t teig_dist_schedule(int64_t n, int64_t nb, const uint8_t* sizes, const uint8_t* flags,
                           int64_t window_size, int32_t world, const int64_t* col_bounds, int64_t* out,
                           int64_t cap);

/* One rank of the distributed reorder.  nccl_comm: from teig_nccl_comm_init
 * (one process per GPU: dS_slabs/dQ_slabs hold THIS rank's slab), or NULL for
 * the loopback mode (all `world` ranks in this process on the current device:
 * dS_slabs/dQ_slabs hold every rank's slab, rank ignored).  S slab of rank r:
 * n x (C[r+1]-C[r]+128) column-major, ld lds (>= n), columns [C[r], C[r+1])
 * plus a 128-column halo; Q slab of rank r: (R[r+1]-R[r]) x n column-major,
 * ld R[r+1]-R[r], rows [R[r], R[r+1]) (dQ_slabs NULL: no Q).  Arguments as
 * teig_reorder_schur_device otherwise. */
int teig_dist_reorder_schur(int64_t n, int32_t world, int32_t rank, void* nccl_comm,
                            double* const* dS_slabs, int64_t lds, double* const* dQ_slabs,
                            const int64_t* col_bounds, const int64_t* row_bounds, int64_t nb,
                            const uint8_t* sizes, const uint8_t* flags, const teig_reorder_opts* opts,
                            int64_t* perm, int64_t* rejected, teig_reorder_info* info, void* stream);

/* Single-process multi-GPU: all `world` ranks in this process, rank r on
 * devices[r] (distinct GPUs), NCCL clique from ncclCommInitAll (created once
 * per device list, kept for the process).  dS_slabs[r] / dQ_slabs[r] are rank
 * r's slabs on devices[r] (layout as teig_dist_reorder_schur); plan as
 * teig_reorder_schur_device.  Synchronous; same result, bit for bit, as
 * teig_reorder_schur_device.  The C++ drop-in takes this path when the
 * TASKEIG_GPUS environment variable asks for GPUs (taskeig_adapter.cpp). */
int teig_dist_reorder_schur_multi(int64_t n, int32_t world, const int32_t* devices,
                                  double* const* dS_slabs, int64_t lds, double* const* dQ_slabs,
                                  const int64_t* col_bounds, const int64_t* row_bounds, int64_t nb,
                                  const uint8_t* sizes, const uint8_t* flags,
                                  const teig_reorder_opts* opts, int64_t* perm, int64_t* rejected,
                                  int64_t* plan, int64_t plan_cap, teig_reorder_info* info);

/* Generalized pencil (C5) across ranks: S and T in column slabs (same
 * layout as dS_slabs), Q and Z in row slabs; window_size <= 64.  Same result,
 * bit for bit, as teig_greorder_schur_device. */
int teig_dist_greorder_schur(int64_t n, int32_t world, int32_t rank, void* nccl_comm,
                             double* const* dS_slabs, double* const* dT_slabs, int64_t lds,
                             double* const* dQ_slabs, double* const* dZ_slabs, const int64_t* col_bounds,
                             const int64_t* row_bounds, int64_t nb, const uint8_t* sizes,
                             const uint8_t* flags, const teig_reorder_opts* opts, int64_t* perm,
                             int64_t* rejected, teig_reorder_info* info, void* stream);

/* NCCL plumbing (libnccl.so.2 resolved at run time). */
int teig_nccl_available(void);
int teig_nccl_unique_id(uint8_t* id128);
int teig_nccl_comm_init(int32_t world, int32_t rank, const uint8_t* id128, void** comm);
int teig_nccl_comm_destroy(void* comm);

/* Slab generators: columns [c0, c1) of the synthetic Schur form into dS
 * (ld lds, column c0 first); rows [r0, r1) of the identity into dQ (ld ldq). */
int teig_gen_schur_input_cols_device(int64_t n, double* dS, int64_t lds, int64_t c0, int64_t c1,
                                     uint64_t fill_seed, void* stream);
int teig_set_identity_rows_device(int64_t n, double* dQ, int64_t ldq, int64_t r0, int64_t r1,
                                  void* stream);


/* ------------------------------------------------------------------------ */
/* Generalized Schur-pair reordering (S, T) with Q and Z (SURVEY.md 8a a16,  */
/* config C5; no reference implementation: LAPACK DTGSEN/DTGEX2 semantics    */
/* over the reference's reorder planner, reorder.cpp:215-404).               */

/* dS upper quasi-triangular (block sizes = sizes, as from S's subdiagonal),
 * dT upper triangular (2x2 diagonal blocks of T upper triangular), both
 * n x n column-major on the device; dQ, dZ (or NULL) updated to Q*Qs, Z*Zs
 * with (S, T) <- Qs^T (S, T) Zs.  opts->window_size 0 means 64 (the limit:
 * the window kernel holds S, T, Q_w and Z_w in shared memory).  Outputs as
 * teig_reorder_schur_device. */
int teig_greorder_schur_device(int64_t n, double* dS, int64_t lds, double* dT, int64_t ldt, double* dQ,
                               int64_t ldq, double* dZ, int64_t ldz, int64_t nb, const uint8_t* sizes,
                               const uint8_t* flags, const teig_reorder_opts* opts, int64_t* perm,
                               int64_t* rejected, teig_reorder_info* info, void* stream);
/* Same on HOST buffers; includes H2D/D2H. */
int teig_greorder_schur_host(int64_t n, double* S, int64_t lds, double* T, int64_t ldt, double* Q,
                             int64_t ldq, double* Z, int64_t ldz, int64_t nb, const uint8_t* sizes,
                             const uint8_t* flags, const teig_reorder_opts* opts, int64_t* perm,
                             int64_t* rejected, teig_reorder_info* info, void* stream);
/* The C5 input T: upper triangular, diagonal 1 + U[0,1),
 * uniform [-1, 1] fill, on the synthetic S's block pattern. */
int teig_gen_pair_t_device(int64_t n, double* dT, int64_t ldt, uint64_t seed, void* stream);

#ifdef __cplusplus
}
#endif
#endif
