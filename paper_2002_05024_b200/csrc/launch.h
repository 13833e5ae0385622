// launch.h -- host-side launchers of the sm_100a kernels (internal).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "device_types.h"

namespace teig {

// devctx.cpp: per-device (thread-safe) kernel attribute cache and SM count
cudaError_t ensure_dyn_smem(const void* func, size_t bytes);
int device_sm_count();
// private per-device stream-ordered pool of the library (devctx.cpp) and its
// retention policy (teig_set_memory_retention)
cudaError_t lib_malloc_async(void** p, size_t bytes, cudaStream_t s);
bool memory_retention();
void set_memory_retention(bool on);
void trim_memory_pools();
struct DeviceGuard {  // current device := the device owning p (restored on exit)
    explicit DeviceGuard(const void* p);
    ~DeviceGuard();
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
    int prev_ = 0;
    bool switched_ = false;
};

size_t window_reorder_smem_bytes(int dmax);

// dev_level (nullable): the pass's deviation level.  A window of level L
// (WinDesc::level) is skipped (status kWinSkipped, Q_w = I) when an earlier
// level deviated (*dev_level < L); a window that deviates (a rejected swap or
// a layout mismatch) lowers *dev_level to its level.  Initialise to INT_MAX.
cudaError_t launch_window_reorder(const WinDesc* wins, int nwin, int dmax, double* S, long long lds,
                                  double* qw_pool, const uint8_t* sizes_pool, const uint8_t* sel_pool,
                                  uint8_t* order_pool, uint8_t* stuck_pool, int32_t* status,
                                  cudaStream_t stream, unsigned long long* prof = nullptr,
                                  int32_t* dev_level = nullptr);
constexpr int kWindowThreads = 256;  // threads of the window kernel (8 warps)

// rows/cols: the extent of the matrix `S`/`M` points at (absolute indices
// [0, rows) x [0, cols)); when given, windows of order 65..128 take the TMA
// kernels of update_tma.cu, otherwise (or for slab bases) the cp.async ones.
// max_ctas > 0 caps the persistent grid of the bulk kernels (the caller keeps
// SMs free for window kernels running beside the launch); max_ctas < 0: as
// many CTAs as tiles (up to the SM count) -- latency-critical launches
cudaError_t launch_update_left(const WinDesc* wins, int nwin, int ntiles, int dmax, const double* qw_pool,
                               double* S, long long lds, int n, cudaStream_t stream, long long rows = -1,
                               long long cols = -1, int max_ctas = 0);

// short_ctas: launch the bulk factor kernel as short CTAs (short_tiles tiles each)
// instead of a persistent grid -- for a caller that runs the factor updates on
// a LOW-priority stream beside a critical path, so critical-path CTAs take SMs
// as they free up.
cudaError_t launch_update_right(const WinDesc* wins, int nwin, int ntiles, int dmax, const double* qw_pool,
                                double* M, long long ldm, int nrows_total, bool factor, cudaStream_t stream,
                                long long rows = -1, long long cols = -1, bool short_ctas = false, int max_ctas = 0,
                                int short_tiles = 8);

// devctx.cpp: a non-blocking stream cached per host thread, device and slot
// (slots: 0 host-path Q upload, 1 host-path drain, 2 generalized reorder's
// factor stream, 3 Schur reduction's side stream); nullptr on failure
cudaStream_t cached_stream(int slot);

// DMMA instructions the update kernels have issued on the current device so
// far (bulk-copy kernels: zero Q_w fragments skipped; cp.async kernels); x 512
// = executed flops.  Synchronous reads (profiling only).
unsigned long long dmma_count_bulk();
unsigned long long dmma_count_cp();

// update_tma.cu: false = not eligible (caller falls back), *err = launch status
bool launch_update_left_tma(const WinDesc* wins, int nwin, int ntiles, int dmax, const double* qw_pool, double* S,
                            long long lds, long long rows, long long cols, cudaStream_t stream, cudaError_t* err,
                            int max_ctas = 0);
bool launch_update_right_tma(const WinDesc* wins, int nwin, int ntiles, int dmax, const double* qw_pool, double* M,
                             long long ldm, long long rows, long long cols, bool factor, cudaStream_t stream,
                             cudaError_t* err, bool short_ctas = false, int max_ctas = 0, int short_tiles = 8);


// synthetic inputs (generate.cu)
cudaError_t launch_gen_schur_input(double* S, long long lds, long long n, uint64_t fill_seed,
                                   cudaStream_t stream);
cudaError_t launch_set_identity(double* Q, long long ldq, long long n, cudaStream_t stream);
// per column c < cols: lo[c] / hi[c] = first / last row < rows with a nonzero
// bit pattern (rows / -1 for a zero column)
cudaError_t launch_column_support(const double* Q, long long ldq, long long rows, long long cols, int32_t* lo,
                                  int32_t* hi, cudaStream_t stream);
cudaError_t launch_gen_hessenberg(double* H, long long ldh, long long n, uint64_t seed, cudaStream_t stream);
cudaError_t launch_gen_pair_t(double* T, long long ldt, long long n, uint64_t seed, cudaStream_t stream);
// generalized (S, T) window kernel (gwindow_reorder.cu), d <= 64
size_t gwindow_smem_bytes(int d);
cudaError_t launch_gwindow_reorder(const WinDesc* wins, int nwin, int dmax, double* S, long long lds, double* T,
                                   long long ldt, double* qw_pool, const uint8_t* sizes_pool,
                                   const uint8_t* sel_pool, uint8_t* order_pool, uint8_t* stuck_pool,
                                   int32_t* status, cudaStream_t stream, int32_t* dev_level = nullptr);
cudaError_t launch_gen_schur_cols(double* S, long long lds, long long n, uint64_t fill_seed, long long c0,
                                  long long c1, cudaStream_t stream);
cudaError_t launch_identity_rows(double* Q, long long ldq, long long n, long long r0, long long r1,
                                 cudaStream_t stream);

// Schur reduction window kernels (schur_window.cu)
#ifndef TEIG_AED_THREADS
#define TEIG_AED_THREADS 256
#endif
constexpr int kAedThreads = TEIG_AED_THREADS;
constexpr int kChaseThreads = 512;
constexpr int kAedMaxWindow = 104;   // AED / small-solve window order limit (shared memory)
constexpr int kChaseMaxWindow = 128; // chase window order limit
size_t aed_window_smem_bytes(int w);
size_t chase_window_smem_bytes(int d);
int chase_window_packed_len(int d);
cudaError_t launch_aed_window(double* H, long long ldh, int mode, int l, int e, int w, const SchurDevOpts& o,
                              double* qw_out, AedDevOut* out, double* shifts_out, cudaStream_t stream,
                              unsigned long long* prof = nullptr, double* snap = nullptr);
cudaError_t launch_chase_window(double* H, long long ldh, const ChaseWin* wins_dev, int idx, int d,
                                const double* shift_pairs, double* qw_pool, cudaStream_t stream);
cudaError_t launch_hess_norm(const double* H, long long ldh, int n, unsigned long long* out, cudaStream_t stream);
cudaError_t launch_scan_active(double* H, long long ldh, int n, int ihi, double hnorm, int* out,
                               cudaStream_t stream);

// backtransform.cu: C = beta C + alpha op(A) op(B) (DMMA, dgemm.cuh) and the reference's
// eigenvector column renormalisation (kind: 0 real, 1 pair start, 2 pair
// second half, other / NULL: finiteness check only; *nonfinite |= 1 on
// Inf / NaN)
// work (optional, work_doubles long): split-K partials for products with few
// output tiles and a long K (reduced in a fixed order: deterministic)
cudaError_t launch_dgemm(bool ta, bool tb, int m, int n, int kdim, double alpha, const double* A, long long lda,
                         const double* B, long long ldb, double beta, double* C, long long ldc, cudaStream_t s,
                         double* work = nullptr, size_t work_doubles = 0);
cudaError_t launch_renorm_columns(int n, double* X, long long ldx, const int8_t* kind_dev, int k, int* nonfinite,
                                  cudaStream_t s);
// distributed deviation flag: mode 0 publish this rank's flag into base[slots[0]],
// mode 1 absorb from the nslots flag slots base[slots[i]]
cudaError_t launch_dist_flag(int32_t* dev_level, double* base, const int64_t* slots, int nslots, int level, int mode,
                             cudaStream_t s);
// element-wise sum of nbuf device buffers into all of them (loopback all-reduce)
cudaError_t launch_sum_buffers(void* const* bufs, int nbuf, size_t count, int elem_bytes, cudaStream_t s);

#ifndef TEIG_UPD_BN
#define TEIG_UPD_BN 64
#endif
#ifndef TEIG_UPD_BM
#define TEIG_UPD_BM 64
#endif
constexpr int kLeftBN = TEIG_UPD_BN;   // columns per left-update tile
constexpr int kRightBM = TEIG_UPD_BM;  // rows per right/factor-update tile

}  // namespace teig
