// launch.h -- host-side launchers of the sm_100a kernels (internal).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "device_types.h"

namespace teig {

size_t window_reorder_smem_bytes(int dmax);

cudaError_t launch_window_reorder(const WinDesc* wins, int nwin, int dmax, double* S, long long lds,
                                  double* qw_pool, const uint8_t* sizes_pool, const uint8_t* sel_pool,
                                  uint8_t* order_pool, uint8_t* stuck_pool, int32_t* status,
                                  cudaStream_t stream, unsigned long long* prof = nullptr);
constexpr int kWindowThreads = 256;  // threads of the window kernel (8 warps)

// rows/cols: the extent of the matrix `S`/`M` points at (absolute indices
// [0, rows) x [0, cols)); when given, windows of order 65..128 take the TMA
// kernels of update_tma.cu, otherwise (or for slab bases) the cp.async ones.
cudaError_t launch_update_left(const WinDesc* wins, int nwin, int ntiles, int dmax, const double* qw_pool,
                               double* S, long long lds, int n, cudaStream_t stream, long long rows = -1,
                               long long cols = -1);

cudaError_t launch_update_right(const WinDesc* wins, int nwin, int ntiles, int dmax, const double* qw_pool,
                                double* M, long long ldm, int nrows_total, bool factor, cudaStream_t stream,
                                long long rows = -1, long long cols = -1);

// update_tma.cu: false = not eligible (caller falls back), *err = launch status
bool launch_update_left_tma(const WinDesc* wins, int nwin, int ntiles, int dmax, const double* qw_pool, double* S,
                            long long lds, long long rows, long long cols, cudaStream_t stream, cudaError_t* err);
bool launch_update_right_tma(const WinDesc* wins, int nwin, int ntiles, int dmax, const double* qw_pool, double* M,
                             long long ldm, long long rows, long long cols, bool factor, cudaStream_t stream,
                             cudaError_t* err);

// keep the stream-ordered allocator's memory between calls (reorder_driver.cpp)
void keep_pool_memory();

// synthetic inputs (generate.cu)
cudaError_t launch_gen_schur_input(double* S, long long lds, long long n, uint64_t fill_seed,
                                   cudaStream_t stream);
cudaError_t launch_set_identity(double* Q, long long ldq, long long n, cudaStream_t stream);
cudaError_t launch_gen_hessenberg(double* H, long long ldh, long long n, uint64_t seed, cudaStream_t stream);
cudaError_t launch_gen_pair_t(double* T, long long ldt, long long n, uint64_t seed, cudaStream_t stream);
// generalized (S, T) window kernel (gwindow_reorder.cu), d <= 64
size_t gwindow_smem_bytes(int d);
cudaError_t launch_gwindow_reorder(const WinDesc* wins, int nwin, int dmax, double* S, long long lds, double* T,
                                   long long ldt, double* qw_pool, const uint8_t* sizes_pool,
                                   const uint8_t* sel_pool, uint8_t* order_pool, uint8_t* stuck_pool,
                                   int32_t* status, cudaStream_t stream);
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
