// device_types.h -- descriptors shared by the host scheduler and the sm_100a
// kernels of the window pipeline.
#pragma once
#include <cstdint>

namespace teig {

// One planned diagonal window of a reordering (or Schur) pass.  Windows are
// stored sorted by level (wavefront); windows of one level are pairwise
// disjoint along the diagonal, so their window kernels, their left (row
// panel) updates and their right (column panel / factor) updates can each
// run concurrently.
struct WinDesc {
    int32_t a;         // first row/column of the window
    int32_t d;         // window order (b = a + d)
    int32_t nb;        // number of diagonal blocks inside the window
    int32_t level;     // wavefront level (deviation flag of the window kernels)
    int64_t qw_off;    // offset (doubles) of this window's Q_w (d x d, ld d)
    int64_t blk_off;   // offset into the per-block pools (sizes/sel/order/stuck)
    int32_t tl_pref;   // exclusive prefix of left-update tiles within the level
    int32_t tr_pref;   // exclusive prefix of right-update tiles (S) within the level
    int32_t tq_pref;   // exclusive prefix of factor-update tiles (Q) within the level
    int32_t pad;
    // index ranges the update kernels cover (absolute matrix coordinates; the
    // matrix pointers passed to the kernels are bases such that absolute
    // (i, j) lives at base[i + j*ld] -- for a column slab / row slab of a
    // distributed matrix the base is offset accordingly):
    int32_t lc0, lc1;  // left update:   S[a:b, lc0:lc1]   (single GPU: b, n)
    int32_t rr0, rr1;  // right update:  S[rr0:rr1, a:b]   (single GPU: 0, a)
    int32_t qr0, qr1;  // factor update: Q[qr0:qr1, a:b]   (single GPU: 0, n)
};

// Per-window outcome flags written by the window kernel.
enum : int32_t {
    kWinExecuted = 1,     // layout matched and the bubble ran
    kWinStuck = 2,        // at least one swap was rejected
    kWinSkipped = 4,      // not run: an earlier level deviated (the plan is stale)
};

// ---- Schur reduction (schur_window.cu) --------------------------------------

// SchurOptions (reference schur.hpp:20-29) as seen by the window kernels
struct SchurDevOpts {
    int32_t deflation;        // 0 classic, 1 norm-stable
    int32_t shift_count;      // 0: default_shift_count
    int32_t aed_window;       // 0: 3m/2
    int32_t small_threshold;  // direct small_schur below this active size
    int32_t flags;            // kSchurFlag* (diagnostics: disable a kernel-internal path)
};

enum { kSchurFlagNoWave = 1, kSchurFlagNoLocal = 2 };

// outcome of one AED / small-solve window (AedResult, schur.hpp:32-39)
struct AedDevOut {
    int32_t deflated;
    int32_t converged;
    int32_t swap_rejected;
    int32_t spike_eliminated;
    int32_t nshifts;
    int32_t pad;
    double newbeta;
};

enum : int32_t { kSchurModeAed = 0, kSchurModeSmall = 1, kSchurModeStd2 = 2 };
enum : int32_t { kChaseHop = 0, kChaseFinal = 1, kChaseIntro = 2 };

// one window of a bulge chain (intro window or a chase window of plan_chase,
// reference schur.cpp:484-505); bulge k (k = 0 bottom-most) enters at row
// p_bot - 3k (bulges stay exactly 3 rows apart)
struct ChaseWin {
    int32_t a, d;        // window rows/cols [a, a+d)
    int32_t ihi;         // end of the active range
    int32_t mode;        // kChaseHop / kChaseFinal / kChaseIntro
    int32_t nb;          // bulges in the window
    int32_t hop;         // steps per bulge (kChaseHop)
    int32_t p_bot;       // entering position of the bottom-most bulge
    int32_t shift_off;   // intro: offset of the (re, im) x 2 shift pairs
    int64_t qw_off;      // offset (doubles) of the window's Q_w
    int32_t packed_len;  // doubles of the packed window band
    int32_t pad;
};

}  // namespace teig
