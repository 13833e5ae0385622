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
    int32_t flags;     // reserved
    int64_t qw_off;    // offset (doubles) of this window's Q_w (d x d, ld d)
    int64_t blk_off;   // offset into the per-block pools (sizes/sel/order/stuck)
    int32_t tl_pref;   // exclusive prefix of left-update tiles within the level
    int32_t tr_pref;   // exclusive prefix of right-update tiles (S) within the level
    int32_t tq_pref;   // exclusive prefix of factor-update tiles (Q) within the level
    int32_t pad;
};

// Per-window outcome flags written by the window kernel.
enum : int32_t {
    kWinExecuted = 1,     // layout matched and the bubble ran
    kWinStuck = 2,        // at least one swap was rejected
};

}  // namespace teig
