// plan.h -- host-side window planner and wavefront scheduler for the
// GPU reordering pass.
#pragma once
#include <cstddef>
#include <cstdint>
#include <algorithm>
#include <vector>

namespace teig {

// Bookkeeping of one diagonal block (reference reorder.cpp:200-204).
struct BlockState {
    uint8_t size;      // 1 or 2
    uint8_t selected;  // still to be moved to the leading part
    uint32_t orig;     // index in the caller's Selection
};

// One planned window (reference reorder.cpp:271-276).
struct PlannedWindow {
    int64_t wtop, wbot;          // rows [wtop, wbot)
    int64_t first_block, count;  // block slots [first_block, first_block + count)
    int64_t group;               // chain (group) index within the plan
    int64_t blk_off;             // offset into ReorderPlan::sizes / sel
    int32_t level;               // wavefront assigned by schedule_levels()
};

struct ReorderPlan {
    std::vector<PlannedWindow> windows;  // in reference (plan) order
    std::vector<uint8_t> sizes, sel;     // per window: `count` entries
    int64_t n_groups = 0;
    int32_t n_levels = 0;
};

// Plans every group's window chain assuming all swaps succeed -- the
// reference's per-group chain simulation (reorder.cpp:241-324) iterated over
// all groups.  `blocks` is not modified.  O(sum of window sizes).
ReorderPlan plan_reorder(const std::vector<BlockState>& blocks, int64_t ws);

// Greedy wavefront levels: a window's level is one more than the deepest
// earlier window whose diagonal range intersects it.  Windows of one level
// are pairwise disjoint; disjoint windows commute exactly (their similarity
// transformations act on disjoint index sets), so level order preserves the
// reference's per-element update order for every overlapping pair.
void schedule_levels(ReorderPlan& plan, int64_t n);

// Row support of an orthogonal factor's columns, tracked through the window
// updates so the factor updates skip rows that are exactly zero.  A window
// [a, b) replaces the columns a..b-1 by combinations of themselves
// (Q[:, a:b] <- Q[:, a:b] Q_w): a row that is zero in all of them stays zero,
// so the columns' supports become the hull of their supports and only those
// rows need the update.  For Q_in = I (the reorder workload) about half of all
// factor-update flops are products of exact zeros (n=40000: 3.1e13 of
// 6.4e13).  Zeros are tested bitwise (+0.0 only), so the skipped rows keep
// exactly the bits a full update would produce (DMMA sums start at +0).
// Intervals are [lo, hi] (lo > hi: an all-zero column).
struct FactorSupport {
    std::vector<int32_t> lo, hi;
    bool on = false;
    void full(int64_t n, int64_t r0, int64_t r1) {  // every row of [r0, r1) may be nonzero
        lo.assign(n, (int32_t)r0);
        hi.assign(n, (int32_t)(r1 - 1));
        on = true;
    }
    // rows [r0, r1) the update of window [a, b) must cover; merges the columns' supports
    void window(int64_t a, int64_t b, int64_t* r0, int64_t* r1) {
        int32_t l = lo[a], h = hi[a];
        for (int64_t c = a + 1; c < b; ++c) {
            if (lo[c] > hi[c]) continue;
            if (l > h) {
                l = lo[c];
                h = hi[c];
            } else {
                l = std::min(l, lo[c]);
                h = std::max(h, hi[c]);
            }
        }
        for (int64_t c = a; c < b; ++c) {
            lo[c] = l;
            hi[c] = h;
        }
        *r0 = l;
        *r1 = l > h ? l : (int64_t)h + 1;
    }
};

// Update flops of a plan: sum 2d^2 (n-b) + 2d^2 a (+ 2d^2 n with Q)
// (SURVEY.md 8d).
double plan_update_flops(const ReorderPlan& plan, int64_t n, bool with_q);
// Algorithmic HBM bytes of the updates: each panel read and written once.
double plan_update_bytes(const ReorderPlan& plan, int64_t n, bool with_q);

// Folds one executed pass's window outcomes into `blocks` in plan order
// (reference reorder.cpp:366-397); returns true when a replan is needed.
bool fold_outcomes(const ReorderPlan& plan, std::vector<BlockState>& blocks, const std::vector<int32_t>& st_by_plan,
                   const std::vector<uint8_t>& order, const std::vector<uint8_t>& stuck,
                   std::vector<int64_t>& rejected, std::vector<int64_t>& plan_log, bool strict);

}  // namespace teig
