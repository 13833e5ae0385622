// plan.cpp -- window planner + wavefront scheduler (host).
#include "plan.h"

#include <algorithm>

namespace teig {

namespace {

// Chains one group upward from its current slots to `target`
// (reference reorder.cpp:277-324): each window spans at most `ws` rows ending
// at the group's bottom, is snapped up to a block boundary, and packs the
// selected blocks inside it to its top.
void chain_group(std::vector<BlockState>& bl, std::vector<int64_t>& start, int64_t target,
                 int64_t gfirst, int64_t glast, int64_t gcount, int64_t ws, int64_t gid,
                 ReorderPlan& plan, std::vector<BlockState>& scratch) {
    for (;;) {
        if (gfirst == target) return;
        const int64_t gbot = start[glast + 1];
        int64_t wtop = std::max<int64_t>(start[target], gbot > ws ? gbot - ws : 0);
        int64_t bfirst = gfirst;
        while (bfirst > target && start[bfirst - 1] >= wtop) --bfirst;
        wtop = start[bfirst];
        const int64_t count = glast - bfirst + 1;
        PlannedWindow w{wtop, gbot, bfirst, count, gid, (int64_t)plan.sizes.size(), 0};
        for (int64_t i = bfirst; i <= glast; ++i) {
            plan.sizes.push_back(bl[i].size);
            plan.sel.push_back(bl[i].selected);
        }
        plan.windows.push_back(w);
        scratch.clear();
        for (int64_t i = bfirst; i <= glast; ++i)
            if (bl[i].selected) scratch.push_back(bl[i]);
        for (int64_t i = bfirst; i <= glast; ++i)
            if (!bl[i].selected) scratch.push_back(bl[i]);
        for (int64_t i = 0; i < count; ++i) {
            bl[bfirst + i] = scratch[i];
            start[bfirst + i + 1] = start[bfirst + i] + scratch[i].size;
        }
        gfirst = bfirst;
        glast = bfirst + gcount - 1;
        if (wtop == start[target]) return;
    }
}

}  // namespace

ReorderPlan plan_reorder(const std::vector<BlockState>& blocks_in, int64_t ws) {
    ReorderPlan plan;
    std::vector<BlockState> bl = blocks_in;
    const int64_t nb = (int64_t)bl.size();
    std::vector<int64_t> start(nb + 1, 0);
    for (int64_t i = 0; i < nb; ++i) start[i + 1] = start[i] + bl[i].size;
    std::vector<BlockState> scratch;
    int64_t target = 0, gid = 0;
    for (;;) {
        while (target < nb && bl[target].selected) ++target;
        int64_t fs = target;
        while (fs < nb && !bl[fs].selected) ++fs;
        if (fs == nb) break;
        // group: selected blocks from fs fitting half a window and spanning
        // at most one window (reorder.cpp:259-267)
        int64_t grows = bl[fs].size, gcount = 1, glast = fs;
        for (int64_t g = fs + 1; g < nb; ++g) {
            if (!bl[g].selected) continue;
            const int64_t span = start[g + 1] - start[fs];
            if (grows + bl[g].size > ws / 2 || span > ws) break;
            grows += bl[g].size;
            ++gcount;
            glast = g;
        }
        chain_group(bl, start, target, fs, glast, gcount, ws, gid, plan, scratch);
        ++gid;
    }
    plan.n_groups = gid;
    return plan;
}

void schedule_levels(ReorderPlan& plan, int64_t n) {
    std::vector<int32_t> row_level(n, -1);
    int32_t maxl = -1;
    for (auto& w : plan.windows) {
        int32_t l = -1;
        for (int64_t r = w.wtop; r < w.wbot; ++r) l = std::max(l, row_level[r]);
        w.level = l + 1;
        for (int64_t r = w.wtop; r < w.wbot; ++r) row_level[r] = w.level;
        maxl = std::max(maxl, w.level);
    }
    plan.n_levels = maxl + 1;
}

double plan_update_flops(const ReorderPlan& plan, int64_t n, bool with_q) {
    double f = 0.0;
    for (const auto& w : plan.windows) {
        const double d = double(w.wbot - w.wtop);
        f += 2.0 * d * d * double(n - w.wbot) + 2.0 * d * d * double(w.wtop);
        if (with_q) f += 2.0 * d * d * double(n);
    }
    return f;
}

double plan_update_bytes(const ReorderPlan& plan, int64_t n, bool with_q) {
    double b = 0.0;
    for (const auto& w : plan.windows) {
        const double d = double(w.wbot - w.wtop);
        b += 16.0 * d * (double(n - w.wbot) + double(w.wtop) + (with_q ? double(n) : 0.0));
    }
    return b;
}

}  // namespace teig
