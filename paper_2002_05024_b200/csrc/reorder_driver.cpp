// reorder_driver.cpp -- the GPU window scheduler for Schur-form reordering
// (host C++ over the sm_100a kernels), exported through the C ABI in
// include/taskeig_b200.h.
//
// Replaces the reference's per-group TaskGraph execution
// (reorder.cpp:241-398, runtime.cpp:47-249):
//   1. plan every group's window chain up front (plan.cpp), exactly the
//      windows the reference would run when every swap succeeds;
//   2. assign wavefront levels -- chains pipeline behind each other instead of
//      running one group at a time;
//   3. per level, three stream-ordered launches: the batched window kernel
//      (one CTA per window), the batched left (row-panel) update, the batched
//      right (column-panel) update; the Q-factor updates of the level run on a
//      second stream, overlapped with the next levels' window work;
//   4. one D2H readback of the window outcomes per pass; fold them in plan
//      order (reorder.cpp:366-397); replan if anything deviated.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/taskeig_b200.h"
#include "device_types.h"
#include "launch.h"
#include "plan.h"
#include "qw_ring.h"
#include "trace.h"

#include <nvtx3/nvToolsExt.h>

namespace teig {

thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

#define TEIG_CUDA(expr)                                                                          \
    do {                                                                                         \
        cudaError_t _e = (expr);                                                                 \
        if (_e != cudaSuccess)                                                                   \
            throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(_e) + " at " + \
                                     __FILE__ + ":" + std::to_string(__LINE__));                 \
    } while (0)

int64_t default_tile_size(int64_t n) {
    // reference tiled_matrix.cpp:168-172
    if (n >= 1000) return 128;
    const int64_t base = std::max<int64_t>(32, n / 8);
    return ((base + 7) / 8) * 8;
}

// Folds the window outcomes of one executed pass into the block bookkeeping,
// in plan order (reference reorder.cpp:366-397).  st_by_plan: status per
// window in plan order; order/stuck: per-block pools (WinDesc::blk_off).
// Returns true when a window deviated from the plan (rejection or layout
// mismatch), i.e. a replanning pass is needed.
//
// Deviation semantics.  The reference plans one group at a time and stops
// folding at the first deviating window (reorder.cpp:372-395); here all
// groups' chains are planned up front and pipelined, so windows of later
// groups may already have run when a window deviates.  The window kernels
// carry a device-side deviation level (window_reorder.cu): once a window of
// level L deviates, every window of a level > L is skipped (status
// kWinSkipped, Q_w = I).  Every window that did run therefore ran on exactly
// its planned layout (no deviation before its level means the plan's
// simulated state is the true state), and folding the executed windows in
// plan order reproduces the device's block arrangement; the skipped windows
// are replanned from that state in the next pass.  Windows that ran at
// levels <= L but belong to groups after the deviating one are folded too
// (the reference would not have run them yet): the final permutation and the
// rejected blocks agree with the reference whenever its swap decisions do,
// and a stale plan can never move an unselected block (the reference's own
// caveat).  `plan` logs every window that ran or deviated, not the
// skipped ones.
bool fold_outcomes(const ReorderPlan& plan, std::vector<BlockState>& blocks, const std::vector<int32_t>& st_by_plan,
                   const std::vector<uint8_t>& order, const std::vector<uint8_t>& stuck,
                   std::vector<int64_t>& rejected, std::vector<int64_t>& plan_log, bool strict) {
    bool deviated = false;
    const int64_t nw = (int64_t)plan.windows.size();
    std::vector<int64_t> start(blocks.size() + 1, 0);
    for (size_t i = 0; i < blocks.size(); ++i) start[i + 1] = start[i] + blocks[i].size;
    std::vector<BlockState> slice;
    for (int64_t wi = 0; wi < nw; ++wi) {
        const PlannedWindow& w = plan.windows[wi];
        const int32_t st = st_by_plan[wi];
        if (st & kWinSkipped) {
            deviated = true;
            continue;
        }
        plan_log.push_back(w.wtop);
        plan_log.push_back(w.wbot - w.wtop);
        plan_log.push_back(w.count);
        if (!(st & kWinExecuted)) {
            deviated = true;
            continue;
        }
        bool consistent = start[w.first_block] == w.wtop &&
                          w.first_block + w.count <= (int64_t)blocks.size();
        for (int64_t i = 0; consistent && i < w.count; ++i)
            consistent = blocks[w.first_block + i].size == plan.sizes[w.blk_off + i];
        if (!consistent)
            throw std::runtime_error("reorder: block bookkeeping diverged from the device layout");
        slice.assign(blocks.begin() + w.first_block, blocks.begin() + w.first_block + w.count);
        for (int64_t i = 0; i < w.count; ++i) blocks[w.first_block + i] = slice[order[w.blk_off + i]];
        for (int64_t i = 0; i < w.count; ++i) start[w.first_block + i + 1] = start[w.first_block + i] + blocks[w.first_block + i].size;
        if (st & kWinStuck) {
            deviated = true;
            for (int64_t i = 0; i < w.count; ++i)
                if (stuck[w.blk_off + i]) {
                    if (strict) throw std::domain_error("reorder_schur: swap rejected in strict mode");
                    rejected.push_back(slice[i].orig);
                    for (auto& b : blocks)
                        if (b.orig == slice[i].orig) b.selected = 0;
                }
        }
    }
    return deviated;
}

namespace {

struct DevBuf {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    DevBuf(size_t bytes, cudaStream_t st) : s(st) {
        if (bytes) TEIG_CUDA(lib_malloc_async(&p, bytes, st));
    }
    ~DevBuf() {
        if (p) cudaFreeAsync(p, s);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

// Device staging of the host entry points.  With memory retention on
// (teig_set_memory_retention) it is kept between calls (the host path of a
// 40000-order problem stages 25.6 GB; mapping it anew every call cost
// 0.14-0.95 s and slowed the first kernels that touched it): one cache per
// DEVICE, grown on demand, guarded for concurrent host calls.  Off (the
// default): allocated per call.
struct HostStaging {
    std::mutex mu;
    void* p = nullptr;
    size_t bytes = 0;
    int dev = 0;
    void release() {
        if (p) {
            int cur = 0;
            cudaGetDevice(&cur);
            cudaSetDevice(dev);
            cudaFree(p);
            cudaSetDevice(cur);
        }
        p = nullptr;
        bytes = 0;
    }
};
std::mutex g_staging_mu;
std::map<int, HostStaging*> g_staging;
HostStaging& host_staging() {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_staging_mu);
    HostStaging*& hs = g_staging[dev];
    if (!hs) {
        hs = new HostStaging;  // lives for the process (released by teig_release_memory)
        hs->dev = dev;
    }
    return *hs;
}

struct PassResult {
    int64_t windows = 0, levels = 0, launches = 0;
    bool deviated = false;
    double ms_window = 0, ms_left = 0, ms_right = 0, ms_factor = 0;
    double flops_factor_exec = 0;
    double flops_dmma = 0;
};

}  // namespace

// Execution trace of the calls made on this thread (teig_trace_enable): one
// task record per kernel launch -- the reference's ExecutionReport schema
// (runtime.hpp:50-60: label, worker = stream, start_ns / end_ns from CUDA
// events relative to the call's first event) -- plus, for reorder calls, one
// record per planned window (pass, level, position, order, blocks, group,
// status).
thread_local TraceState g_trace;

void TraceState::begin(cudaStream_t s) {
    tasks.clear();
    wins.clear();
    pass = 0;
    if (!origin) TEIG_CUDA(cudaEventCreate(&origin));
    TEIG_CUDA(cudaEventRecord(origin, s));
}

namespace {

// Event pairs bracketing launches when profiling is on.
struct EventLog {
    bool on = false;
    std::vector<cudaEvent_t> ev;
    std::vector<std::pair<int, int>> spans[4];  // (start idx, end idx) per class
    struct Meta {
        int cls, level, worker, start, end;
    };
    std::vector<Meta> meta;  // every span in launch order (trace)
    int record(cudaStream_t s) {
        cudaEvent_t e;
        TEIG_CUDA(cudaEventCreate(&e));
        TEIG_CUDA(cudaEventRecord(e, s));
        ev.push_back(e);
        return (int)ev.size() - 1;
    }
    double total(int cls) {
        double t = 0;
        for (auto& sp : spans[cls]) {
            float ms = 0;
            TEIG_CUDA(cudaEventElapsedTime(&ms, ev[sp.first], ev[sp.second]));
            t += ms;
        }
        return t;
    }
    ~EventLog() {
        for (auto e : ev) cudaEventDestroy(e);
    }
};

// Host entry point only: device -> host copies of the parts of S and Q that
// no later level touches, issued on a copy stream while the remaining levels
// run.  A window [a, b) writes S rows [0, b) only (window block, left panel
// rows, right panel rows above) and Q columns [a, b) only, so after level L
// the S rows >= max b and the Q columns outside [min a, max b) of the levels
// after L are final.  s_hi: S rows [s_hi, n) copied; Q columns [0, q_lo) and
// [q_hi, n) copied.  A replanning pass invalidates the early copies (the
// final copy then moves everything).
struct HostDrain {
    double* hS = nullptr;
    int64_t lds = 0;
    double* hQ = nullptr;
    int64_t ldq = 0;
    cudaStream_t ds = nullptr;
    cudaEvent_t evS = nullptr, evQ = nullptr;
    int64_t s_hi = 0, q_lo = 0, q_hi = 0;
    bool valid = true;
    int64_t min_chunk = 512;
    int64_t d2h_bytes = 0;  // drained so far
};

// Executes one planned pass on the device and folds the outcomes into `blocks`.
PassResult run_pass(ReorderPlan& plan, int64_t n, double* dS, int64_t lds, double* dQ, int64_t ldq,
                    std::vector<BlockState>& blocks, std::vector<int64_t>& rejected,
                    std::vector<int64_t>& plan_log, bool strict, bool overlap, bool profile,
                    cudaStream_t stream, cudaStream_t stream2, cudaEvent_t ev, bool short_q,
                    HostDrain* drain = nullptr, FactorSupport* qsupp = nullptr, cudaStream_t stream3 = nullptr) {
    PassResult pr;
    EventLog lg;
    lg.on = profile || g_trace.on;
    // profiling: the update kernels' DMMA counters around the pass (device
    // syncs: a measurement mode)
    unsigned long long dmma0 = 0;
    if (profile) {
        TEIG_CUDA(cudaDeviceSynchronize());
        dmma0 = dmma_count_bulk() + dmma_count_cp();
    }
    const int64_t nw = (int64_t)plan.windows.size();
    schedule_levels(plan, n);
    const int32_t nl = plan.n_levels;
    // order windows by level (stable: plan order inside a level)
    std::vector<int64_t> idx(nw);
    for (int64_t i = 0; i < nw; ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(),
                     [&](int64_t x, int64_t y) { return plan.windows[x].level < plan.windows[y].level; });
    std::vector<WinDesc> descs(nw);
    std::vector<int64_t> lvl_off(nl + 1, 0), tl(nl, 0), tr(nl, 0), tq(nl, 0);
    int dmax = 0;
    int64_t qw_total = 0;
    for (int64_t k = 0; k < nw; ++k) {
        const PlannedWindow& w = plan.windows[idx[k]];
        WinDesc& dsc = descs[k];
        const int L = w.level;
        dsc.a = (int32_t)w.wtop;
        dsc.d = (int32_t)(w.wbot - w.wtop);
        dsc.nb = (int32_t)w.count;
        dsc.level = L;
        dsc.qw_off = qw_total;
        qw_total += (int64_t)dsc.d * dsc.d;
        dsc.blk_off = w.blk_off;
        dsc.tl_pref = (int32_t)tl[L];
        dsc.tr_pref = (int32_t)tr[L];
        dsc.tq_pref = (int32_t)tq[L];
        dsc.pad = 0;
        dsc.lc0 = (int32_t)w.wbot;
        dsc.lc1 = (int32_t)n;
        dsc.rr0 = 0;
        dsc.rr1 = (int32_t)w.wtop;
        int64_t q0 = 0, q1 = n;  // factor rows: all, or the tracked support (plan.h)
        if (dQ && qsupp && qsupp->on) qsupp->window(w.wtop, w.wbot, &q0, &q1);
        pr.flops_factor_exec += 2.0 * double(dsc.d) * double(dsc.d) * double(q1 - q0);
        dsc.qr0 = (int32_t)q0;
        dsc.qr1 = (int32_t)q1;
        tl[L] += (n - w.wbot + kLeftBN - 1) / kLeftBN;
        tr[L] += (w.wtop + kRightBM - 1) / kRightBM;
        if (dQ) tq[L] += (q1 - q0 + kRightBM - 1) / kRightBM;
        lvl_off[L + 1]++;
        dmax = std::max(dmax, dsc.d);
    }
    for (int L = 0; L < nl; ++L) lvl_off[L + 1] += lvl_off[L];
    const int dmax_k = dmax <= 64 ? 64 : 128;
    // Q_w ring: level L's accumulators live in region L % K; region reuse by
    // level L + K waits for level L's factor update (the only reader not
    // already ordered before it on the critical-path stream)
    const QwRing ring = make_qw_ring(descs, lvl_off, nl, 1);
    qw_total = ring.total;
    // Look-ahead (overlap mode): the S updates of level L split into the tiles
    // that touch a level-(L+1) window's diagonal block -- "critical", run on
    // the window stream right after window L -- and the rest -- "bulk", on a
    // third stream, concurrently with window L+1 (on SMs the capped bulk grid
    // leaves free).  A window's right panel meets a next-level window W' only
    // in rows [a', a) when W' straddles a, its left panel only in columns
    // [b, b') when W' straddles b, so each window's critical part is one row
    // range of its right update and one column range of its left update (the
    // hull over the next-level windows it overlaps).  Every S element still
    // receives its updates in level order (critical L+1 waits for bulk L) and,
    // within a level, left before right (below); a row / column of an update
    // does not depend on how the rows / columns are tiled: the result is bit
    // for bit the serial order's.
    // TEIG_NO_LOOKAHEAD=1: the serial order.
    const bool no_la = getenv("TEIG_NO_LOOKAHEAD") && atoi(getenv("TEIG_NO_LOOKAHEAD"));  // read per pass (tests toggle it)
    const bool lookahead = overlap && stream3 && !no_la && nl > 1;
    std::vector<WinDesc> cdesc, bdesc;
    std::vector<int64_t> ctl(nl, 0), ctr(nl, 0), btl(nl, 0), btr(nl, 0);
    std::vector<int> bulk_cap(nl, 0);
    if (lookahead) {
        cdesc = descs;
        bdesc = descs;
        const int sms = device_sm_count();
        std::vector<std::pair<int32_t, int32_t>> nx;
        for (int L = 0; L < nl; ++L) {
            nx.clear();
            if (L + 1 < nl)
                for (int64_t k = lvl_off[L + 1]; k < lvl_off[L + 2]; ++k)
                    nx.push_back({descs[k].a, descs[k].a + descs[k].d});
            std::sort(nx.begin(), nx.end());  // disjoint: also sorted by end
            const int64_t k0 = lvl_off[L], k1 = lvl_off[L + 1];
            std::vector<int32_t> xs(k1 - k0), ys(k1 - k0);
            for (int64_t k = k0; k < k1; ++k) {
                const int32_t a = descs[k].a, b = descs[k].a + descs[k].d;
                int32_t x = a, y = b;
                auto it = std::partition_point(nx.begin(), nx.end(),
                                               [&](const std::pair<int32_t, int32_t>& w) { return w.second <= a; });
                for (; it != nx.end() && it->first < b; ++it) {
                    x = std::min(x, it->first);
                    y = std::max(y, it->second);
                }
                xs[k - k0] = x;
                ys[k - k0] = y;
            }
            // same-level order: an element where window V's left panel meets
            // window W's right panel gets V's left update before W's right
            // one (the serial launch order; the two commute only up to
            // rounding).  W's critical right rows [x_W, a_W) run before the
            // bulk left updates, so every V whose rows they reach takes the
            // columns up to b_W into its critical left range.
            for (int64_t k = k0; k < k1; ++k) {
                const int32_t aw = descs[k].a, bw = aw + descs[k].d, xw = xs[k - k0];
                if (xw >= aw) continue;
                for (int64_t v = k0; v < k1; ++v) {
                    const int32_t av = descs[v].a, bv = av + descs[v].d;
                    if (bv <= aw && bv > xw) ys[v - k0] = std::max(ys[v - k0], bw);
                }
            }
            for (int64_t k = k0; k < k1; ++k) {
                const int32_t a = descs[k].a, b = descs[k].a + descs[k].d;
                const int32_t x = xs[k - k0], y = std::min<int32_t>(ys[k - k0], (int32_t)n);
                WinDesc& c = cdesc[k];
                WinDesc& u = bdesc[k];
                c.lc0 = b;
                c.lc1 = y;
                c.rr0 = x;
                c.rr1 = a;
                u.lc0 = y;
                u.lc1 = (int32_t)n;
                u.rr0 = 0;
                u.rr1 = x;
                c.tl_pref = (int32_t)ctl[L];
                c.tr_pref = (int32_t)ctr[L];
                u.tl_pref = (int32_t)btl[L];
                u.tr_pref = (int32_t)btr[L];
                ctl[L] += (y - b + kLeftBN - 1) / kLeftBN;
                ctr[L] += (a - x + kRightBM - 1) / kRightBM;
                btl[L] += (n - y + kLeftBN - 1) / kLeftBN;
                btr[L] += (x + kRightBM - 1) / kRightBM;
            }
            if (L + 1 < nl) {
                // split only where it pays: the bulk and factor updates,
                // squeezed onto the SMs the next level's window CTAs leave
                // free, must end before window + bulk would in the serial order
                // (where the factor updates fill the SMs the window kernel
                // leaves idle), with a 10 % margin for the extra launches.
                // Window ~0.65 ms per order-128 step chain on this B200, tiles
                // ~25 TF/s.  C2's levels split; C4's do not (~92 windows per
                // level, and 40000-long panels where there are fewer).
                const int64_t nwn = lvl_off[L + 2] - lvl_off[L + 1];
                const double tile_ms = 2.0 * 64.0 * double(dmax) * double(dmax) / 25e12 * 1e3;
                const double bulk_ms = double(btl[L] + btr[L]) * tile_ms;
                const double side_ms = bulk_ms + (dQ ? double(tq[L]) * tile_ms : 0.0);
                const double win_ms = 0.65 * double(dmax) / 128.0;
                if (nwn <= sms / 2 && side_ms * sms / double(sms - nwn) < 0.9 * (win_ms + bulk_ms))
                    bulk_cap[L] = sms - (int)nwn;
            }
        }
    }
    // early host drain: max b / min a over the levels after L
    std::vector<int64_t> after_hi, after_lo;
    if (drain && drain->valid) {
        after_hi.assign(nl + 1, 0);
        after_lo.assign(nl + 1, n);
        for (int L = nl - 1; L >= 0; --L) {
            after_hi[L] = after_hi[L + 1];
            after_lo[L] = after_lo[L + 1];
            for (int64_t k = lvl_off[L]; k < lvl_off[L + 1]; ++k) {
                after_hi[L] = std::max<int64_t>(after_hi[L], descs[k].a + descs[k].d);
                after_lo[L] = std::min<int64_t>(after_lo[L], descs[k].a);
            }
        }
    }

    const size_t ne = plan.sizes.size();
    DevBuf d_desc(sizeof(WinDesc) * nw, stream), d_qw(sizeof(double) * std::max<int64_t>(qw_total, 1), stream),
        d_sizes(ne + 1, stream), d_sel(ne + 1, stream), d_order(ne + 1, stream), d_stuck(ne + 1, stream),
        d_status(sizeof(int32_t) * nw, stream), d_devlvl(sizeof(int32_t), stream);
    TEIG_CUDA(cudaMemsetAsync(d_devlvl.p, 0x7f, sizeof(int32_t), stream));
    TEIG_CUDA(cudaMemcpyAsync(d_desc.p, descs.data(), sizeof(WinDesc) * nw, cudaMemcpyHostToDevice, stream));
    DevBuf d_cdesc(lookahead ? sizeof(WinDesc) * nw : 0, stream), d_bdesc(lookahead ? sizeof(WinDesc) * nw : 0, stream);
    StreamEvents la_ev(lookahead ? 2 : 0);  // [0] critical(L) done, [1] bulk(L) done
    if (lookahead) {
        TEIG_CUDA(cudaMemcpyAsync(d_cdesc.p, cdesc.data(), sizeof(WinDesc) * nw, cudaMemcpyHostToDevice, stream));
        TEIG_CUDA(cudaMemcpyAsync(d_bdesc.p, bdesc.data(), sizeof(WinDesc) * nw, cudaMemcpyHostToDevice, stream));
        TEIG_CUDA(cudaEventRecord(la_ev.ev[0], stream));  // the third stream starts after the uploads
        TEIG_CUDA(cudaStreamWaitEvent(stream3, la_ev.ev[0], 0));
    }
    TEIG_CUDA(cudaMemcpyAsync(d_sizes.p, plan.sizes.data(), ne, cudaMemcpyHostToDevice, stream));
    TEIG_CUDA(cudaMemcpyAsync(d_sel.p, plan.sel.data(), ne, cudaMemcpyHostToDevice, stream));

    const WinDesc* dd = d_desc.as<WinDesc>();
    RingEvents ring_ev(ring.k > 0 && dQ && overlap ? ring.k : 0);
    int64_t launches = 0;
    // TEIG_WINDOW_PROF=1: per-warp phase timing of every window CTA (diagnostics)
    static const bool wprof = getenv("TEIG_WINDOW_PROF") && atoi(getenv("TEIG_WINDOW_PROF")) != 0;
    DevBuf d_prof(wprof ? sizeof(unsigned long long) * nw * kWindowThreads / 32 * 4 : 0, stream);
    if (wprof) TEIG_CUDA(cudaMemsetAsync(d_prof.p, 0, sizeof(unsigned long long) * nw * kWindowThreads / 32 * 4, stream));
    // runs `f` on stream `st`, bracketed by events of class `cls` when profiling
    int cur_level = 0;
    auto timed = [&](int cls, cudaStream_t st, int64_t ntiles, auto&& f) {
        if (ntiles <= 0) return;
        int e0 = lg.on ? lg.record(st) : -1;
        TEIG_CUDA(f());
        ++launches;
        if (lg.on) {
            const int e1 = lg.record(st);
            lg.spans[cls].push_back({e0, e1});
            lg.meta.push_back({cls, cur_level, st == stream ? 0 : 1, e0, e1});
        }
    };
    // TEIG_LAUNCH_LOG=1: per-level tile counts on stderr (to pair ncu launch
    // indices with algorithmic bytes / flops)
    const bool launch_log = getenv("TEIG_LAUNCH_LOG") && atoi(getenv("TEIG_LAUNCH_LOG"));
    for (int L = 0; L < nl; ++L) {
        const int64_t o = lvl_off[L], cnt = lvl_off[L + 1] - lvl_off[L];
        cur_level = L;
        nvtxRangePushA("teig reorder level");
        if (launch_log)
            fprintf(stderr, "[teig level] %d windows %lld left_tiles %lld right_tiles %lld factor_tiles %lld split %d\n",
                    L, (long long)cnt, (long long)tl[L], (long long)tr[L], (long long)tq[L],
                    lookahead && bulk_cap[L] > 0 ? 1 : 0);
        if (ring_ev.n && L >= ring.k) TEIG_CUDA(cudaStreamWaitEvent(stream, ring_ev.ev[L % ring.k], 0));
        timed(0, stream, cnt, [&] {
            return launch_window_reorder(dd + o, (int)cnt, dmax_k, dS, lds, d_qw.as<double>(), d_sizes.as<uint8_t>(),
                                         d_sel.as<uint8_t>(), d_order.as<uint8_t>(), d_stuck.as<uint8_t>(),
                                         d_status.as<int32_t>() + o, stream,
                                         wprof ? d_prof.as<unsigned long long>() + o * (kWindowThreads / 32) * 4 : nullptr,
                                         d_devlvl.as<int32_t>());
        });
        // the factor updates of level L on the low-priority stream (after the
        // window; in look-ahead mode after the critical tiles too, so its
        // short CTAs do not take the SMs those need)
        auto factor_overlapped = [&](int short_tiles) {
            TEIG_CUDA(cudaEventRecord(ev, stream));
            TEIG_CUDA(cudaStreamWaitEvent(stream2, ev, 0));
            timed(3, stream2, tq[L], [&] {
                return launch_update_right(dd + o, (int)cnt, (int)tq[L], dmax_k, d_qw.as<double>(), dQ, ldq, (int)n,
                                           true, stream2, n, n, short_q, 0, short_tiles);
            });
            if (ring_ev.n) TEIG_CUDA(cudaEventRecord(ring_ev.ev[L % ring.k], stream2));
        };
        // look-ahead split of this level (next level's window kernels find
        // free SMs beside its bulk updates); otherwise its S updates run
        // whole on the window stream, as in the serial order
        const bool split = lookahead && bulk_cap[L] > 0;
        if (lookahead && L > 0) TEIG_CUDA(cudaStreamWaitEvent(stream, la_ev.ev[1], 0));  // bulk(L-1) first
        if (dQ && overlap && !split) factor_overlapped(8);
        if (split) {
            const WinDesc* cd = d_cdesc.as<WinDesc>() + o;
            const WinDesc* bd = d_bdesc.as<WinDesc>() + o;
            // the critical tiles gate window L+1: one tile per CTA (-1)
            timed(1, stream, ctl[L], [&] {
                return launch_update_left(cd, (int)cnt, (int)ctl[L], dmax_k, d_qw.as<double>(), dS, lds, (int)n,
                                          stream, n, n, -1);
            });
            timed(2, stream, ctr[L], [&] {
                return launch_update_right(cd, (int)cnt, (int)ctr[L], dmax_k, d_qw.as<double>(), dS, lds, (int)n,
                                           false, stream, n, n, false, -1);
            });
            TEIG_CUDA(cudaEventRecord(la_ev.ev[0], stream));
            TEIG_CUDA(cudaStreamWaitEvent(stream3, la_ev.ev[0], 0));
            // a split level's window chain is the critical path: shorter factor
            // CTAs (2 tiles) free the SMs the next window kernel needs sooner
            if (dQ) factor_overlapped(2);
            timed(1, stream3, btl[L], [&] {
                return launch_update_left(bd, (int)cnt, (int)btl[L], dmax_k, d_qw.as<double>(), dS, lds, (int)n,
                                          stream3, n, n, bulk_cap[L]);
            });
            timed(2, stream3, btr[L], [&] {
                return launch_update_right(bd, (int)cnt, (int)btr[L], dmax_k, d_qw.as<double>(), dS, lds, (int)n,
                                           false, stream3, n, n, false, bulk_cap[L]);
            });
            TEIG_CUDA(cudaEventRecord(la_ev.ev[1], stream3));
        } else {
            timed(1, stream, tl[L], [&] {
                return launch_update_left(dd + o, (int)cnt, (int)tl[L], dmax_k, d_qw.as<double>(), dS, lds, (int)n,
                                          stream, n, n);
            });
            timed(2, stream, tr[L], [&] {
                return launch_update_right(dd + o, (int)cnt, (int)tr[L], dmax_k, d_qw.as<double>(), dS, lds, (int)n,
                                           false, stream, n, n);
            });
        }
        if (dQ && !overlap)
            timed(3, stream, tq[L], [&] {
                return launch_update_right(dd + o, (int)cnt, (int)tq[L], dmax_k, d_qw.as<double>(), dQ, ldq, (int)n,
                                           true, stream, n, n);
            });
        if (drain && drain->valid && L + 1 < nl) {
            const int64_t hi = after_hi[L + 1], lo = after_lo[L + 1];
            if (drain->s_hi - hi >= drain->min_chunk) {  // S rows [hi, s_hi): final after this level's S work
                TEIG_CUDA(cudaEventRecord(drain->evS, split ? stream3 : stream));
                TEIG_CUDA(cudaStreamWaitEvent(drain->ds, drain->evS, 0));
                // row r of a Schur form is zero left of column r-1: columns [hi-1, n)
                const int64_t c0 = std::max<int64_t>(hi - 1, 0);
                TEIG_CUDA(cudaMemcpy2DAsync(drain->hS + hi + c0 * drain->lds, drain->lds * sizeof(double),
                                            dS + hi + c0 * lds, lds * sizeof(double),
                                            (size_t)(drain->s_hi - hi) * sizeof(double), (size_t)(n - c0),
                                            cudaMemcpyDeviceToHost, drain->ds));
                drain->d2h_bytes += (drain->s_hi - hi) * (n - c0) * (int64_t)sizeof(double);
                drain->s_hi = hi;
            }
            if (dQ && drain->hQ &&
                (drain->q_hi - hi >= drain->min_chunk || lo - drain->q_lo >= drain->min_chunk)) {
                TEIG_CUDA(cudaEventRecord(drain->evQ, overlap ? stream2 : stream));
                TEIG_CUDA(cudaStreamWaitEvent(drain->ds, drain->evQ, 0));
                auto cols = [&](int64_t c0, int64_t c1) {
                    if (c1 > c0) {
                        TEIG_CUDA(cudaMemcpy2DAsync(drain->hQ + c0 * drain->ldq, drain->ldq * sizeof(double),
                                                    dQ + c0 * ldq, ldq * sizeof(double), (size_t)n * sizeof(double),
                                                    (size_t)(c1 - c0), cudaMemcpyDeviceToHost, drain->ds));
                        drain->d2h_bytes += n * (c1 - c0) * (int64_t)sizeof(double);
                    }
                };
                if (drain->q_hi - hi >= drain->min_chunk) {
                    cols(hi, drain->q_hi);
                    drain->q_hi = hi;
                }
                if (lo - drain->q_lo >= drain->min_chunk) {
                    cols(drain->q_lo, lo);
                    drain->q_lo = lo;
                }
            }
        }
        nvtxRangePop();
    }
    if (dQ && overlap) {
        TEIG_CUDA(cudaEventRecord(ev, stream2));
        TEIG_CUDA(cudaStreamWaitEvent(stream, ev, 0));
    }
    if (lookahead) TEIG_CUDA(cudaStreamWaitEvent(stream, la_ev.ev[1], 0));  // the last bulk updates
    // one readback of all window outcomes
    std::vector<int32_t> status(nw);
    std::vector<uint8_t> order(ne + 1), stuck(ne + 1);
    TEIG_CUDA(cudaMemcpyAsync(status.data(), d_status.p, sizeof(int32_t) * nw, cudaMemcpyDeviceToHost, stream));
    TEIG_CUDA(cudaMemcpyAsync(order.data(), d_order.p, ne, cudaMemcpyDeviceToHost, stream));
    TEIG_CUDA(cudaMemcpyAsync(stuck.data(), d_stuck.p, ne, cudaMemcpyDeviceToHost, stream));
    TEIG_CUDA(cudaStreamSynchronize(stream));
    if (wprof) {
        const int NW = kWindowThreads / 32;
        std::vector<unsigned long long> pf((size_t)nw * NW * 4);
        TEIG_CUDA(cudaMemcpy(pf.data(), d_prof.p, pf.size() * 8, cudaMemcpyDeviceToHost));
        double p1[8] = {0}, p2[8] = {0}, steps = 0, kc = 0, kmax = 0;
        for (int64_t k = 0; k < nw; ++k) {
            for (int w = 0; w < NW; ++w) {
                p1[w] += pf[(k * NW + w) * 4 + 0];
                p2[w] += pf[(k * NW + w) * 4 + 1];
            }
            steps += pf[(k * NW) * 4 + 2];
            kc += pf[(k * NW) * 4 + 3];
            kmax = std::max(kmax, (double)pf[(k * NW) * 4 + 3]);
        }
        fprintf(stderr, "[teig window prof] windows=%lld levels=%d steps/window=%.1f kernel cycles/window=%.0f\n",
                (long long)nw, nl, steps / nw, kc / nw);
        for (int w = 0; w < NW; ++w)
            fprintf(stderr, "  warp %d: phase1 cycles/step=%.0f phase2 cycles/step=%.0f\n", w, p1[w] / steps,
                    p2[w] / steps);
        fprintf(stderr, "  kernel cycles per step (window avg) = %.0f\n", kc / steps);
    }
    std::vector<int32_t> st_by_plan(nw);
    for (int64_t k = 0; k < nw; ++k) st_by_plan[idx[k]] = status[k];
    pr.deviated = fold_outcomes(plan, blocks, st_by_plan, order, stuck, rejected, plan_log, strict);
    pr.windows = 0;
    for (int32_t st : status) pr.windows += (st & kWinSkipped) ? 0 : 1;  // = entries logged in `plan`
    pr.levels = nl;
    pr.launches = launches;
    if (profile) {
        TEIG_CUDA(cudaDeviceSynchronize());
        pr.flops_dmma = 512.0 * double(dmma_count_bulk() + dmma_count_cp() - dmma0);
    }
    if (g_trace.on) {  // everything above synchronized: the events are complete
        static const char* kCls[4] = {"W", "L", "R", "Q"};
        for (const auto& m : lg.meta) {
            float t0 = 0, t1 = 0;
            TEIG_CUDA(cudaEventElapsedTime(&t0, g_trace.origin, lg.ev[m.start]));
            TEIG_CUDA(cudaEventElapsedTime(&t1, g_trace.origin, lg.ev[m.end]));
            g_trace.tasks.push_back({std::string("reorder:") + kCls[m.cls] + ":p" + std::to_string(g_trace.pass) +
                                         ":l" + std::to_string(m.level),
                                     m.worker, (int64_t)(t0 * 1e6), (int64_t)(t1 * 1e6)});
        }
        for (int64_t k = 0; k < nw; ++k) {
            const PlannedWindow& w = plan.windows[idx[k]];
            g_trace.wins.push_back({g_trace.pass, w.level, w.wtop, w.wbot - w.wtop, w.count, w.group, status[k]});
        }
        ++g_trace.pass;
    }
    if (lg.on) {
        pr.ms_window = lg.total(0);
        pr.ms_left = lg.total(1);
        pr.ms_right = lg.total(2);
        pr.ms_factor = lg.total(3);
    }
    return pr;
}

// The window kernels and S updates (the critical path) run on an internal
// highest-priority stream ordered after / before the caller's stream, the Q
// updates on a lowest-priority one in short CTAs (update_tma.cu), so window
// CTAs take SMs ahead of pending Q-update CTAs as they free up: C2 (n=10000,
// window kernels ~50 % of the step) 0.161 -> 0.149 s, C4 unchanged.
// TEIG_NO_PRIO=1: both on default priority, Q updates persistent.
// Whatever happens inside the call (a CUDA error thrown mid-pass included),
// the destructor joins both internal streams into the caller's stream before
// releasing them, so no enqueued work outlives the call unordered.
// The internal streams are created once per host thread and device and then
// reused: a stream's hardware work queue is fixed when it is created, and
// creating three fresh streams per call cycled them through the device's
// queues (8 by default) so that every few calls one shared a queue with the
// caller's stream -- false dependencies, C2 calls at 107 instead of 101 ms.
struct InternalStreams {
    cudaStream_t hi = nullptr, lo = nullptr, mid = nullptr;
    ~InternalStreams() {  // thread exit (errors ignored: the context may be gone)
        if (hi) cudaStreamDestroy(hi);
        if (lo) cudaStreamDestroy(lo);
        if (mid) cudaStreamDestroy(mid);
        cudaGetLastError();
    }
};
InternalStreams& internal_streams(bool prio) {
    thread_local std::map<std::pair<int, bool>, InternalStreams> cache;
    int dev = 0;
    TEIG_CUDA(cudaGetDevice(&dev));
    InternalStreams& st = cache[{dev, prio}];
    if (!st.lo) {
        int least = 0, greatest = 0;
        TEIG_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        TEIG_CUDA(cudaStreamCreateWithPriority(&st.lo, cudaStreamNonBlocking, prio ? least : 0));
        // the look-ahead S updates (run_pass): between the two
        TEIG_CUDA(cudaStreamCreateWithPriority(&st.mid, cudaStreamNonBlocking, prio ? (least + greatest) / 2 : 0));
        if (prio) TEIG_CUDA(cudaStreamCreateWithPriority(&st.hi, cudaStreamNonBlocking, greatest));
    }
    return st;
}

struct StreamPair {
    cudaStream_t s1 = nullptr, s2 = nullptr, s3 = nullptr, caller = nullptr;
    cudaEvent_t ev = nullptr, join = nullptr;
    bool prio = true;
    explicit StreamPair(cudaStream_t user) : s1(user), caller(user) {
        prio = !(getenv("TEIG_NO_PRIO") && atoi(getenv("TEIG_NO_PRIO")));
        try {
            TEIG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            TEIG_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
            InternalStreams& st = internal_streams(prio);
            s2 = st.lo;
            s3 = st.mid;
            // every internal stream starts after the caller's earlier work
            TEIG_CUDA(cudaEventRecord(join, user));
            TEIG_CUDA(cudaStreamWaitEvent(s2, join, 0));
            TEIG_CUDA(cudaStreamWaitEvent(s3, join, 0));
            if (prio) {
                s1 = st.hi;
                TEIG_CUDA(cudaStreamWaitEvent(s1, join, 0));
            }
        } catch (...) {
            release();
            throw;
        }
    }
    // the factor updates run in short CTAs on the low-priority stream
    bool short_factor_ctas(bool overlap) const { return prio && overlap; }
    void finish() {
        if (s1 != caller) {
            TEIG_CUDA(cudaEventRecord(join, s1));
            TEIG_CUDA(cudaStreamWaitEvent(caller, join, 0));
        }
    }
    void release() {
        // join (errors ignored: this also runs on the error path)
        if (join) {
            if (s2 && cudaEventRecord(join, s2) == cudaSuccess) cudaStreamWaitEvent(caller, join, 0);
            if (s3 && cudaEventRecord(join, s3) == cudaSuccess) cudaStreamWaitEvent(caller, join, 0);
            if (s1 && s1 != caller && cudaEventRecord(join, s1) == cudaSuccess) cudaStreamWaitEvent(caller, join, 0);
        }
        if (ev) cudaEventDestroy(ev);
        if (join) cudaEventDestroy(join);  // (the streams are kept: internal_streams)
        ev = join = nullptr;
        s2 = s3 = nullptr;
        s1 = caller;
        cudaGetLastError();
    }
    ~StreamPair() { release(); }
};

}  // namespace

int reorder_schur_device(int64_t n, double* dS, int64_t lds, double* dQ, int64_t ldq, int64_t nb,
                         const uint8_t* sizes, const uint8_t* flags, const teig_reorder_opts* opts,
                         int64_t* perm, int64_t* rejected_out, int64_t* plan_out, int64_t plan_cap,
                         teig_reorder_info* info, cudaStream_t stream, cudaEvent_t q_ready = nullptr,
                         HostDrain* drain = nullptr, FactorSupport* qsupp_in = nullptr) {
    if (n < 1) return set_error(-1, "n must be >= 1");
    if (!dS) return set_error(-2, "S is null");
    if (lds < n) return set_error(-3, "lds < n");
    if (dQ && ldq < n) return set_error(-5, "ldq < n");
    if (nb < 0 || (nb > 0 && (!sizes || !flags))) return set_error(-6, "malformed selection");
    teig_reorder_opts o;
    teig_reorder_opts_default(&o);
    if (opts) o = *opts;
    int64_t ws = std::max<int64_t>(o.window_size ? o.window_size : default_tile_size(n), 8);
    // windows larger than one CTA's shared memory holds run at 128 (the
    // reference takes any size, reorder.cpp:221-222): same final arrangement,
    // a different window plan
    ws = std::min<int64_t>(ws, 128);
    if (n > (int64_t)2147483647) return set_error(TEIG_ERR_UNSUPPORTED, "n too large");

    std::vector<BlockState> blocks(nb);
    int64_t rows = 0;
    for (int64_t i = 0; i < nb; ++i) {
        if (sizes[i] != 1 && sizes[i] != 2) return set_error(-8, "block sizes must be 1 or 2");
        blocks[i] = BlockState{sizes[i], (uint8_t)(flags[i] ? 1 : 0), (uint32_t)i};
        rows += sizes[i];
    }
    if (rows != n) return set_error(-8, "reorder_schur: selection does not match s");

    teig_reorder_info inf{};
    inf.clean = 1;
    std::vector<int64_t> rejected, plan_log;
    try {
        StreamPair sp(stream);
        if (g_trace.on) g_trace.begin(sp.s1);  // time origin of this call's trace records
        // the factor's row support (plan.h FactorSupport): from the host path's
        // scan, else one device scan of Q (n^2 reads, ~3 ms at n=40000)
        FactorSupport qsupp;
        static const bool no_supp = getenv("TEIG_NO_Q_SUPPORT") && atoi(getenv("TEIG_NO_Q_SUPPORT"));
        if (dQ && !no_supp && !o.full_factor) {
            if (qsupp_in && qsupp_in->on) {
                qsupp = *qsupp_in;
            } else if (!q_ready) {  // (Q still arriving and no host scan: full updates)
                DevBuf dlo(sizeof(int32_t) * n, sp.s1), dhi(sizeof(int32_t) * n, sp.s1);
                qsupp.lo.resize(n);
                qsupp.hi.resize(n);
                TEIG_CUDA(launch_column_support(dQ, ldq, n, n, dlo.as<int32_t>(), dhi.as<int32_t>(), sp.s1));
                TEIG_CUDA(cudaMemcpyAsync(qsupp.lo.data(), dlo.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, sp.s1));
                TEIG_CUDA(cudaMemcpyAsync(qsupp.hi.data(), dhi.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, sp.s1));
                TEIG_CUDA(cudaStreamSynchronize(sp.s1));
                qsupp.on = true;
            }
        }
        // Q may still be arriving (host entry point): only the Q updates wait
        if (q_ready && dQ) TEIG_CUDA(cudaStreamWaitEvent(o.overlap_factor ? sp.s2 : sp.s1, q_ready, 0));
        double plan_ms = 0.0;
        for (int pass = 0; pass < 64; ++pass) {
            const auto t0 = std::chrono::steady_clock::now();
            ReorderPlan plan = plan_reorder(blocks, ws);
            const auto t1 = std::chrono::steady_clock::now();
            plan_ms += std::chrono::duration<double, std::milli>(t1 - t0).count();
            if (plan.windows.empty()) break;
            if (pass == 0) inf.n_groups = plan.n_groups;
            inf.update_flops += plan_update_flops(plan, n, dQ != nullptr);
            inf.update_bytes += plan_update_bytes(plan, n, dQ != nullptr);
            for (const auto& w : plan.windows) {
                const double d = double(w.wbot - w.wtop);
                inf.flops_left += 2.0 * d * d * double(n - w.wbot);
                inf.flops_right += 2.0 * d * d * double(w.wtop);
                if (dQ) inf.flops_factor += 2.0 * d * d * double(n);
            }
            PassResult pr = run_pass(plan, n, dS, lds, dQ, ldq, blocks, rejected, plan_log, o.strict != 0,
                                     o.overlap_factor != 0, o.profile != 0, sp.s1, sp.s2, sp.ev,
                                     sp.short_factor_ctas(o.overlap_factor != 0),
                                     pass == 0 ? drain : nullptr, &qsupp, sp.s3);
            inf.flops_factor_exec += pr.flops_factor_exec;
            inf.flops_dmma += pr.flops_dmma;
            inf.n_windows += pr.windows;
            inf.n_levels += pr.levels;
            inf.n_launches += pr.launches;
            inf.ms_window += pr.ms_window;
            inf.ms_left += pr.ms_left;
            inf.ms_right += pr.ms_right;
            inf.ms_factor += pr.ms_factor;
            inf.n_passes += 1;
            if (!pr.deviated) break;
            if (drain) drain->valid = false;  // a replanning pass rewrites anything
        }
        sp.finish();
        inf.plan_ms = plan_ms;
    } catch (const std::domain_error& e) {
        return set_error(TEIG_ERR_STRICT, e.what());
    } catch (const std::exception& e) {
        return set_error(TEIG_ERR_CUDA, e.what());
    }
    // clean: no rejection and every still-selected block leads
    bool leading = true;
    {
        bool seen_unsel = false;
        for (const auto& b : blocks) {
            if (!b.selected) seen_unsel = true;
            else if (seen_unsel) leading = false;
        }
    }
    // ascending original index: the reference's order of discovery (it runs
    // the groups top-down and a window's stuck blocks in slice order, so its
    // rejected_blocks come out sorted; pipelined groups here fold out of it)
    std::sort(rejected.begin(), rejected.end());
    inf.n_rejected = (int64_t)rejected.size();
    inf.clean = (rejected.empty() && leading) ? 1 : 0;
    if (perm)
        for (int64_t i = 0; i < nb; ++i) perm[blocks[i].orig] = i;
    if (rejected_out)
        for (size_t i = 0; i < rejected.size(); ++i) rejected_out[i] = rejected[i];
    if (plan_out)
        for (int64_t i = 0; i < (int64_t)plan_log.size() / 3 && i < plan_cap; ++i)
            for (int k = 0; k < 3; ++k) plan_out[3 * i + k] = plan_log[3 * i + k];
    if (info) *info = inf;
    return 0;
}

}  // namespace teig

// ============================================================================
// C ABI
// ============================================================================
using namespace teig;

extern "C" {

const char* teig_last_error(void) { return g_last_error.c_str(); }
int teig_version(void) { return 1; }

void teig_reorder_opts_default(teig_reorder_opts* o) {
    o->window_size = 0;
    o->strict = 0;
    o->overlap_factor = 1;
    o->profile = 0;
    o->full_factor = 0;
}

int teig_reorder_schur_device(int64_t n, double* dS, int64_t lds, double* dQ, int64_t ldq, int64_t nb,
                              const uint8_t* sizes, const uint8_t* flags, const teig_reorder_opts* opts,
                              int64_t* perm, int64_t* rejected, int64_t* plan, int64_t plan_cap,
                              teig_reorder_info* info, void* stream) {
    DeviceGuard device_guard(dS);
    return reorder_schur_device(n, dS, lds, dQ, ldq, nb, sizes, flags, opts, perm, rejected, plan, plan_cap, info,
                                (cudaStream_t)stream);
}

void teig_release_host_staging(void) {
    std::lock_guard<std::mutex> lk(g_staging_mu);
    for (auto& kv : g_staging) {
        std::lock_guard<std::mutex> g(kv.second->mu);
        kv.second->release();
    }
}

void teig_trace_enable(int32_t on) { g_trace.on = on != 0; }

int64_t teig_trace_task_count(void) { return (int64_t)g_trace.tasks.size(); }

int teig_trace_task(int64_t i, char* label, int64_t cap, int32_t* worker, int64_t* start_ns, int64_t* end_ns) {
    if (i < 0 || i >= (int64_t)g_trace.tasks.size()) return set_error(-1, "trace task index out of range");
    const TraceTask& t = g_trace.tasks[i];
    if (label && cap > 0) {
        const size_t k = std::min<size_t>(t.label.size(), (size_t)cap - 1);
        std::memcpy(label, t.label.data(), k);
        label[k] = 0;
    }
    if (worker) *worker = t.worker;
    if (start_ns) *start_ns = t.start_ns;
    if (end_ns) *end_ns = t.end_ns;
    return 0;
}

int64_t teig_trace_json(char* buf, int64_t cap) {
    std::string j = "{\"tasks\": [";
    for (size_t i = 0; i < g_trace.tasks.size(); ++i) {
        const auto& t = g_trace.tasks[i];
        j += (i ? ", " : "") + std::string("{\"label\": \"") + t.label + "\", \"worker\": " + std::to_string(t.worker) +
             ", \"start_ns\": " + std::to_string(t.start_ns) + ", \"end_ns\": " + std::to_string(t.end_ns) + "}";
    }
    j += "], \"stalls\": [], \"windows\": [";
    for (size_t i = 0; i < g_trace.wins.size(); ++i) {
        const auto& w = g_trace.wins[i];
        j += (i ? ", " : "") + std::string("{\"pass\": ") + std::to_string(w.pass) + ", \"level\": " +
             std::to_string(w.level) + ", \"position\": " + std::to_string(w.a) + ", \"extent\": " +
             std::to_string(w.d) + ", \"blocks\": " + std::to_string(w.nb) + ", \"group\": " +
             std::to_string(w.group) + ", \"status\": \"" +
             ((w.status & kWinSkipped) ? "skipped"
                                       : (w.status & kWinExecuted) ? ((w.status & kWinStuck) ? "stuck" : "executed")
                                                                   : "layout-mismatch") +
             "\"}";
    }
    j += "]}";
    if (buf && cap > (int64_t)j.size()) std::memcpy(buf, j.c_str(), j.size() + 1);
    return (int64_t)j.size();
}

void teig_set_memory_retention(int32_t on) {
    set_memory_retention(on != 0);
    if (!on) teig_release_host_staging();
}

int32_t teig_memory_retention(void) { return memory_retention() ? 1 : 0; }

void teig_release_memory(void) {
    teig_release_host_staging();
    trim_memory_pools();
}

// columns per host<->device copy of S's upper Hessenberg part (each copy
// carries a rectangle: ~kHessCopyCols^2 / 2 extra doubles per block)
constexpr int64_t kHessCopyCols = 512;

thread_local int64_t g_host_h2d = 0, g_host_d2h = 0;  // teig_host_transfer_bytes

void teig_host_transfer_bytes(int64_t* h2d, int64_t* d2h) {
    if (h2d) *h2d = g_host_h2d;
    if (d2h) *d2h = g_host_d2h;
}

int teig_reorder_schur_host(int64_t n, double* S, int64_t lds, double* Q, int64_t ldq, int64_t nb,
                            const uint8_t* sizes, const uint8_t* flags, const teig_reorder_opts* opts,
                            int64_t* perm, int64_t* rejected, int64_t* plan, int64_t plan_cap,
                            teig_reorder_info* info, void* stream_v) {
    if (n < 1) return set_error(-1, "n must be >= 1");
    if (!S) return set_error(-2, "S is null");
    if (lds < n) return set_error(-3, "lds < n");
    if (Q && ldq < n) return set_error(-5, "ldq < n");
    cudaStream_t stream = (cudaStream_t)stream_v;
    cudaStream_t qs = nullptr;
    cudaEvent_t q_ready = nullptr;
    const bool hprof = getenv("TEIG_HOST_PROF") && atoi(getenv("TEIG_HOST_PROF"));
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    const auto h0 = now();
    const bool no_cache = !memory_retention();
    HostStaging& hs = host_staging();
    std::unique_lock<std::mutex> lock(hs.mu, std::defer_lock);
    try {
        const size_t pitch = (size_t)n * sizeof(double);
        const size_t need = pitch * n * (Q ? 2 : 1);
        int64_t h2d = 0;
        g_host_h2d = g_host_d2h = 0;
        struct Plain {  // per-call staging (cudaFree synchronizes)
            void* p = nullptr;
            ~Plain() {
                if (p) cudaFree(p);
            }
        } tmp;
        double* base = nullptr;
        if (no_cache) {
            TEIG_CUDA(cudaMalloc(&tmp.p, need));
            base = static_cast<double*>(tmp.p);
        } else {
            lock.lock();
            if (hs.bytes < need) {
                if (hs.p) TEIG_CUDA(cudaFree(hs.p));
                hs.p = nullptr;
                hs.bytes = 0;
                TEIG_CUDA(cudaMalloc(&hs.p, need));
                hs.bytes = need;
            }
            base = static_cast<double*>(hs.p);
        }
        double* const dS = base;
        double* const dQ = Q ? base + (size_t)n * n : nullptr;
        TEIG_CUDA(cudaStreamSynchronize(stream));  // staging visible to the side stream
        const auto h1 = now();
        // the factor's row support (plan.h FactorSupport), scanned on the host
        // cores while S travels to the device (hidden behind the upload)
        FactorSupport qsupp;
        std::vector<std::thread> scan;
        const bool no_supp = getenv("TEIG_NO_Q_SUPPORT") && atoi(getenv("TEIG_NO_Q_SUPPORT"));
        if (Q && !no_supp && !(opts && opts->full_factor)) {
            qsupp.lo.resize(n);
            qsupp.hi.resize(n);
            const int nt = (int)std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
            for (int t = 0; t < nt; ++t)
                scan.emplace_back([&qsupp, Q, ldq, n, nt, t] {  // nt by value: it leaves scope before the join
                    for (int64_t c = n * t / nt; c < n * (t + 1) / nt; ++c) {
                        // first / last nonzero bit pattern: 8-word OR blocks (vectorised), then the word
                        const uint64_t* col = reinterpret_cast<const uint64_t*>(Q + c * ldq);
                        int64_t l = 0, h = n - 1;
                        for (; l + 8 <= n; l += 8) {
                            uint64_t o = 0;
                            for (int k = 0; k < 8; ++k) o |= col[l + k];
                            if (o) break;
                        }
                        while (l < n && col[l] == 0) ++l;
                        for (; h - 7 > l; h -= 8) {
                            uint64_t o = 0;
                            for (int k = 0; k < 8; ++k) o |= col[h - k];
                            if (o) break;
                        }
                        while (h > l && col[h] == 0) --h;
                        qsupp.lo[c] = (int32_t)l;
                        qsupp.hi[c] = l < n ? (int32_t)h : -1;
                    }
                });
        }
        struct Join {
            std::vector<std::thread>& v;
            ~Join() {
                for (auto& t : v)
                    if (t.joinable()) t.join();
            }
        } join_scan{scan};
        // S travels as its upper Hessenberg part only (column j: rows 0..j+1,
        // in blocks of 512 columns): nothing on the path reads or writes below
        // the first subdiagonal -- neither does the reference (windows and
        // panels lie on and above it) -- so the strictly lower part keeps its
        // input values, which is also what comes back (half the bytes each
        // way).  The device copy's lower part is zeroed first.
        TEIG_CUDA(cudaMemsetAsync(dS, 0, pitch * n, stream));
        for (int64_t j0 = 0; j0 < n; j0 += kHessCopyCols) {
            const int64_t j1 = std::min<int64_t>(n, j0 + kHessCopyCols), rows = std::min<int64_t>(n, j1 + 1);
            TEIG_CUDA(cudaMemcpy2DAsync(dS + j0 * n, pitch, S + j0 * lds, lds * sizeof(double),
                                        (size_t)rows * sizeof(double), (size_t)(j1 - j0), cudaMemcpyHostToDevice,
                                        stream));
            h2d += rows * (j1 - j0) * (int64_t)sizeof(double);
        }
        // S on the device before the levels are enqueued: measured, letting the
        // host enqueue thousands of launches while the 12.8 GB upload runs made
        // the device phase 0.3-4.5 s slower and erratic at n=40000
        TEIG_CUDA(cudaStreamSynchronize(stream));
        for (auto& t : scan) t.join();
        qsupp.on = !scan.empty();
        if (Q) {  // Q travels on a side stream while the S-side work starts (measured:
                  // uploading Q before the work starts costs +0.5 s at n=40000)
            qs = cached_stream(0);
            if (!qs) throw std::runtime_error("stream creation failed");
            TEIG_CUDA(cudaEventCreateWithFlags(&q_ready, cudaEventDisableTiming));
            if (qsupp.on) {
                // only the row hull of each block of columns (the scan's
                // support; exact zeros elsewhere, +0.0 bit patterns): Q_in = I
                // is 0.17 GB instead of 12.8 GB at n=40000
                TEIG_CUDA(cudaMemsetAsync(dQ, 0, pitch * n, qs));
                for (int64_t j0 = 0; j0 < n; j0 += kHessCopyCols) {
                    const int64_t j1 = std::min<int64_t>(n, j0 + kHessCopyCols);
                    int64_t lo = n, hi = -1;
                    for (int64_t c = j0; c < j1; ++c) {
                        lo = std::min<int64_t>(lo, qsupp.lo[c]);
                        hi = std::max<int64_t>(hi, qsupp.hi[c]);
                    }
                    if (hi < lo) continue;
                    TEIG_CUDA(cudaMemcpy2DAsync(dQ + j0 * n + lo, pitch, Q + j0 * ldq + lo, ldq * sizeof(double),
                                                (size_t)(hi - lo + 1) * sizeof(double), (size_t)(j1 - j0),
                                                cudaMemcpyHostToDevice, qs));
                    h2d += (hi - lo + 1) * (j1 - j0) * (int64_t)sizeof(double);
                }
            } else {
                TEIG_CUDA(cudaMemcpy2DAsync(dQ, pitch, Q, ldq * sizeof(double), pitch, n, cudaMemcpyHostToDevice, qs));
                h2d += n * n * (int64_t)sizeof(double);
            }
            TEIG_CUDA(cudaEventRecord(q_ready, qs));
        }
        const auto h2 = now();
        // the final parts of S and Q stream back while the last levels run
        // (TEIG_NO_DRAIN=1: everything after the end)
        HostDrain dr;
        dr.hS = S;
        dr.lds = lds;
        dr.hQ = Q;
        dr.ldq = ldq;
        dr.s_hi = n;
        dr.q_lo = 0;
        dr.q_hi = n;
        // early copies only into page-locked buffers (a copy to pageable memory
        // would block the thread that enqueues the remaining levels)
        auto pinned = [](const void* p) {
            if (!p) return true;
            cudaPointerAttributes at{};
            if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
                cudaGetLastError();
                return false;
            }
            return at.type == cudaMemoryTypeHost;
        };
        const bool drain_on = !(getenv("TEIG_NO_DRAIN") && atoi(getenv("TEIG_NO_DRAIN"))) && pinned(S) && pinned(Q);
        struct DrainRes {
            HostDrain& d;
            ~DrainRes() {
                if (d.ds) cudaStreamSynchronize(d.ds);  // (cached: not destroyed)
                if (d.evS) cudaEventDestroy(d.evS);
                if (d.evQ) cudaEventDestroy(d.evQ);
            }
        } drain_res{dr};
        dr.ds = cached_stream(1);
        if (!dr.ds) throw std::runtime_error("stream creation failed");
        TEIG_CUDA(cudaEventCreateWithFlags(&dr.evS, cudaEventDisableTiming));
        TEIG_CUDA(cudaEventCreateWithFlags(&dr.evQ, cudaEventDisableTiming));
        const int rc = reorder_schur_device(n, dS, n, dQ, n, nb, sizes, flags, opts, perm, rejected, plan, plan_cap,
                                            info, stream, q_ready, drain_on ? &dr : nullptr, &qsupp);
        TEIG_CUDA(cudaStreamSynchronize(stream));
        if (qs) TEIG_CUDA(cudaStreamSynchronize(qs));
        const auto h3 = now();
        if (rc != 0) {
            if (qs) cudaStreamSynchronize(qs);
            if (q_ready) cudaEventDestroy(q_ready);
            return rc;
        }
        if (!dr.valid) {  // replanned: move everything
            dr.s_hi = n;
            dr.q_lo = 0;
            dr.q_hi = n;
        }
        TEIG_CUDA(cudaEventRecord(dr.evS, stream));  // all device work (the Q stream joined `stream`)
        TEIG_CUDA(cudaStreamWaitEvent(dr.ds, dr.evS, 0));
        if (dr.s_hi > 0) {  // rows [0, s_hi): columns < s_hi down to their subdiagonal, the rest whole
            for (int64_t j0 = 0; j0 < std::min<int64_t>(dr.s_hi, n); j0 += kHessCopyCols) {
                const int64_t j1 = std::min<int64_t>(dr.s_hi, j0 + kHessCopyCols);
                const int64_t rows = std::min<int64_t>(dr.s_hi, j1 + 1);
                TEIG_CUDA(cudaMemcpy2DAsync(S + j0 * lds, lds * sizeof(double), dS + j0 * n, pitch,
                                            (size_t)rows * sizeof(double), (size_t)(j1 - j0), cudaMemcpyDeviceToHost,
                                            dr.ds));
                dr.d2h_bytes += rows * (j1 - j0) * (int64_t)sizeof(double);
            }
            if (dr.s_hi < n) {
                TEIG_CUDA(cudaMemcpy2DAsync(S + dr.s_hi * lds, lds * sizeof(double), dS + dr.s_hi * n, pitch,
                                            (size_t)dr.s_hi * sizeof(double), (size_t)(n - dr.s_hi),
                                            cudaMemcpyDeviceToHost, dr.ds));
                dr.d2h_bytes += dr.s_hi * (n - dr.s_hi) * (int64_t)sizeof(double);
            }
        }
        if (Q && dr.q_hi > dr.q_lo) {
            TEIG_CUDA(cudaMemcpy2DAsync(Q + dr.q_lo * ldq, ldq * sizeof(double), dQ + dr.q_lo * (size_t)n, pitch,
                                        pitch, (size_t)(dr.q_hi - dr.q_lo), cudaMemcpyDeviceToHost, dr.ds));
            dr.d2h_bytes += n * (dr.q_hi - dr.q_lo) * (int64_t)sizeof(double);
        }
        TEIG_CUDA(cudaStreamSynchronize(dr.ds));
        if (qs) TEIG_CUDA(cudaStreamSynchronize(qs));
        g_host_h2d = h2d;
        g_host_d2h = dr.d2h_bytes;
        if (hprof)
            fprintf(stderr, "[teig host] alloc %.1f ms  h2d(S) %.1f ms  device %.1f ms  d2h %.1f ms\n", ms(h0, h1),
                    ms(h1, h2), ms(h2, h3), ms(h3, now()));
    } catch (const std::exception& e) {
        if (qs) cudaStreamSynchronize(qs);
        if (q_ready) cudaEventDestroy(q_ready);
        return set_error(TEIG_ERR_CUDA, e.what());
    }
    if (q_ready) cudaEventDestroy(q_ready);
    return 0;
}

int64_t teig_scan_blocks_device(int64_t n, const double* dS, int64_t lds, uint8_t* sizes, void* stream_v) {
    DeviceGuard device_guard(dS);
    if (n < 1) return set_error(-1, "n must be >= 1");
    cudaStream_t stream = (cudaStream_t)stream_v;
    std::vector<double> sub(n > 1 ? n - 1 : 1, 0.0);
    try {
        if (n > 1) {
            TEIG_CUDA(cudaMemcpy2DAsync(sub.data(), sizeof(double), dS + 1, (lds + 1) * sizeof(double), sizeof(double),
                                        n - 1, cudaMemcpyDeviceToHost, stream));
            TEIG_CUDA(cudaStreamSynchronize(stream));
        }
    } catch (const std::exception& e) {
        return set_error(TEIG_ERR_CUDA, e.what());
    }
    int64_t nb = 0;
    for (int64_t i = 0; i < n;) {
        if (i + 1 < n && sub[i] != 0.0) {
            sizes[nb++] = 2;
            i += 2;
        } else {
            sizes[nb++] = 1;
            i += 1;
        }
    }
    return nb;
}

int64_t teig_plan_reorder(int64_t n, int64_t nb, const uint8_t* sizes, const uint8_t* flags, int64_t window_size,
                          int64_t* win, int64_t cap, int64_t* n_levels, int64_t* n_groups, double* flops) {
    if (n < 1) return set_error(-1, "n must be >= 1");
    std::vector<BlockState> blocks(nb);
    int64_t rows = 0;
    for (int64_t i = 0; i < nb; ++i) {
        if (sizes[i] != 1 && sizes[i] != 2) return set_error(-3, "block sizes must be 1 or 2");
        blocks[i] = BlockState{sizes[i], (uint8_t)(flags[i] ? 1 : 0), (uint32_t)i};
        rows += sizes[i];
    }
    if (rows != n) return set_error(-3, "selection does not match n");
    const int64_t ws = std::min<int64_t>(std::max<int64_t>(window_size ? window_size : default_tile_size(n), 8), 128);
    ReorderPlan plan = plan_reorder(blocks, ws);
    schedule_levels(plan, n);
    if (win)
        for (int64_t i = 0; i < (int64_t)plan.windows.size() && i < cap; ++i) {
            const auto& w = plan.windows[i];
            win[5 * i] = w.wtop;
            win[5 * i + 1] = w.wbot;
            win[5 * i + 2] = w.count;
            win[5 * i + 3] = w.group;
            win[5 * i + 4] = w.level;
        }
    if (n_levels) *n_levels = plan.n_levels;
    if (n_groups) *n_groups = plan.n_groups;
    if (flops) *flops = plan_update_flops(plan, n, true);
    return (int64_t)plan.windows.size();
}

int teig_select_fraction(int64_t nb, double fraction, uint64_t seed, uint8_t* flags) {
    if (fraction < 0.0 || fraction > 1.0) return set_error(-2, "selection fraction must be in [0, 1]");
    // Philox4x32-10 stream (philox.hpp), Fisher-Yates over block indices
    struct Stream {
        uint32_t k0, k1;
        uint64_t ctr = 0;
        uint32_t buf[4];
        int have = 0;
        uint64_t next() {
            if (!have) {
                uint32_t c[4] = {(uint32_t)ctr, (uint32_t)(ctr >> 32), 0u, 0u};
                uint32_t a = k0, b = k1;
                for (int r = 0; r < 10; ++r) {
                    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
                    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ a, n1 = (uint32_t)p1;
                    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ b, n3 = (uint32_t)p0;
                    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
                    a += 0x9E3779B9u;
                    b += 0xBB67AE85u;
                }
                std::memcpy(buf, c, sizeof c);
                ++ctr;
                have = 2;
            }
            const int i = 2 - have;
            --have;
            return ((uint64_t)buf[2 * i + 1] << 32) | buf[2 * i];
        }
    };
    const uint64_t s = seed ^ 0x5e1ec7u;
    Stream rng{(uint32_t)s, (uint32_t)(s >> 32)};
    const int64_t want = (int64_t)(fraction * (double)nb);
    std::vector<int64_t> idx(nb);
    for (int64_t i = 0; i < nb; ++i) idx[i] = i;
    for (int64_t i = 0; i < want && i + 1 < nb; ++i) {
        const int64_t j = i + (int64_t)(rng.next() % (uint64_t)(nb - i));
        std::swap(idx[i], idx[j]);
    }
    std::memset(flags, 0, (size_t)nb);
    for (int64_t i = 0; i < want; ++i) flags[idx[i]] = 1;
    return 0;
}

int teig_window_reorder_device(int64_t d, double* dW, int64_t ldw, int64_t nb, const uint8_t* sizes,
                               const uint8_t* sel, double* dAcc, uint32_t* order, uint8_t* stuck,
                               int32_t* executed, void* stream_v) {
    DeviceGuard device_guard(dW);
    if (d < 1 || d > 128) return set_error(d < 1 ? -1 : TEIG_ERR_UNSUPPORTED, "window order must be in [1, 128]");
    if (ldw < d) return set_error(-3, "ldw < d");
    if (nb < 1 || nb > d) return set_error(-4, "bad block count");
    cudaStream_t stream = (cudaStream_t)stream_v;
    try {
        WinDesc wd{};
        wd.a = 0;
        wd.d = (int32_t)d;
        wd.nb = (int32_t)nb;
        wd.qw_off = 0;
        wd.blk_off = 0;
        DevBuf ddesc(sizeof(WinDesc), stream), dsz(nb, stream), dsel(nb, stream), dord(nb, stream), dstk(nb, stream),
            dst(sizeof(int32_t), stream);
        TEIG_CUDA(cudaMemcpyAsync(ddesc.p, &wd, sizeof wd, cudaMemcpyHostToDevice, stream));
        TEIG_CUDA(cudaMemcpyAsync(dsz.p, sizes, nb, cudaMemcpyHostToDevice, stream));
        TEIG_CUDA(cudaMemcpyAsync(dsel.p, sel, nb, cudaMemcpyHostToDevice, stream));
        TEIG_CUDA(launch_window_reorder(ddesc.as<WinDesc>(), 1, d <= 64 ? 64 : 128, dW, ldw, dAcc, dsz.as<uint8_t>(),
                                        dsel.as<uint8_t>(), dord.as<uint8_t>(), dstk.as<uint8_t>(), dst.as<int32_t>(),
                                        stream));
        std::vector<uint8_t> o(nb), s(nb);
        int32_t st = 0;
        TEIG_CUDA(cudaMemcpyAsync(o.data(), dord.p, nb, cudaMemcpyDeviceToHost, stream));
        TEIG_CUDA(cudaMemcpyAsync(s.data(), dstk.p, nb, cudaMemcpyDeviceToHost, stream));
        TEIG_CUDA(cudaMemcpyAsync(&st, dst.p, sizeof st, cudaMemcpyDeviceToHost, stream));
        TEIG_CUDA(cudaStreamSynchronize(stream));
        *executed = (st & kWinExecuted) ? 1 : 0;
        for (int64_t i = 0; i < nb; ++i) {
            if (order) order[i] = *executed ? o[i] : (uint32_t)i;
            if (stuck) stuck[i] = *executed ? s[i] : 0;
        }
    } catch (const std::exception& e) {
        return set_error(TEIG_ERR_CUDA, e.what());
    }
    return 0;
}

int teig_apply_window_updates_device(int64_t n, double* dS, int64_t lds, double* dQ, int64_t ldq, int64_t a,
                                     int64_t d, const double* dQw, void* stream_v) {
    DeviceGuard device_guard(dS);
    if (n < 1) return set_error(-1, "n must be >= 1");
    if (lds < n) return set_error(-3, "lds < n");
    if (dQ && ldq < n) return set_error(-5, "ldq < n");
    if (a < 0 || d < 1 || a + d > n) return set_error(-6, "window out of range");
    if (d > 128) return set_error(TEIG_ERR_UNSUPPORTED, "window order must be <= 128");
    cudaStream_t stream = (cudaStream_t)stream_v;
    try {
        WinDesc wd{};
        wd.a = (int32_t)a;
        wd.d = (int32_t)d;
        wd.nb = 0;
        wd.qw_off = 0;
        wd.lc0 = (int32_t)(a + d);
        wd.lc1 = (int32_t)n;
        wd.rr0 = 0;
        wd.rr1 = (int32_t)a;
        wd.qr0 = 0;
        wd.qr1 = (int32_t)n;
        DevBuf ddesc(sizeof(WinDesc), stream);
        TEIG_CUDA(cudaMemcpyAsync(ddesc.p, &wd, sizeof wd, cudaMemcpyHostToDevice, stream));
        const int dm = d <= 64 ? 64 : 128;
        const int tl = (int)((n - a - d + kLeftBN - 1) / kLeftBN);
        const int tr = (int)((a + kRightBM - 1) / kRightBM);
        const int tq = (int)((n + kRightBM - 1) / kRightBM);
        TEIG_CUDA(launch_update_left(ddesc.as<WinDesc>(), 1, tl, dm, dQw, dS, lds, (int)n, stream, n, n));
        TEIG_CUDA(launch_update_right(ddesc.as<WinDesc>(), 1, tr, dm, dQw, dS, lds, (int)n, false, stream, n, n));
        if (dQ)
            TEIG_CUDA(launch_update_right(ddesc.as<WinDesc>(), 1, tq, dm, dQw, dQ, ldq, (int)n, true, stream, n, n));
        TEIG_CUDA(cudaStreamSynchronize(stream));
    } catch (const std::exception& e) {
        return set_error(TEIG_ERR_CUDA, e.what());
    }
    return 0;
}

int teig_update_panel_device(int32_t side, int64_t d, const double* dQw, int64_t a, double* dM, int64_t ldm,
                             int64_t rows, int64_t cols, int64_t i0, int64_t i1, void* stream_v) {
    DeviceGuard device_guard(dM);
    if (side < 0 || side > 2) return set_error(-1, "side must be 0 (left), 1 (right) or 2 (factor)");
    if (d < 1 || d > 128) return set_error(d < 1 ? -2 : TEIG_ERR_UNSUPPORTED, "window order must be in [1, 128]");
    if (!dQw || !dM) return set_error(-3, "null pointer");
    if (ldm < rows || rows < 1 || cols < 1) return set_error(-6, "bad extent");
    if (a < 0 || i0 < 0 || i1 < i0) return set_error(-5, "bad range");
    if (side == 0 ? (a + d > rows || i1 > cols) : (a + d > cols || i1 > rows)) return set_error(-5, "range outside M");
    if (i1 == i0) return 0;
    cudaStream_t stream = (cudaStream_t)stream_v;
    try {
        WinDesc wd{};
        wd.a = (int32_t)a;
        wd.d = (int32_t)d;
        wd.lc0 = (int32_t)i0;
        wd.lc1 = (int32_t)i1;
        wd.rr0 = wd.qr0 = (int32_t)i0;
        wd.rr1 = wd.qr1 = (int32_t)i1;
        DevBuf ddesc(sizeof(WinDesc), stream);
        TEIG_CUDA(cudaMemcpyAsync(ddesc.p, &wd, sizeof wd, cudaMemcpyHostToDevice, stream));
        const int dm = d <= 64 ? 64 : 128;
        if (side == 0) {
            const int tiles = (int)((i1 - i0 + kLeftBN - 1) / kLeftBN);
            TEIG_CUDA(launch_update_left(ddesc.as<WinDesc>(), 1, tiles, dm, dQw, dM, ldm, (int)rows, stream, rows, cols));
        } else {
            const int tiles = (int)((i1 - i0 + kRightBM - 1) / kRightBM);
            TEIG_CUDA(launch_update_right(ddesc.as<WinDesc>(), 1, tiles, dm, dQw, dM, ldm, (int)rows, side == 2, stream,
                                          rows, cols));
        }
        TEIG_CUDA(cudaStreamSynchronize(stream));
    } catch (const std::exception& e) {
        return set_error(TEIG_ERR_CUDA, e.what());
    }
    return 0;
}

int teig_gen_schur_input_device(int64_t n, double* dS, int64_t lds, uint64_t fill_seed, void* stream) {
    DeviceGuard device_guard(dS);
    if (n < 1 || lds < n) return set_error(-1, "bad shape");
    cudaError_t e = launch_gen_schur_input(dS, lds, n, fill_seed, (cudaStream_t)stream);
    return e == cudaSuccess ? 0 : set_error(TEIG_ERR_CUDA, cudaGetErrorString(e));
}

int teig_gen_hessenberg_device(int64_t n, double* dH, int64_t ldh, uint64_t seed, void* stream) {
    DeviceGuard device_guard(dH);
    if (n < 1 || ldh < n) return set_error(-1, "bad shape");
    cudaError_t e = launch_gen_hessenberg(dH, ldh, n, seed, (cudaStream_t)stream);
    return e == cudaSuccess ? 0 : set_error(TEIG_ERR_CUDA, cudaGetErrorString(e));
}

int teig_set_identity_device(int64_t n, double* dQ, int64_t ldq, void* stream) {
    DeviceGuard device_guard(dQ);
    if (n < 1 || ldq < n) return set_error(-1, "bad shape");
    cudaError_t e = launch_set_identity(dQ, ldq, n, (cudaStream_t)stream);
    return e == cudaSuccess ? 0 : set_error(TEIG_ERR_CUDA, cudaGetErrorString(e));
}

}  // extern "C"
