// greorder_driver.cpp -- generalized Schur-pair reordering (S, T) with Q and
// Z on one B200, exported through the C
// ABI in include/taskeig_b200.h.
//
// The reference has no generalized path ("parity unpinned by
// the reference"); the semantics are those of the standard driver
// (reorder.cpp:215-404: the same planner, wavefront levels, one readback per
// pass, fold in plan order, replan on deviation) with LAPACK DTGEX2/DTGSEN's
// pair swap, and the pencil updated from both sides:
//   left  (row panels):    [S; T][a:b, b:n]  <- Q_w^T [S; T][a:b, b:n]
//   right (column panels): [S; T][0:a, a:b]  <- [S; T][0:a, a:b] Z_w
//   factors:               Q[:, a:b] <- Q[:, a:b] Q_w,  Z[:, a:b] <- Z[:, a:b] Z_w
// with the same DMMA update kernels as the standard path (two accumulators per
// window: Q_w at qw_off, Z_w right behind it).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/taskeig_b200.h"
#include "device_types.h"
#include "launch.h"
#include "plan.h"
#include "qw_ring.h"

namespace teig {

int set_error(int code, const std::string& msg);
int64_t default_tile_size(int64_t n);

namespace {

#define TEIG_CUDA(expr)                                                                          \
    do {                                                                                         \
        cudaError_t _e = (expr);                                                                 \
        if (_e != cudaSuccess)                                                                   \
            throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(_e) + " at " + \
                                     __FILE__ + ":" + std::to_string(__LINE__));                 \
    } while (0)

template <typename T>
struct DBuf {
    T* p = nullptr;
    cudaStream_t s;
    DBuf(size_t n, cudaStream_t st) : s(st) {
        if (n) TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&p), n * sizeof(T), st));
    }
    ~DBuf() {
        if (p) cudaFreeAsync(p, s);
    }
};

struct GPass {
    int64_t windows = 0, levels = 0, launches = 0;
    bool deviated = false;
};

GPass run_gpass(ReorderPlan& plan, int64_t n, double* dS, int64_t lds, double* dT, int64_t ldt, double* dQ,
                int64_t ldq, double* dZ, int64_t ldz, std::vector<BlockState>& blocks, std::vector<int64_t>& rejected,
                std::vector<int64_t>& plan_log, bool strict, cudaStream_t s, cudaStream_t s2, cudaEvent_t ev,
                FactorSupport& qsupp, FactorSupport& zsupp, double* flops_exec) {
    GPass gp;
    const int64_t nw = (int64_t)plan.windows.size();
    schedule_levels(plan, n);
    const int nl = plan.n_levels;
    std::vector<int64_t> idx(nw);
    for (int64_t i = 0; i < nw; ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(),
                     [&](int64_t x, int64_t y) { return plan.windows[x].level < plan.windows[y].level; });
    std::vector<WinDesc> dq(nw), dz(nw);
    std::vector<int64_t> lvl_off(nl + 1, 0), tl(nl, 0), tr(nl, 0), tq(nl, 0), tz(nl, 0);
    int dmax = 0;
    int64_t pool = 0;
    for (int64_t k = 0; k < nw; ++k) {
        const PlannedWindow& w = plan.windows[idx[k]];
        const int L = w.level;
        WinDesc& d = dq[k];
        std::memset(&d, 0, sizeof d);
        d.a = (int32_t)w.wtop;
        d.d = (int32_t)(w.wbot - w.wtop);
        d.nb = (int32_t)w.count;
        d.level = L;
        d.qw_off = pool;
        pool += 2 * (int64_t)d.d * d.d;
        d.blk_off = w.blk_off;
        d.tl_pref = (int32_t)tl[L];
        d.tr_pref = (int32_t)tr[L];
        d.tq_pref = (int32_t)tq[L];
        d.lc0 = (int32_t)w.wbot;
        d.lc1 = (int32_t)n;
        d.rr0 = 0;
        d.rr1 = (int32_t)w.wtop;
        // factor rows: the tracked supports of Q's and Z's columns (plan.h)
        int64_t q0 = 0, q1 = n, z0 = 0, z1 = n;
        if (dQ && qsupp.on) qsupp.window(w.wtop, w.wbot, &q0, &q1);
        if (dZ && zsupp.on) zsupp.window(w.wtop, w.wbot, &z0, &z1);
        const double dd2 = 2.0 * double(d.d) * double(d.d);
        *flops_exec += (dQ ? dd2 * double(q1 - q0) : 0.0) + (dZ ? dd2 * double(z1 - z0) : 0.0);
        d.qr0 = (int32_t)q0;
        d.qr1 = (int32_t)q1;
        tl[L] += (n - w.wbot + kLeftBN - 1) / kLeftBN;
        tr[L] += (w.wtop + kRightBM - 1) / kRightBM;
        tq[L] += (q1 - q0 + kRightBM - 1) / kRightBM;
        lvl_off[L + 1]++;
        dmax = std::max(dmax, d.d);
        dz[k] = d;
        dz[k].qw_off = d.qw_off + (int64_t)d.d * d.d;  // Z_w behind Q_w
        dz[k].qr0 = (int32_t)z0;
        dz[k].qr1 = (int32_t)z1;
        dz[k].tq_pref = (int32_t)tz[L];
        tz[L] += (z1 - z0 + kRightBM - 1) / kRightBM;
    }
    for (int L = 0; L < nl; ++L) lvl_off[L + 1] += lvl_off[L];
    const int dm = dmax <= 64 ? 64 : 128;
    // accumulators in a per-level ring (qw_ring.h): Q_w at qw_off, Z_w behind it
    const QwRing ring = make_qw_ring(dq, lvl_off, nl, 2);
    pool = ring.total;
    for (int64_t k = 0; k < nw; ++k) dz[k].qw_off = dq[k].qw_off + (int64_t)dq[k].d * dq[k].d;
    RingEvents ring_ev(ring.k > 0 && (dQ || dZ) ? ring.k : 0);
    const size_t ne = plan.sizes.size();
    DBuf<WinDesc> d_q(nw, s), d_z(nw, s);
    DBuf<double> d_pool(std::max<int64_t>(pool, 1), s);
    DBuf<uint8_t> d_sizes(ne + 1, s), d_sel(ne + 1, s), d_order(ne + 1, s), d_stuck(ne + 1, s);
    DBuf<int32_t> d_status(std::max<int64_t>(nw, 1), s), d_devlvl(1, s);
    TEIG_CUDA(cudaMemsetAsync(d_devlvl.p, 0x7f, sizeof(int32_t), s));
    TEIG_CUDA(cudaMemcpyAsync(d_q.p, dq.data(), sizeof(WinDesc) * nw, cudaMemcpyHostToDevice, s));
    TEIG_CUDA(cudaMemcpyAsync(d_z.p, dz.data(), sizeof(WinDesc) * nw, cudaMemcpyHostToDevice, s));
    TEIG_CUDA(cudaMemcpyAsync(d_sizes.p, plan.sizes.data(), ne, cudaMemcpyHostToDevice, s));
    TEIG_CUDA(cudaMemcpyAsync(d_sel.p, plan.sel.data(), ne, cudaMemcpyHostToDevice, s));
    int64_t launches = 0;
    for (int L = 0; L < nl; ++L) {
        const int64_t o = lvl_off[L], cnt = lvl_off[L + 1] - lvl_off[L];
        if (!cnt) continue;
        if (ring_ev.n && L >= ring.k) TEIG_CUDA(cudaStreamWaitEvent(s, ring_ev.ev[L % ring.k], 0));
        TEIG_CUDA(launch_gwindow_reorder(d_q.p + o, (int)cnt, dmax, dS, lds, dT, ldt, d_pool.p, d_sizes.p, d_sel.p,
                                         d_order.p, d_stuck.p, d_status.p + o, s, d_devlvl.p));
        ++launches;
        if (dQ || dZ) {  // factor updates on the second stream
            TEIG_CUDA(cudaEventRecord(ev, s));
            TEIG_CUDA(cudaStreamWaitEvent(s2, ev, 0));
            if (dQ) {
                TEIG_CUDA(launch_update_right(d_q.p + o, (int)cnt, (int)tq[L], dm, d_pool.p, dQ, ldq, (int)n, true, s2, n, n));
                ++launches;
            }
            if (dZ) {
                TEIG_CUDA(launch_update_right(d_z.p + o, (int)cnt, (int)tz[L], dm, d_pool.p, dZ, ldz, (int)n, true, s2, n, n));
                ++launches;
            }
            if (ring_ev.n) TEIG_CUDA(cudaEventRecord(ring_ev.ev[L % ring.k], s2));
        }
        if (tl[L]) {
            TEIG_CUDA(launch_update_left(d_q.p + o, (int)cnt, (int)tl[L], dm, d_pool.p, dS, lds, (int)n, s, n, n));
            TEIG_CUDA(launch_update_left(d_q.p + o, (int)cnt, (int)tl[L], dm, d_pool.p, dT, ldt, (int)n, s, n, n));
            launches += 2;
        }
        if (tr[L]) {
            TEIG_CUDA(launch_update_right(d_z.p + o, (int)cnt, (int)tr[L], dm, d_pool.p, dS, lds, (int)n, false, s, n, n));
            TEIG_CUDA(launch_update_right(d_z.p + o, (int)cnt, (int)tr[L], dm, d_pool.p, dT, ldt, (int)n, false, s, n, n));
            launches += 2;
        }
    }
    if (dQ || dZ) {
        TEIG_CUDA(cudaEventRecord(ev, s2));
        TEIG_CUDA(cudaStreamWaitEvent(s, ev, 0));
    }
    std::vector<int32_t> status(std::max<int64_t>(nw, 1));
    std::vector<uint8_t> order(ne + 1), stuck(ne + 1);
    TEIG_CUDA(cudaMemcpyAsync(status.data(), d_status.p, sizeof(int32_t) * nw, cudaMemcpyDeviceToHost, s));
    TEIG_CUDA(cudaMemcpyAsync(order.data(), d_order.p, ne, cudaMemcpyDeviceToHost, s));
    TEIG_CUDA(cudaMemcpyAsync(stuck.data(), d_stuck.p, ne, cudaMemcpyDeviceToHost, s));
    TEIG_CUDA(cudaStreamSynchronize(s));
    std::vector<int32_t> st_by_plan(nw);
    for (int64_t k = 0; k < nw; ++k) st_by_plan[idx[k]] = status[k];
    gp.deviated = fold_outcomes(plan, blocks, st_by_plan, order, stuck, rejected, plan_log, strict);
    gp.windows = 0;
    for (int64_t k = 0; k < nw; ++k) gp.windows += (status[k] & kWinSkipped) ? 0 : 1;
    gp.levels = nl;
    gp.launches = launches;
    return gp;
}

}  // namespace

int greorder_schur_device(int64_t n, double* dS, int64_t lds, double* dT, int64_t ldt, double* dQ, int64_t ldq,
                          double* dZ, int64_t ldz, int64_t nb, const uint8_t* sizes, const uint8_t* flags,
                          const teig_reorder_opts* opts, int64_t* perm, int64_t* rejected_out,
                          teig_reorder_info* info, cudaStream_t stream) {
    if (n < 1) return set_error(-1, "n must be >= 1");
    if (!dS || !dT) return set_error(-2, "S or T is null");
    if (lds < n || ldt < n) return set_error(-3, "lds/ldt < n");
    if ((dQ && ldq < n) || (dZ && ldz < n)) return set_error(-5, "ldq/ldz < n");
    teig_reorder_opts o;
    teig_reorder_opts_default(&o);
    if (opts) o = *opts;
    const int64_t ws = std::min<int64_t>(std::max<int64_t>(o.window_size ? o.window_size : 64, 8), 64);  // shared memory holds S, T, Q_w, Z_w of one window
    std::vector<BlockState> blocks(nb);
    int64_t rows = 0;
    for (int64_t i = 0; i < nb; ++i) {
        if (sizes[i] != 1 && sizes[i] != 2) return set_error(-8, "block sizes must be 1 or 2");
        blocks[i] = BlockState{sizes[i], (uint8_t)(flags[i] ? 1 : 0), (uint32_t)i};
        rows += sizes[i];
    }
    if (rows != n) return set_error(-8, "reorder: selection does not match (S, T)");
    teig_reorder_info inf{};
    std::vector<int64_t> rejected, plan_log;
    cudaStream_t s2 = nullptr;
    cudaEvent_t ev = nullptr;
    try {
        s2 = cached_stream(2);  // kept between calls (launch.h)
        if (!s2) throw std::runtime_error("stream creation failed");
        TEIG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        // row supports of Q's and Z's columns (one device scan each)
        FactorSupport qsupp, zsupp;
        static const bool no_supp = getenv("TEIG_NO_Q_SUPPORT") && atoi(getenv("TEIG_NO_Q_SUPPORT"));
        auto scan = [&](const double* M, int64_t ld, FactorSupport& fs) {
            if (!M || no_supp || o.full_factor) return;
            DBuf<int32_t> dlo(n, stream), dhi(n, stream);
            fs.lo.resize(n);
            fs.hi.resize(n);
            TEIG_CUDA(launch_column_support(M, ld, n, n, dlo.p, dhi.p, stream));
            TEIG_CUDA(cudaMemcpyAsync(fs.lo.data(), dlo.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, stream));
            TEIG_CUDA(cudaMemcpyAsync(fs.hi.data(), dhi.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, stream));
            TEIG_CUDA(cudaStreamSynchronize(stream));
            fs.on = true;
        };
        scan(dQ, ldq, qsupp);
        scan(dZ, ldz, zsupp);
        double exec = 0.0;
        for (int pass = 0; pass < 64; ++pass) {
            ReorderPlan plan = plan_reorder(blocks, ws);
            if (plan.windows.empty()) break;
            if (pass == 0) inf.n_groups = plan.n_groups;
            // two panels per side and two factors: twice the standard flops
            inf.update_flops += 2.0 * plan_update_flops(plan, n, dQ != nullptr || dZ != nullptr);
            inf.update_bytes += 2.0 * plan_update_bytes(plan, n, dQ != nullptr || dZ != nullptr);
            for (const auto& w : plan.windows) {  // per class: (S, T) panels, (Q, Z) factors
                const double d2 = 2.0 * double(w.wbot - w.wtop) * double(w.wbot - w.wtop);
                inf.flops_left += 2.0 * d2 * double(n - w.wbot);
                inf.flops_right += 2.0 * d2 * double(w.wtop);
                inf.flops_factor += ((dQ ? 1.0 : 0.0) + (dZ ? 1.0 : 0.0)) * d2 * double(n);
            }
            GPass gp = run_gpass(plan, n, dS, lds, dT, ldt, dQ, ldq, dZ, ldz, blocks, rejected, plan_log,
                                 o.strict != 0, stream, s2, ev, qsupp, zsupp, &exec);
            inf.n_windows += gp.windows;
            inf.n_levels += gp.levels;
            inf.n_launches += gp.launches;
            inf.n_passes += 1;
            if (!gp.deviated) break;
        }
        inf.flops_factor_exec = exec;
    } catch (const std::domain_error& e) {
        if (s2) cudaStreamSynchronize(s2);
        if (ev) cudaEventDestroy(ev);
        return set_error(TEIG_ERR_STRICT, e.what());
    } catch (const std::exception& e) {
        if (s2) cudaStreamSynchronize(s2);
        if (ev) cudaEventDestroy(ev);
        return set_error(TEIG_ERR_CUDA, e.what());
    }
    cudaEventDestroy(ev);
    bool leading = true, seen = false;
    for (const auto& b : blocks) {
        if (!b.selected) seen = true;
        else if (seen) leading = false;
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
    if (info) *info = inf;
    return 0;
}

}  // namespace teig

using namespace teig;

extern "C" {

int teig_greorder_schur_device(int64_t n, double* dS, int64_t lds, double* dT, int64_t ldt, double* dQ, int64_t ldq,
                               double* dZ, int64_t ldz, int64_t nb, const uint8_t* sizes, const uint8_t* flags,
                               const teig_reorder_opts* opts, int64_t* perm, int64_t* rejected,
                               teig_reorder_info* info, void* stream) {
    DeviceGuard device_guard(dS);
    return greorder_schur_device(n, dS, lds, dT, ldt, dQ, ldq, dZ, ldz, nb, sizes, flags, opts, perm, rejected, info,
                                 (cudaStream_t)stream);
}

int teig_greorder_schur_host(int64_t n, double* S, int64_t lds, double* T, int64_t ldt, double* Q, int64_t ldq,
                             double* Z, int64_t ldz, int64_t nb, const uint8_t* sizes, const uint8_t* flags,
                             const teig_reorder_opts* opts, int64_t* perm, int64_t* rejected,
                             teig_reorder_info* info, void* stream_v) {
    if (n < 1) return set_error(-1, "n must be >= 1");
    if (!S || !T) return set_error(-2, "S or T is null");
    if (lds < n || ldt < n) return set_error(-3, "lds/ldt < n");
    if ((Q && ldq < n) || (Z && ldz < n)) return set_error(-5, "ldq/ldz < n");
    cudaStream_t s = (cudaStream_t)stream_v;
    const size_t pitch = (size_t)n * sizeof(double);
    double* d[4] = {nullptr, nullptr, nullptr, nullptr};
    double* h[4] = {S, T, Q, Z};
    const int64_t ld[4] = {lds, ldt, ldq, ldz};
    int rc = 0;
    try {
        for (int k = 0; k < 4; ++k)
            if (h[k]) {
                TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&d[k]), pitch * n, s));
                TEIG_CUDA(cudaMemcpy2DAsync(d[k], pitch, h[k], ld[k] * sizeof(double), pitch, n, cudaMemcpyHostToDevice, s));
            }
        rc = greorder_schur_device(n, d[0], n, d[1], n, d[2], n, d[3], n, nb, sizes, flags, opts, perm, rejected,
                                   info, s);
        for (int k = 0; k < 4; ++k)
            if (h[k]) {
                if (rc == 0)
                    TEIG_CUDA(cudaMemcpy2DAsync(h[k], ld[k] * sizeof(double), d[k], pitch, pitch, n,
                                                cudaMemcpyDeviceToHost, s));
                TEIG_CUDA(cudaFreeAsync(d[k], s));
            }
        TEIG_CUDA(cudaStreamSynchronize(s));
    } catch (const std::exception& e) {
        return set_error(TEIG_ERR_CUDA, e.what());
    }
    return rc;
}

int teig_gen_pair_t_device(int64_t n, double* dT, int64_t ldt, uint64_t seed, void* stream) {
    DeviceGuard device_guard(dT);
    if (n < 1 || ldt < n) return set_error(-1, "bad shape");
    cudaError_t e = launch_gen_pair_t(dT, ldt, n, seed, (cudaStream_t)stream);
    return e == cudaSuccess ? 0 : set_error(TEIG_ERR_CUDA, cudaGetErrorString(e));
}

}  // extern "C"
