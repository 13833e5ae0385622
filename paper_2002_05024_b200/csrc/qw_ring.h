// qw_ring.h -- the per-level ring of window accumulators shared by the
// reorder drivers (reorder_driver.cpp, greorder_driver.cpp).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "device_types.h"

namespace teig {

// The accumulators of one pass as a ring of per-level regions instead of one
// slot per window (n=40000: 6.4 GB for the whole pass vs ~0.3-1 GB): window
// descriptors (level-ordered) get qw_off = region(L) + prefix within level.
// K = how many levels' regions fit the budget (TEIG_QW_RING_MB, default
// 1024).  A region's readers on another stream (the factor updates) are
// ordered before its reuse with RingEvents.  per_win: number
// of d x d accumulators per window (1: Q_w; 2: Q_w and Z_w).
struct QwRing {
    int64_t total = 0;  // doubles
    int k = 0;          // regions (0: no ring, every window its own slot)
};
inline QwRing make_qw_ring(std::vector<WinDesc>& descs, const std::vector<int64_t>& lvl_off, int nl, int per_win) {
    QwRing r;
    int64_t lmax = 0;
    std::vector<int64_t> lsz(nl, 0);
    for (int L = 0; L < nl; ++L) {
        for (int64_t k = lvl_off[L]; k < lvl_off[L + 1]; ++k) lsz[L] += per_win * (int64_t)descs[k].d * descs[k].d;
        lmax = std::max(lmax, lsz[L]);
    }
    static const int64_t budget_mb = getenv("TEIG_QW_RING_MB") ? atoll(getenv("TEIG_QW_RING_MB")) : 1024;
    int64_t kreg = lmax > 0 ? std::max<int64_t>(4, (budget_mb << 20) / 8 / lmax) : nl;
    if (budget_mb <= 0 || kreg >= nl) {  // everything fits: one slot per window, no reuse
        int64_t off = 0;
        for (auto& d : descs) {
            d.qw_off = off;
            off += per_win * (int64_t)d.d * d.d;
        }
        r.total = off;
        r.k = 0;
        return r;
    }
    r.k = (int)kreg;
    for (int L = 0; L < nl; ++L) {
        int64_t off = (L % r.k) * lmax;
        for (int64_t k = lvl_off[L]; k < lvl_off[L + 1]; ++k) {
            descs[k].qw_off = off;
            off += per_win * (int64_t)descs[k].d * descs[k].d;
        }
    }
    r.total = (int64_t)r.k * lmax;
    return r;
}

// a set of timing-free events (RAII)
struct StreamEvents {
    std::vector<cudaEvent_t> ev;
    explicit StreamEvents(int k) {
        ev.assign(k, nullptr);
        for (auto& e : ev) {
            cudaError_t err = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
            if (err != cudaSuccess) throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(err));
        }
    }
    ~StreamEvents() {
        for (auto e : ev)
            if (e) cudaEventDestroy(e);
    }
};

// one event per ring region (recorded after the region's last off-stream reader)
struct RingEvents {
    int n = 0;
    std::vector<cudaEvent_t> ev;
    explicit RingEvents(int k) : n(k) {
        ev.assign(k, nullptr);
        for (auto& e : ev) {
            cudaError_t err = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
            if (err != cudaSuccess) throw std::runtime_error(std::string("CUDA error ") + cudaGetErrorString(err));
        }
    }
    ~RingEvents() {
        for (auto e : ev)
            if (e) cudaEventDestroy(e);
    }
};

}  // namespace teig
