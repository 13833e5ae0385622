// schur_driver.cpp -- host driver of the multishift-QR Schur reduction with
// aggressive early deflation (reference schur.cpp:599-906) over the sm_100a
// window kernels (schur_window.cu) and the DMMA update kernels
// (update_dmma.cu); exported through the C ABI in include/taskeig_b200.h.
//
// The control flow is the reference's schur_reduce round for round -- AED
// rounds, the merged "intro window + chase windows + next AED" round, the
// pending-AED handling, the half-window retry, exceptional shifts, the
// small-block and 2x2 endings -- so convergence behaviour matches the
// reference's constants.  The reference builds one
// TaskGraph per round; here a round is a stream-ordered sequence:
//   * window kernels (one CTA each) and the left (row-panel) updates on the
//     main stream -- the left panel of window k holds the columns window
//     k+1 will read;
//   * the right (column-panel) and Schur-vector updates on a second stream,
//     released by an event after each window kernel (no later window of the
//     round reads the rows above an earlier window);
//   * one readback per round of the AED outcome (deflation count, shifts) --
//     the only host decision points, as in the reference.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/taskeig_b200.h"
#include "device_types.h"
#include "launch.h"
#include "plan.h"
#include "trace.h"

namespace teig {

// plan_chase (schur.cpp:484-505): the chase windows of a chain of nb bulges
// whose bottom bulge enters at p_bot, window order cw, active range end ihi.
std::vector<ChaseWin> plan_chase_windows(int64_t p_bot, int64_t nb, int64_t ihi, int64_t cw) {
    std::vector<ChaseWin> out;
    for (;;) {
        const int64_t p_top = p_bot - 3 * (nb - 1);
        const int64_t a = p_top - 1;
        const int64_t b = std::min(a + cw, ihi);
        ChaseWin c{};
        c.a = (int32_t)a;
        c.d = (int32_t)(b - a);
        c.ihi = (int32_t)ihi;
        c.nb = (int32_t)nb;
        c.p_bot = (int32_t)p_bot;
        c.packed_len = chase_window_packed_len(c.d);
        if (b == ihi) {
            c.mode = kChaseFinal;
            out.push_back(c);
            return out;
        }
        const int64_t hop = (b >= p_bot + 4) ? (b - 4 - p_bot) : 0;
        if (hop == 0) throw std::logic_error("chase window too small for the chain");
        c.mode = kChaseHop;
        c.hop = (int32_t)hop;
        out.push_back(c);
        p_bot += hop;
    }
}

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

constexpr double kEps = 2.220446049250313e-16;
constexpr int64_t kSlot = 128 * 128;  // doubles per Q_w slot

// standardize_2x2 eigenvalues (kernels.cpp:126-219), host copy for the
// exceptional shifts (schur.cpp:815-823)
void std2x2_eigs(double a, double b, double c, double d, std::complex<double>& l1, std::complex<double>& l2) {
    auto sgn = [](double x) { return x >= 0.0 ? 1.0 : -1.0; };
    double cs = 1.0, sn = 0.0;
    const double mx = std::max(std::max(std::fabs(a), std::fabs(b)), std::max(std::fabs(c), std::fabs(d)));
    int ex = 0;
    if (mx > 0.0 && (mx > 1e150 || mx < 1e-150)) {
        ex = std::ilogb(mx);
        const double sc = std::ldexp(1.0, -ex);
        a *= sc; b *= sc; c *= sc; d *= sc;
    }
    if (c == 0.0) {
    } else if (b == 0.0) {
        const double ta = a;
        a = d;
        d = ta;
        b = -c;
        c = 0.0;
    } else if ((a - d) == 0.0 && sgn(b) != sgn(c)) {
    } else {
        const double p = 0.5 * (a - d), q = b + c;
        const double r2 = std::hypot(2.0 * p, q), sig = sgn(q);
        const double cos2 = sig * q / r2, sin2 = -sig * 2.0 * p / r2;
        cs = std::sqrt(0.5 * (1.0 + cos2));
        sn = sin2 / (2.0 * cs);
        const double aa = cs * a + sn * c, bb = cs * b + sn * d;
        const double cc = -sn * a + cs * c, dd = -sn * b + cs * d;
        a = aa * cs + bb * sn;
        b = -aa * sn + bb * cs;
        c = cc * cs + dd * sn;
        d = -cc * sn + dd * cs;
        const double m = 0.5 * (a + d);
        a = m;
        d = m;
        if (c == 0.0) {
        } else if (b == 0.0) {
            b = -c;
            c = 0.0;
        } else if (sgn(b) != sgn(c)) {
        } else {
            const double sab = std::sqrt(std::fabs(b)), sac = std::sqrt(std::fabs(c));
            a = m + sab * sac;
            d = m - sab * sac;
            b = b - c;
            c = 0.0;
        }
    }
    const double back = std::ldexp(1.0, ex);
    if (c == 0.0) {
        l1 = {a * back, 0.0};
        l2 = {d * back, 0.0};
    } else {
        const double beta = std::sqrt(std::fabs(b)) * std::sqrt(std::fabs(c)) * back;
        l1 = {a * back, beta};
        l2 = {a * back, -beta};
    }
}

int64_t default_shift_count(int64_t active) {  // schur.cpp:119-129
    int64_t m = std::max<int64_t>(4, (active / 16) & ~int64_t{1});
    m = std::min<int64_t>(m, 64);
    if (3 * (m / 2) + 2 > active) {
        const int64_t nb = (active >= 6) ? (active - 2) / 3 : 1;
        m = std::min<int64_t>(std::max<int64_t>(2, 2 * nb), 64);
    }
    return m;
}

std::vector<std::complex<double>> pick_shifts(const std::vector<std::complex<double>>& harvest, size_t m_max) {
    std::vector<std::complex<double>> out;  // schur.cpp:97-117
    std::vector<double> reals;
    for (size_t i = 0; i < harvest.size() && out.size() + 1 < m_max + 1; ++i) {
        const auto& z = harvest[i];
        if (z.imag() > 0.0) {
            if (out.size() + 2 <= m_max) {
                out.push_back(z);
                out.push_back(std::conj(z));
            }
        } else if (z.imag() == 0.0) {
            reals.push_back(z.real());
        }
    }
    for (size_t i = 0; i + 1 < reals.size() && out.size() + 2 <= m_max; i += 2) {
        out.emplace_back(reals[i], 0.0);
        out.emplace_back(reals[i + 1], 0.0);
    }
    return out;
}

struct AedHost {
    int64_t window = 0, deflated = 0;
    bool converged = true, swap_rejected = false, spike_eliminated = false;
    std::vector<std::complex<double>> shifts;
};

template <typename T>
struct Grow {  // device buffer that only grows
    T* p = nullptr;
    size_t cap = 0;
    void need(size_t cnt, cudaStream_t s) {
        if (cnt <= cap) return;
        if (p) TEIG_CUDA(cudaFreeAsync(p, s));
        cap = std::max(cnt, cap * 2);
        TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&p), cap * sizeof(T), s));
    }
    void release(cudaStream_t s) {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
    }
};

class SchurRunner {
   public:
    SchurRunner(int64_t n, double* dH, int64_t ldh, double* dQ, int64_t ldq, const teig_schur_opts& o,
                cudaStream_t s)
        : n_(n), dH_(dH), ldh_(ldh), dQ_(dQ), ldq_(ldq), o_(o), s_(s) {
        dopts_.deflation = o.deflation;
        dopts_.shift_count = o.shift_count;
        dopts_.aed_window = o.aed_window;
        dopts_.small_threshold = o.small_threshold;
        dopts_.flags = 0;
        if (getenv("TEIG_NO_WAVE") && atoi(getenv("TEIG_NO_WAVE"))) dopts_.flags |= kSchurFlagNoWave;
        if (getenv("TEIG_NO_LOCAL") && atoi(getenv("TEIG_NO_LOCAL"))) dopts_.flags |= kSchurFlagNoLocal;
        tile_ = o.tile_size ? o.tile_size : default_tile_size(n);
        s2_ = cached_stream(3);  // kept between calls (launch.h)
        if (!s2_) throw std::runtime_error("stream creation failed");
        TEIG_CUDA(cudaEventCreateWithFlags(&ev_, cudaEventDisableTiming));
        TEIG_CUDA(cudaMallocHost(&h_out_, sizeof(AedDevOut) + sizeof(int) * 4 + sizeof(double) * 2 * kAedMaxWindow + 64));
        h_int_ = reinterpret_cast<int*>(h_out_ + 1);
        h_sh_ = reinterpret_cast<double*>(h_int_ + 4);
        TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&d_out_), sizeof(AedDevOut), s_));
        TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&d_int_), sizeof(unsigned long long) * 2, s_));
        TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&d_sh_), sizeof(double) * 2 * kAedMaxWindow, s_));
        TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&d_snap_),
                                  sizeof(double) * 2 * kAedMaxWindow * kAedMaxWindow, s_));
        if (getenv("TEIG_AED_PROF") && atoi(getenv("TEIG_AED_PROF"))) {
            TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&d_prof_), sizeof(unsigned long long) * 16, s_));
            TEIG_CUDA(cudaMemsetAsync(d_prof_, 0, sizeof(unsigned long long) * 16, s_));
        }
        // the factor's row support (plan.h FactorSupport): its updates skip the
        // rows of Q[:, a:b] that are exact zeros (Q_in = I)
        if (dQ_ && !(getenv("TEIG_NO_Q_SUPPORT") && atoi(getenv("TEIG_NO_Q_SUPPORT")))) {
            int32_t *dlo = nullptr, *dhi = nullptr;
            TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&dlo), sizeof(int32_t) * n, s_));
            TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&dhi), sizeof(int32_t) * n, s_));
            qsupp_.lo.resize(n);
            qsupp_.hi.resize(n);
            TEIG_CUDA(launch_column_support(dQ_, ldq_, n, n, dlo, dhi, s_));
            TEIG_CUDA(cudaMemcpyAsync(qsupp_.lo.data(), dlo, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s_));
            TEIG_CUDA(cudaMemcpyAsync(qsupp_.hi.data(), dhi, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s_));
            TEIG_CUDA(cudaFreeAsync(dlo, s_));
            TEIG_CUDA(cudaFreeAsync(dhi, s_));
            TEIG_CUDA(cudaStreamSynchronize(s_));
            qsupp_.on = true;
        }
    }
    ~SchurRunner() {
        if (d_prof_) {
            unsigned long long pf[16] = {0};
            cudaMemcpy(pf, d_prof_, sizeof pf, cudaMemcpyDeviceToHost);
            fprintf(stderr,
                    "[teig aed prof] windows(aed)=%lld chase=%lld | Mcycles: total %.1f small %.1f swap %.1f (n=%llu) "
                    "sweep %.1f spike %.1f | sim_steps %llu small_sweeps %llu | wave steps %llu decide %.1f plan %.1f | "
                    "local %.1f (n=%llu: small %.1f deflate %.1f)\n",
                    (long long)aed_windows_, (long long)chase_windows_, pf[0] / 1e6, pf[1] / 1e6, pf[2] / 1e6, pf[3],
                    pf[4] / 1e6, pf[5] / 1e6, pf[6], pf[7], pf[8], pf[9] / 1e6, pf[10] / 1e6, pf[11] / 1e6, pf[14], pf[12] / 1e6, pf[13] / 1e6);
            cudaFree(d_prof_);
        }
        qw_.release(s_);
        descs_.release(s_);
        cwins_.release(s_);
        pairs_.release(s_);
        if (d_out_) cudaFreeAsync(d_out_, s_);
        if (d_int_) cudaFreeAsync(d_int_, s_);
        if (d_sh_) cudaFreeAsync(d_sh_, s_);
        if (d_snap_) cudaFreeAsync(d_snap_, s_);
        cudaStreamSynchronize(s_);
        if (h_out_) cudaFreeHost(h_out_);
        for (auto e : evpool_) cudaEventDestroy(e);
        if (ev_) cudaEventDestroy(ev_);
        if (s2_) cudaStreamSynchronize(s2_);  // (cached: not destroyed)
    }

    double hnorm() {
        TEIG_CUDA(launch_hess_norm(dH_, ldh_, (int)n_, reinterpret_cast<unsigned long long*>(d_int_), s_));
        double h = 0.0;
        TEIG_CUDA(cudaMemcpyAsync(&h, d_int_, sizeof(double), cudaMemcpyDeviceToHost, s_));
        TEIG_CUDA(cudaStreamSynchronize(s_));
        ++launches_;
        return h;
    }

    int64_t scan(int64_t ihi, double hnorm) {
        TEIG_CUDA(launch_scan_active(dH_, ldh_, (int)n_, (int)ihi, hnorm, d_int_, s_));
        TEIG_CUDA(cudaMemcpyAsync(h_int_, d_int_, sizeof(int), cudaMemcpyDeviceToHost, s_));
        TEIG_CUDA(cudaStreamSynchronize(s_));
        ++launches_;
        return *h_int_;
    }

    // ---- a round: a list of windows executed in order, then one readback
    struct Win {
        int kind;  // 0 AED/small/std2 (mode), 1 chase window
        int mode;
        int64_t a, d, l;
        int cw_idx;
    };

    void begin_round() {
        wins_.clear();
        hchase_.clear();
        hpairs_.clear();
    }
    void add_aed(int mode, int64_t l, int64_t e, int64_t w) { wins_.push_back(Win{0, mode, e, w, l, -1}); }
    void add_chase(const ChaseWin& c) {
        wins_.push_back(Win{1, c.mode, c.a, c.d, 0, (int)hchase_.size()});
        hchase_.push_back(c);
    }

    // runs the round; returns the outcome of its last AED window (if any)
    AedHost run_round() {
        const int64_t nw = (int64_t)wins_.size();
        qw_.need((size_t)nw * kSlot, s_);
        std::vector<WinDesc> descs(nw);
        hdesc_rows_.assign(nw, 0);
        for (int64_t k = 0; k < nw; ++k) {
            WinDesc& w = descs[k];
            std::memset(&w, 0, sizeof w);
            w.a = (int32_t)wins_[k].a;
            w.d = (int32_t)wins_[k].d;
            w.qw_off = k * kSlot;
            w.lc0 = (int32_t)(wins_[k].a + wins_[k].d);
            w.lc1 = (int32_t)n_;
            int64_t q0 = 0, q1 = n_;  // factor rows (windows in execution order)
            if (dQ_ && qsupp_.on) qsupp_.window(wins_[k].a, wins_[k].a + wins_[k].d, &q0, &q1);
            w.rr0 = 0;
            w.rr1 = (int32_t)wins_[k].a;
            w.qr0 = (int32_t)q0;
            w.qr1 = (int32_t)q1;
            hdesc_rows_[k] = q1 - q0;
            if (wins_[k].kind == 1) hchase_[wins_[k].cw_idx].qw_off = k * kSlot;
        }
        descs_.need(nw, s_);
        TEIG_CUDA(cudaMemcpyAsync(descs_.p, descs.data(), sizeof(WinDesc) * nw, cudaMemcpyHostToDevice, s_));
        if (!hchase_.empty()) {
            cwins_.need(hchase_.size(), s_);
            TEIG_CUDA(cudaMemcpyAsync(cwins_.p, hchase_.data(), sizeof(ChaseWin) * hchase_.size(),
                                      cudaMemcpyHostToDevice, s_));
        }
        if (!hpairs_.empty()) {
            pairs_.need(hpairs_.size(), s_);
            TEIG_CUDA(cudaMemcpyAsync(pairs_.p, hpairs_.data(), sizeof(double) * hpairs_.size(),
                                      cudaMemcpyHostToDevice, s_));
        }
        int last_aed = -1, last0 = -1;
        for (int64_t k = 0; k < nw; ++k) {
            const Win& w = wins_[k];
            const int ew0 = prof_begin(s_);
            if (w.kind == 0) {
                last0 = (int)k;
                TEIG_CUDA(launch_aed_window(dH_, ldh_, w.mode, (int)w.l, (int)w.a, (int)w.d, dopts_,
                                            qw_.p + k * kSlot, d_out_, d_sh_, s_, d_prof_, d_snap_));
                if (w.mode == kSchurModeAed) {
                    last_aed = (int)k;
                    ++aed_windows_;
                }
            } else {
                TEIG_CUDA(launch_chase_window(dH_, ldh_, cwins_.p, w.cw_idx, (int)w.d, pairs_.p, qw_.p, s_));
                ++chase_windows_;
            }
            prof_end(0, ew0, s_, w.kind == 0 ? 'A' : 'C');
            ++launches_;
            updates(k, w.a, w.d);
        }
        // join the second stream, read the AED outcome
        TEIG_CUDA(cudaEventRecord(ev_, s2_));
        TEIG_CUDA(cudaStreamWaitEvent(s_, ev_, 0));
        AedHost r;
        if (last0 >= 0) TEIG_CUDA(cudaMemcpyAsync(h_out_, d_out_, sizeof(AedDevOut), cudaMemcpyDeviceToHost, s_));
        if (last_aed >= 0) {
            TEIG_CUDA(cudaMemcpyAsync(h_sh_, d_sh_, sizeof(double) * 2 * wins_[last_aed].d, cudaMemcpyDeviceToHost, s_));
        }
        TEIG_CUDA(cudaStreamSynchronize(s_));
        prof_collect();
        ++rounds_;
        if (last_aed >= 0) {
            const AedDevOut& o = *h_out_;
            r.window = wins_[last_aed].d;
            r.deflated = o.deflated;
            r.converged = o.converged != 0;
            r.swap_rejected = o.swap_rejected != 0;
            r.spike_eliminated = o.spike_eliminated != 0;
            for (int i = 0; i < o.nshifts; ++i) r.shifts.emplace_back(h_sh_[2 * i], h_sh_[2 * i + 1]);
        }
        last_converged_ = last0 >= 0 ? h_out_->converged != 0 : true;
        return r;
    }

    // converged flag of the last small-solve window (read after run_round)
    bool last_small_converged() const { return last_converged_; }

    // intro window (introduce_bulges, schur.cpp:628-647 / :833-867)
    void plan_intro(int64_t l, int64_t ihi, const std::vector<std::complex<double>>& shifts, int64_t nb) {
        const int64_t wi = std::min(l + 3 * nb + 2, ihi);
        ChaseWin in{};
        in.a = (int32_t)l;
        in.d = (int32_t)(wi - l);
        in.ihi = (int32_t)ihi;
        in.mode = kChaseIntro;
        in.nb = (int32_t)nb;
        in.p_bot = (int32_t)(l + 1 + 3 * (nb - 1));
        in.shift_off = (int32_t)hpairs_.size();
        in.packed_len = chase_window_packed_len(in.d);
        for (int64_t j = 0; j < nb; ++j) {
            hpairs_.push_back(shifts[2 * j].real());
            hpairs_.push_back(shifts[2 * j].imag());
            hpairs_.push_back(shifts[2 * j + 1].real());
            hpairs_.push_back(shifts[2 * j + 1].imag());
        }
        add_chase(in);
    }

    // merged-round planning: intro window + plan_chase (schur.cpp:828-871)
    void plan_sweep(int64_t l, int64_t ihi, const std::vector<std::complex<double>>& shifts, int64_t nb, int64_t cw) {
        plan_intro(l, ihi, shifts, nb);
        plan_chain(l + 1 + 3 * (nb - 1), nb, ihi, cw);
    }

    // plan_chase (schur.cpp:484-505) for a chain whose bottom bulge enters at p_bot
    void plan_chain(int64_t p_bot, int64_t nb, int64_t ihi, int64_t cw) {
        for (const ChaseWin& c : plan_chase_windows(p_bot, nb, ihi, cw)) add_chase(c);
    }

    int64_t round_windows() const { return (int64_t)wins_.size(); }

    void fill_info(teig_schur_info* info) const {
        info->rounds = rounds_;
        info->aed_windows = aed_windows_;
        info->chase_windows = chase_windows_;
        info->n_launches = launches_;
        info->update_flops = flops_;
        info->ms_window = ms_[0];
        info->ms_update = ms_[1];
    }

    int64_t tile() const { return tile_; }

   private:
    void updates(int64_t k, int64_t a, int64_t d) {
        const int64_t b = a + d;
        const int dm = d <= 64 ? 64 : 128;
        const WinDesc* dd = descs_.p + k;
        const int tl = (int)((n_ - b + kLeftBN - 1) / kLeftBN);
        const int tr = (int)((a + kRightBM - 1) / kRightBM);
        const int64_t qrows = dQ_ ? (int64_t)hdesc_rows_[k] : 0;
        const int tq = dQ_ ? (int)((qrows + kRightBM - 1) / kRightBM) : 0;
        const double dd2 = 2.0 * double(d) * double(d);
        flops_ += dd2 * double(n_ - b) + dd2 * double(a) + (dQ_ ? dd2 * double(n_) : 0.0);
        if (tl > 0) {
            const int e0 = prof_begin(s_);
            TEIG_CUDA(launch_update_left(dd, 1, tl, dm, qw_.p, dH_, ldh_, (int)n_, s_, n_, n_));
            prof_end(1, e0, s_, 'L');
            ++launches_;
        }
        if (tr > 0 || tq > 0) {
            TEIG_CUDA(cudaEventRecord(ev_, s_));
            TEIG_CUDA(cudaStreamWaitEvent(s2_, ev_, 0));
        }
        if (tr > 0) {
            const int e0 = prof_begin(s2_);
            TEIG_CUDA(launch_update_right(dd, 1, tr, dm, qw_.p, dH_, ldh_, (int)n_, false, s2_, n_, n_));
            prof_end(1, e0, s2_, 'R');
            ++launches_;
        }
        if (tq > 0) {
            const int e0 = prof_begin(s2_);
            TEIG_CUDA(launch_update_right(dd, 1, tq, dm, qw_.p, dQ_, ldq_, (int)n_, true, s2_, n_, n_));
            prof_end(1, e0, s2_, 'Q');
            ++launches_;
        }
    }

    int prof_begin(cudaStream_t s) {
        if (!o_.profile) return -1;
        if (nev_ == evpool_.size()) {
            cudaEvent_t e;
            TEIG_CUDA(cudaEventCreate(&e));
            evpool_.push_back(e);
        }
        TEIG_CUDA(cudaEventRecord(evpool_[nev_], s));
        return (int)nev_++;
    }
    // kind (trace label): 'A' AED / small-solve window, 'C' chase window,
    // 'L' / 'R' / 'Q' updates
    void prof_end(int cls, int e0, cudaStream_t s, char kind = '?') {
        if (e0 < 0) return;
        const int e1 = prof_begin(s);
        spans_.push_back({cls, e0, e1, kind, s == s_ ? 0 : 1});
    }
    void prof_collect() {
        for (auto& sp : spans_) {
            float ms = 0.f;
            TEIG_CUDA(cudaEventElapsedTime(&ms, evpool_[sp.e0], evpool_[sp.e1]));
            ms_[sp.cls] += ms;
            if (g_trace.on) {  // SchurOptions::keep_reports: one record per launch
                float t0 = 0.f, t1 = 0.f;
                TEIG_CUDA(cudaEventElapsedTime(&t0, g_trace.origin, evpool_[sp.e0]));
                TEIG_CUDA(cudaEventElapsedTime(&t1, g_trace.origin, evpool_[sp.e1]));
                g_trace.tasks.push_back({std::string("schur:") + sp.kind + ":r" + std::to_string(rounds_), sp.worker,
                                         (int64_t)(t0 * 1e6), (int64_t)(t1 * 1e6)});
            }
        }
        spans_.clear();
        nev_ = 0;
    }

    struct Span {
        int cls, e0, e1;
        char kind;
        int worker;
    };

    int64_t n_;
    double* dH_;
    int64_t ldh_;
    double* dQ_;
    int64_t ldq_;
    teig_schur_opts o_;
    cudaStream_t s_, s2_ = nullptr;
    cudaEvent_t ev_ = nullptr;
    SchurDevOpts dopts_{};
    int64_t tile_ = 128;
    Grow<double> qw_, pairs_;
    Grow<WinDesc> descs_;
    Grow<ChaseWin> cwins_;
    AedDevOut* h_out_ = nullptr;
    int* h_int_ = nullptr;
    double* h_sh_ = nullptr;
    AedDevOut* d_out_ = nullptr;
    int* d_int_ = nullptr;
    double* d_sh_ = nullptr;
    unsigned long long* d_prof_ = nullptr;
    double* d_snap_ = nullptr;
    std::vector<Win> wins_;
    std::vector<ChaseWin> hchase_;
    std::vector<double> hpairs_;
    std::vector<cudaEvent_t> evpool_;
    size_t nev_ = 0;
    std::vector<Span> spans_;
    FactorSupport qsupp_;
    std::vector<int64_t> hdesc_rows_;  // factor rows of each window of the round
    double ms_[2] = {0, 0};
    double flops_ = 0;
    bool last_converged_ = true;
    int64_t launches_ = 0, rounds_ = 0, aed_windows_ = 0, chase_windows_ = 0;
};

// Validates the options and clamps the window sizes to what one CTA's shared
// memory holds (the reference takes any size, schur.cpp:777, 869): a larger
// AED window / small-solve threshold runs at 104, a larger chase window at
// 128, a larger shift count at 64 (the reference's own default cap) -- the
// result satisfies the same contract (Schur form, residuals, eigenvalues);
// only the convergence history differs.
int check_opts(teig_schur_opts& o) {
    if (o.deflation != 0 && o.deflation != 1) return set_error(-7, "deflation must be 0 (classic) or 1 (norm-stable)");
    if (o.shift_count < 0 || o.aed_window < 0 || o.small_threshold < 0 || o.iteration_limit < 0 || o.tile_size < 0)
        return set_error(-7, "negative option");
    o.shift_count = std::min<int32_t>(o.shift_count, 64);
    o.aed_window = std::min<int32_t>(o.aed_window, kAedMaxWindow);
    o.small_threshold = std::min<int32_t>(o.small_threshold, kAedMaxWindow);
    o.tile_size = std::min<int64_t>(o.tile_size, kChaseMaxWindow);
    return 0;
}

}  // namespace

int schur_reduce_device(int64_t n, double* dH, int64_t ldh, double* dQ, int64_t ldq, const teig_schur_opts* opts,
                        double* eig_re, double* eig_im, teig_schur_info* info, cudaStream_t stream) {
    if (n < 1) return set_error(-1, "n must be >= 1");
    if (!dH) return set_error(-2, "H is null");
    if (ldh < n) return set_error(-3, "ldh < n");
    if (dQ && ldq < n) return set_error(-5, "ldq < n");
    if (n > 2147483647LL) return set_error(TEIG_ERR_UNSUPPORTED, "n too large");
    teig_schur_opts o;
    teig_schur_opts_default(&o);
    if (opts) o = *opts;
    if (int rc = check_opts(o)) return rc;
    const int64_t thr = o.small_threshold;
    teig_schur_info inf{};
    const auto t0 = std::chrono::steady_clock::now();
    try {
        if (g_trace.on) {  // the trace needs the per-launch events
            o.profile = 1;
            g_trace.begin(stream);
        }
        SchurRunner R(n, dH, ldh, dQ, ldq, o, stream);
        const int64_t limit = o.iteration_limit ? o.iteration_limit : 30 * n;
        const double hnorm = R.hnorm();
        auto aed_window_for = [&](int64_t active) {
            const int64_t m = o.shift_count ? o.shift_count : default_shift_count(active);
            int64_t w = o.aed_window ? o.aed_window : (3 * m) / 2;
            return std::min(std::max<int64_t>(w, 4), active);
        };
        auto aed_round = [&](int64_t l, int64_t ihi, int64_t w) {  // aed_step (schur.cpp:599-609)
            w = std::min(w, ihi - l);
            R.begin_round();
            R.add_aed(kSchurModeAed, l, ihi - w, w);
            return R.run_round();
        };
        int64_t ihi = n, stagnation = 0, sweeps = 0;
        bool pending = false, hard_fail = false;
        AedHost pend;
        if (n > (int64_t)kAedMaxWindow * 1000000) throw std::runtime_error("n too large");
        while (ihi > 0 && !hard_fail) {
            AedHost res;
            bool have_aed = false;
            int64_t l = 0;
            if (pending) {
                res = pend;
                pending = false;
                have_aed = true;
                if (!res.converged) {
                    const int64_t w2 = std::max<int64_t>(4, res.window / 2);
                    l = R.scan(ihi, hnorm);
                    if (w2 < res.window && ihi - l >= w2) res = aed_round(l, ihi, w2);
                    if (!res.converged) {
                        hard_fail = true;
                        break;
                    }
                }
                ihi -= res.deflated;
                stagnation = (res.deflated == 0) ? stagnation + 1 : 0;
                if (ihi == 0) break;
            }
            l = R.scan(ihi, hnorm);
            int64_t active = ihi - l;
            if (active == 1) {
                ihi = l;
                pending = false;
                continue;
            }
            if (active == 2) {  // schur.cpp:728-757
                R.begin_round();
                R.add_aed(kSchurModeStd2, l, l, 2);
                R.run_round();
                ihi = l;
                continue;
            }
            if (active <= thr) {  // schur.cpp:758-772
                R.begin_round();
                R.add_aed(kSchurModeSmall, l, l, active);
                R.run_round();
                if (!R.last_small_converged()) {
                    hard_fail = true;
                    break;
                }
                ihi = l;
                continue;
            }
            if (!have_aed) {
                const int64_t w = aed_window_for(active);
                res = aed_round(l, ihi, w);
                if (!res.converged) {
                    const int64_t w2 = std::max<int64_t>(4, w / 2);
                    if (w2 < w) res = aed_round(l, ihi, w2);
                    if (!res.converged) {
                        hard_fail = true;
                        break;
                    }
                }
                ihi -= res.deflated;
                stagnation = (res.deflated == 0) ? stagnation + 1 : 0;
                if (ihi == 0) break;
                l = R.scan(ihi, hnorm);
                active = ihi - l;
                if (active < 4) continue;
            }
            if (res.deflated > 0 && 100 * res.deflated >= 14 * res.window) continue;
            if (active <= thr) continue;
            if (sweeps >= limit) {
                hard_fail = true;
                break;
            }
            ++sweeps;
            const int64_t m_want = o.shift_count ? o.shift_count : default_shift_count(active);
            auto shifts = pick_shifts(res.shifts, (size_t)m_want);
            if (stagnation >= 6 || shifts.size() < 2) {  // schur.cpp:815-823
                double hv[3] = {0, 0, 0};
                TEIG_CUDA(cudaMemcpyAsync(&hv[0], dH + (ihi - 1) + (ihi - 2) * ldh, sizeof(double), cudaMemcpyDeviceToHost, stream));
                TEIG_CUDA(cudaMemcpyAsync(&hv[2], dH + (ihi - 1) + (ihi - 1) * ldh, sizeof(double), cudaMemcpyDeviceToHost, stream));
                if (ihi >= l + 3)
                    TEIG_CUDA(cudaMemcpyAsync(&hv[1], dH + (ihi - 2) + (ihi - 3) * ldh, sizeof(double), cudaMemcpyDeviceToHost, stream));
                TEIG_CUDA(cudaStreamSynchronize(stream));
                const double sp = std::fabs(hv[0]) + ((ihi >= l + 3) ? std::fabs(hv[1]) : 0.0);
                const double h11 = 0.75 * sp + hv[2];
                std::complex<double> l1, l2;
                std2x2_eigs(h11, -0.4375 * sp, sp, h11, l1, l2);
                shifts = {l1, l2};
                stagnation = 0;
            }
            const int64_t nb = std::min<int64_t>((int64_t)shifts.size() / 2, (active - 2) / 3);
            if (nb == 0) continue;
            shifts.resize(2 * nb);
            // merged round: intro window + chase windows + the next AED
            const int64_t cw = std::max<int64_t>(R.tile(), 3 * nb + 6);
            if (cw > kChaseMaxWindow) throw std::domain_error("chase window > 128 (shift count too large)");
            R.begin_round();
            R.plan_sweep(l, ihi, shifts, nb, cw);
            const int64_t w2 = aed_window_for(active);
            R.add_aed(kSchurModeAed, l, ihi - w2, w2);
            pend = R.run_round();
            pending = true;
        }
        inf.sweeps = sweeps;
        inf.converged = hard_fail ? 0 : 1;
        inf.converged_trailing = n - ihi;
        R.fill_info(&inf);
    } catch (const std::domain_error& e) {
        return set_error(TEIG_ERR_UNSUPPORTED, e.what());
    } catch (const std::exception& e) {
        return set_error(TEIG_ERR_CUDA, e.what());
    }
    inf.ms_total_host = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    // eigenvalue read-off (schur.cpp:888-904)
    if (inf.converged && (eig_re || eig_im)) {
        std::vector<double> dg(n), sub(n, 0.0), sup(n, 0.0);
        try {
            TEIG_CUDA(cudaMemcpy2DAsync(dg.data(), sizeof(double), dH, (ldh + 1) * sizeof(double), sizeof(double), n,
                                        cudaMemcpyDeviceToHost, stream));
            if (n > 1) {
                TEIG_CUDA(cudaMemcpy2DAsync(sub.data(), sizeof(double), dH + 1, (ldh + 1) * sizeof(double), sizeof(double),
                                            n - 1, cudaMemcpyDeviceToHost, stream));
                TEIG_CUDA(cudaMemcpy2DAsync(sup.data(), sizeof(double), dH + ldh, (ldh + 1) * sizeof(double),
                                            sizeof(double), n - 1, cudaMemcpyDeviceToHost, stream));
            }
            TEIG_CUDA(cudaStreamSynchronize(stream));
        } catch (const std::exception& e) {
            return set_error(TEIG_ERR_CUDA, e.what());
        }
        for (int64_t i = 0; i < n;) {
            if (i + 1 < n && sub[i] != 0.0) {
                const double im = std::sqrt(std::fabs(sup[i])) * std::sqrt(std::fabs(sub[i]));
                if (eig_re) eig_re[i] = eig_re[i + 1] = dg[i];
                if (eig_im) {
                    eig_im[i] = im;
                    eig_im[i + 1] = -im;
                }
                i += 2;
            } else {
                if (eig_re) eig_re[i] = dg[i];
                if (eig_im) eig_im[i] = 0.0;
                i += 1;
            }
        }
    }
    if (info) *info = inf;
    return 0;
}

}  // namespace teig

// ============================================================================
// C ABI
// ============================================================================
using namespace teig;

extern "C" {

void teig_schur_opts_default(teig_schur_opts* o) {
    std::memset(o, 0, sizeof *o);
    o->deflation = 1;
    o->small_threshold = 64;
}

int teig_deflation_check(double spike, double diag_sum, int32_t deflation, double wnorm) {
    if (!deflation) return spike <= std::fmax(kEps * diag_sum, 2.2250738585072014e-308) ? 1 : 0;
    return spike <= kEps * wnorm ? 1 : 0;
}

int teig_schur_reduce_device(int64_t n, double* dH, int64_t ldh, double* dQ, int64_t ldq, const teig_schur_opts* o,
                             double* eig_re, double* eig_im, teig_schur_info* info, void* stream) {
    DeviceGuard device_guard(dH);
    return schur_reduce_device(n, dH, ldh, dQ, ldq, o, eig_re, eig_im, info, (cudaStream_t)stream);
}

int teig_schur_reduce_host(int64_t n, double* H, int64_t ldh, double* Q, int64_t ldq, const teig_schur_opts* o,
                           double* eig_re, double* eig_im, teig_schur_info* info, void* stream_v) {
    if (n < 1) return set_error(-1, "n must be >= 1");
    if (!H) return set_error(-2, "H is null");
    if (ldh < n) return set_error(-3, "ldh < n");
    if (Q && ldq < n) return set_error(-5, "ldq < n");
    cudaStream_t stream = (cudaStream_t)stream_v;
    double *dH = nullptr, *dQ = nullptr;
    int rc = 0;
    try {
        const size_t pitch = (size_t)n * sizeof(double);
        TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&dH), pitch * n, stream));
        if (Q) TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&dQ), pitch * n, stream));
        TEIG_CUDA(cudaMemcpy2DAsync(dH, pitch, H, ldh * sizeof(double), pitch, n, cudaMemcpyHostToDevice, stream));
        if (Q) TEIG_CUDA(cudaMemcpy2DAsync(dQ, pitch, Q, ldq * sizeof(double), pitch, n, cudaMemcpyHostToDevice, stream));
        rc = schur_reduce_device(n, dH, n, dQ, n, o, eig_re, eig_im, info, stream);
        if (rc == 0) {
            TEIG_CUDA(cudaMemcpy2DAsync(H, ldh * sizeof(double), dH, pitch, pitch, n, cudaMemcpyDeviceToHost, stream));
            if (Q) TEIG_CUDA(cudaMemcpy2DAsync(Q, ldq * sizeof(double), dQ, pitch, pitch, n, cudaMemcpyDeviceToHost, stream));
        }
        TEIG_CUDA(cudaFreeAsync(dH, stream));
        if (dQ) TEIG_CUDA(cudaFreeAsync(dQ, stream));
        TEIG_CUDA(cudaStreamSynchronize(stream));
    } catch (const std::exception& e) {
        return set_error(TEIG_ERR_CUDA, e.what());
    }
    return rc;
}

int teig_aed_step_device(int64_t n, double* dH, int64_t ldh, double* dQ, int64_t ldq, int64_t l, int64_t ihi,
                         int64_t window, const teig_schur_opts* opts, teig_aed_result* r, double* shifts, void* stream) {
    DeviceGuard device_guard(dH);
    if (n < 1) return set_error(-1, "n must be >= 1");
    if (!dH || ldh < n) return set_error(-3, "bad H");
    if (dQ && ldq < n) return set_error(-5, "ldq < n");
    if (l < 0 || ihi > n || l >= ihi) return set_error(-6, "bad active range");
    if (window < 4) return set_error(-8, "aed_step: window must be >= 4");  // schur.cpp:601
    teig_schur_opts o;
    teig_schur_opts_default(&o);
    if (opts) o = *opts;
    if (int rc = check_opts(o)) return rc;
    window = std::min(window, ihi - l);
    window = std::min<int64_t>(window, kAedMaxWindow);  // one CTA's shared memory (see check_opts)
    try {
        SchurRunner R(n, dH, ldh, dQ, ldq, o, (cudaStream_t)stream);
        R.begin_round();
        R.add_aed(kSchurModeAed, l, ihi - window, window);
        AedHost a = R.run_round();
        if (r) {
            r->window = window;
            r->deflated = a.deflated;
            r->nshifts = (int64_t)a.shifts.size();
            r->spike_eliminated = a.spike_eliminated;
            r->converged = a.converged;
            r->swap_rejected = a.swap_rejected;
        }
        if (shifts)
            for (size_t i = 0; i < a.shifts.size(); ++i) {
                shifts[2 * i] = a.shifts[i].real();
                shifts[2 * i + 1] = a.shifts[i].imag();
            }
    } catch (const std::exception& e) {
        return set_error(TEIG_ERR_CUDA, e.what());
    }
    return 0;
}

int teig_introduce_bulges_device(int64_t n, double* dH, int64_t ldh, double* dQ, int64_t ldq, int64_t l, int64_t ihi,
                                 int64_t nshifts, const double* shifts, int64_t* positions, void* stream) {
    DeviceGuard device_guard(dH);
    if (n < 1) return set_error(-1, "n must be >= 1");
    if (!dH || ldh < n) return set_error(-3, "bad H");
    if (dQ && ldq < n) return set_error(-5, "ldq < n");
    if (l < 0 || ihi > n || l >= ihi) return set_error(-6, "bad active range");
    // schur.cpp:614-626
    if (nshifts < 2) return set_error(-8, "introduce_bulges: need at least two shifts");
    if (nshifts % 2 != 0) return set_error(-8, "introduce_bulges: shifts must come in pairs");
    for (int64_t j = 0; j + 1 < nshifts; j += 2) {
        const double r1 = shifts[2 * j], i1 = shifts[2 * j + 1], r2 = shifts[2 * j + 2], i2 = shifts[2 * j + 3];
        if (i1 != 0.0 && (r1 != r2 || i1 != -i2)) return set_error(-8, "introduce_bulges: shift pair not conjugate");
    }
    const int64_t nb = nshifts / 2;
    if (l + 3 * nb + 2 > ihi) return set_error(-8, "introduce_bulges: too many shifts for range");
    if (3 * nb + 2 > kChaseMaxWindow) return set_error(TEIG_ERR_UNSUPPORTED, "too many bulges for one window");
    teig_schur_opts o;
    teig_schur_opts_default(&o);
    try {
        SchurRunner R(n, dH, ldh, dQ, ldq, o, (cudaStream_t)stream);
        std::vector<std::complex<double>> sh;
        for (int64_t i = 0; i < nshifts; ++i) sh.emplace_back(shifts[2 * i], shifts[2 * i + 1]);
        R.begin_round();
        // intro window only (introduce_bulges, schur.cpp:628-647)
        R.plan_intro(l, ihi, sh, nb);
        R.run_round();
    } catch (const std::exception& e) {
        return set_error(TEIG_ERR_CUDA, e.what());
    }
    if (positions)
        for (int64_t j = 0; j < nb; ++j) positions[j] = l + 1 + 3 * (nb - 1 - j);  // bottom first
    return 0;
}

int teig_chase_bulges_device(int64_t n, double* dH, int64_t ldh, double* dQ, int64_t ldq, int64_t chain_end,
                             int64_t nb, const int64_t* positions, int64_t window_size, int64_t* n_windows,
                             void* stream) {
    DeviceGuard device_guard(dH);
    if (n < 1) return set_error(-1, "n must be >= 1");
    if (!dH || ldh < n) return set_error(-3, "bad H");
    if (dQ && ldq < n) return set_error(-5, "ldq < n");
    if (chain_end > n || chain_end < 1) return set_error(-6, "bad chain end");
    if (nb == 0) {
        if (n_windows) *n_windows = 0;
        return 0;
    }
    if (nb < 0 || !positions) return set_error(-7, "bad chain");
    for (int64_t k = 0; k < nb; ++k)
        if (positions[k] != positions[0] - 3 * k || positions[k] < 1)
            return set_error(-8, "bulge positions must be bottom first and 3 rows apart (introduce_bulges)");
    const int64_t cw = std::max<int64_t>(window_size, 3 * nb + 6);  // schur.cpp:655
    if (cw > kChaseMaxWindow) return set_error(TEIG_ERR_UNSUPPORTED, "chase window > 128");
    teig_schur_opts o;
    teig_schur_opts_default(&o);
    try {
        SchurRunner R(n, dH, ldh, dQ, ldq, o, (cudaStream_t)stream);
        R.begin_round();
        R.plan_chain(positions[0], nb, chain_end, cw);
        if (n_windows) *n_windows = R.round_windows();
        R.run_round();
    } catch (const std::logic_error& e) {
        return set_error(-9, e.what());
    } catch (const std::exception& e) {
        return set_error(TEIG_ERR_CUDA, e.what());
    }
    return 0;
}

int64_t teig_plan_chase(int64_t nb, const int64_t* positions, int64_t chain_end, int64_t window_size,
                        int64_t* win, int64_t cap) {
    if (nb <= 0) return 0;
    if (!positions) return set_error(-2, "positions is null");
    const int64_t cw = std::max<int64_t>(window_size, 3 * nb + 6);
    try {
        const auto w = plan_chase_windows(positions[0], nb, chain_end, cw);
        for (int64_t i = 0; win && i < (int64_t)w.size() && i < cap; ++i) {
            win[3 * i] = w[i].a;
            win[3 * i + 1] = w[i].d;
            win[3 * i + 2] = w[i].mode;
        }
        return (int64_t)w.size();
    } catch (const std::logic_error& e) {
        return set_error(-9, e.what());
    }
}

int teig_small_schur_device(int64_t k, double* dH, int64_t ldh, double* dQ, int32_t* converged, void* stream) {
    DeviceGuard device_guard(dH);
    if (k < 1) return set_error(-1, "k must be >= 1");
    if (!dH || ldh < k) return set_error(-3, "bad H");
    if (!dQ) return set_error(-4, "Q is null");
    if (k > kAedMaxWindow) return set_error(TEIG_ERR_UNSUPPORTED, "small_schur order > 104");
    teig_schur_opts o;
    teig_schur_opts_default(&o);
    try {
        AedDevOut* dout = nullptr;
        AedDevOut hout{};
        cudaStream_t s = (cudaStream_t)stream;
        TEIG_CUDA(lib_malloc_async(reinterpret_cast<void**>(&dout), sizeof(AedDevOut), s));
        SchurDevOpts d{o.deflation, o.shift_count, o.aed_window, o.small_threshold, 0};
        TEIG_CUDA(launch_aed_window(dH, ldh, kSchurModeSmall, 0, 0, (int)k, d, dQ, dout, nullptr, s));
        TEIG_CUDA(cudaMemcpyAsync(&hout, dout, sizeof hout, cudaMemcpyDeviceToHost, s));
        TEIG_CUDA(cudaFreeAsync(dout, s));
        TEIG_CUDA(cudaStreamSynchronize(s));
        if (converged) *converged = hout.converged;
    } catch (const std::exception& e) {
        return set_error(TEIG_ERR_CUDA, e.what());
    }
    return 0;
}

}  // extern "C"
