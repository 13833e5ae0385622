// taskeig_adapter.cpp -- the C++ drop-in: the reference's `taskeig::` entry
// points of the window-based update path, implemented over the B200 C ABI
// (include/taskeig_b200.h).
//
// Compiled against the reference's OWN public headers (proj/include/taskeig,
// unmodified) so the types are the reference's types, this translation unit
// replaces exactly the two reference objects that implement the path:
//   reorder.o   (reorder.hpp:22-89):  Selection::selected_rows,
//               select_eigenvalues x2, select_fraction, select_by_name,
//               window_reorder, reorder_schur
//   schur.o     (schur.hpp:62-95):    deflation_check, aed_step,
//               introduce_bulges, chase_bulges, schur_reduce
// A reference build links this object and libtaskeig_b200.so instead of
// reorder.o / schur.o; every other reference object (TiledMatrix, kernels,
// Hessenberg reduction, eigenvectors, verify, IO) is unchanged
// (tests/refcpp runs the reference's own test_reorder.cpp and
// test_schur.cpp this way).
//
// TiledMatrix <-> device.  A TiledMatrix stores column-major tiles
// (tiled_matrix.hpp:27-35); the device layout is one column-major matrix with
// ld = n.  A block column of tiles (n x tile) is packed into one of two pinned
// staging chunks and copied with ONE cudaMemcpyAsync while the host packs the
// next block column into the other chunk (and the reverse on the way back):
// one host pass + one H2D/D2H pass over the matrix, bounded pinned memory
// (2 n tile doubles).
//
// Errors map onto the reference's conventions: argument errors
// (C ABI status < 0) -> std::invalid_argument with the library's message;
// strict-mode rejection -> std::runtime_error (reorder.cpp:383-385); device /
// unsupported-size failures -> std::runtime_error.  Non-convergence stays a
// flag (SchurDecomposition::converged).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <complex>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "taskeig/reorder.hpp"
#include "taskeig/schur.hpp"
#include "taskeig/tiled_matrix.hpp"
#include "taskeig_b200.h"

namespace taskeig {

namespace {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("taskeig_b200: ") + what + ": " + cudaGetErrorString(e));
}

// C ABI status -> the reference's exception types
void teig_check(int rc, const char* fn) {
    if (rc == 0) return;
    const std::string msg = std::string(fn) + ": " + teig_last_error();
    if (rc == TEIG_ERR_STRICT) throw std::runtime_error("reorder_schur: swap rejected in strict mode");
    if (rc < 0 && rc > TEIG_ERR_CUDA) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

// one stream + RAII device buffers per call
struct Stream {
    cudaStream_t s = nullptr;
    Stream() { cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream"); }
    ~Stream() {
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    }
};

struct DevBuf {
    double* p = nullptr;
    DevBuf() = default;
    explicit DevBuf(size_t doubles) {
        if (doubles) cuda_check(cudaMalloc(reinterpret_cast<void**>(&p), doubles * sizeof(double)), "cudaMalloc");
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

// two pinned chunks of one block column each, with their copy events
struct Staging {
    double* chunk[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    explicit Staging(size_t doubles) {
        for (int b = 0; b < 2; ++b) {
            cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&chunk[b]), std::max<size_t>(doubles, 1) * sizeof(double),
                                     cudaHostAllocDefault),
                       "cudaHostAlloc");
            cuda_check(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming), "event");
        }
    }
    ~Staging() {
        for (int b = 0; b < 2; ++b) {
            if (ev[b]) {
                cudaEventSynchronize(ev[b]);
                cudaEventDestroy(ev[b]);
            }
            if (chunk[b]) cudaFreeHost(chunk[b]);
        }
    }
};

// TiledMatrix (rows x cols) -> device column-major, ld = rows
void upload(const TiledMatrix& m, double* d, cudaStream_t s) {
    const size_t rows = m.rows(), ts = m.tile_size();
    Staging st(rows * ts);
    for (size_t tj = 0; tj < m.grid_cols(); ++tj) {
        const int b = (int)(tj & 1);
        cuda_check(cudaEventSynchronize(st.ev[b]), "staging");  // chunk b's previous copy is done
        size_t tcols = 0;
        for (size_t ti = 0; ti < m.grid_rows(); ++ti) {
            const Tile& t = m.tile(ti, tj);
            tcols = t.cols;
            for (size_t j = 0; j < t.cols; ++j)
                std::memcpy(st.chunk[b] + ti * ts + j * rows, t.data.data() + j * t.rows, t.rows * sizeof(double));
        }
        cuda_check(cudaMemcpyAsync(d + tj * ts * rows, st.chunk[b], rows * tcols * sizeof(double),
                                   cudaMemcpyHostToDevice, s),
                   "H2D");
        cuda_check(cudaEventRecord(st.ev[b], s), "event");
    }
    cuda_check(cudaStreamSynchronize(s), "H2D");
}

// device column-major (ld = rows) -> TiledMatrix
void download(const double* d, TiledMatrix& m, cudaStream_t s) {
    const size_t rows = m.rows(), ts = m.tile_size(), gc = m.grid_cols();
    Staging st(rows * ts);
    auto cols_of = [&](size_t tj) { return m.tile(0, tj).cols; };
    auto fetch = [&](size_t tj) {
        const int b = (int)(tj & 1);
        cuda_check(cudaMemcpyAsync(st.chunk[b], d + tj * ts * rows, rows * cols_of(tj) * sizeof(double),
                                   cudaMemcpyDeviceToHost, s),
                   "D2H");
        cuda_check(cudaEventRecord(st.ev[b], s), "event");
    };
    if (gc) fetch(0);
    for (size_t tj = 0; tj < gc; ++tj) {
        const int b = (int)(tj & 1);
        cuda_check(cudaEventSynchronize(st.ev[b]), "D2H");
        if (tj + 1 < gc) fetch(tj + 1);  // the next block column streams while this one unpacks
        for (size_t ti = 0; ti < m.grid_rows(); ++ti) {
            Tile& t = m.tile(ti, tj);
            for (size_t j = 0; j < t.cols; ++j)
                std::memcpy(t.data.data() + j * t.rows, st.chunk[b] + ti * ts + j * rows, t.rows * sizeof(double));
        }
    }
}

// the matrix (and optional factor) resident on the device for one call
struct DeviceProblem {
    Stream st;
    size_t n;
    DevBuf h, q;
    DeviceProblem(const TiledMatrix& m, const TiledMatrix* f) : n(m.rows()), h(n * n), q(f ? n * n : 0) {
        upload(m, h.p, st.s);
        if (f) upload(*f, q.p, st.s);
    }
    void back(TiledMatrix& m, TiledMatrix* f) {
        download(h.p, m, st.s);
        if (f) download(q.p, *f, st.s);
    }
};

// Multi-GPU from the reference's in-process API: TASKEIG_GPUS=k (the GPU
// counterpart of the reference's TASKEIG_WORKERS, runtime.cpp:251-258) runs
// reorder_schur over min(k, visible GPUs) devices in this process
// (teig_dist_reorder_schur_multi: S column slabs, Q row slabs, NCCL clique);
// the result is bitwise the single-GPU one.  Unset: one GPU.  Problems too
// small for the slab layout (< 256 columns per rank) use fewer ranks.
int gpu_world(size_t n) {
    const char* e = getenv("TASKEIG_GPUS");
    if (!e || atoi(e) <= 0) return 0;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int world = std::min(std::min(atoi(e), ndev), 16);
    while (world > 1 && n < (size_t)256 * world) --world;
    return n >= 256 ? world : 0;
}

void reorder_multi(DeviceProblem& dp, int world, const teig_reorder_opts& o, size_t nb, const uint8_t* sizes,
                   const uint8_t* flags, int64_t* perm, int64_t* rej, int64_t* plan, int64_t cap,
                   teig_reorder_info* info) {
    const int64_t n = (int64_t)dp.n;
    std::vector<int64_t> cb(world + 1), rb(world + 1);
    teig_check(teig_dist_balance(n, (int64_t)nb, sizes, flags, o.window_size, world, cb.data(), rb.data()),
               "reorder_schur (slabs)");
    int cur = 0;
    cuda_check(cudaGetDevice(&cur), "device");
    std::vector<int32_t> devs(world);
    for (int r = 0; r < world; ++r) devs[r] = r;
    std::vector<double*> ss(world, nullptr), qs(world, nullptr);
    struct Free {
        std::vector<double*>& a;
        std::vector<double*>& b;
        ~Free() {
            for (double* p : a)
                if (p) cudaFree(p);
            for (double* p : b)
                if (p) cudaFree(p);
        }
    } release{ss, qs};
    const bool with_q = dp.q.p != nullptr;
    for (int r = 0; r < world; ++r) {  // scatter: S column slabs (+ halo), Q row slabs
        cuda_check(cudaSetDevice(devs[r]), "device");
        const int64_t w = cb[r + 1] - cb[r], h = rb[r + 1] - rb[r];
        cuda_check(cudaMalloc(reinterpret_cast<void**>(&ss[r]), sizeof(double) * n * (w + 128)), "cudaMalloc");
        cuda_check(cudaMemcpy(ss[r], dp.h.p + cb[r] * n, sizeof(double) * n * w, cudaMemcpyDefault), "scatter S");
        if (with_q) {
            cuda_check(cudaMalloc(reinterpret_cast<void**>(&qs[r]), sizeof(double) * std::max<int64_t>(h, 1) * n),
                       "cudaMalloc");
            if (h > 0)
                cuda_check(cudaMemcpy2D(qs[r], h * 8, dp.q.p + rb[r], n * 8, h * 8, n, cudaMemcpyDefault), "scatter Q");
        }
    }
    cuda_check(cudaSetDevice(cur), "device");
    teig_check(teig_dist_reorder_schur_multi(n, world, devs.data(), ss.data(), n, with_q ? qs.data() : nullptr,
                                             cb.data(), rb.data(), (int64_t)nb, sizes, flags, &o, perm, rej, plan, cap,
                                             info),
               "reorder_schur");
    for (int r = 0; r < world; ++r) {  // gather
        const int64_t w = cb[r + 1] - cb[r], h = rb[r + 1] - rb[r];
        cuda_check(cudaMemcpy(dp.h.p + cb[r] * n, ss[r], sizeof(double) * n * w, cudaMemcpyDefault), "gather S");
        if (with_q && h > 0)
            cuda_check(cudaMemcpy2D(dp.q.p + rb[r], n * 8, qs[r], h * 8, h * 8, n, cudaMemcpyDefault), "gather Q");
    }
}

// scan_blocks: diagonal blocks by exact-zero subdiagonal (reorder.cpp:21-43)
std::vector<Selection::Block> scan(const TiledMatrix& s) {
    const size_t n = s.rows();
    std::vector<Selection::Block> out;
    for (size_t i = 0; i < n;) {
        Selection::Block b;
        b.start = i;
        if (i + 1 < n && s.at(i + 1, i) != 0.0) {
            b.size = 2;
            b.eigenvalue = {s.at(i, i), std::sqrt(std::fabs(s.at(i, i + 1))) * std::sqrt(std::fabs(s.at(i + 1, i)))};
            i += 2;
        } else {
            b.size = 1;
            b.eigenvalue = {s.at(i, i), 0.0};
            i += 1;
        }
        out.push_back(b);
    }
    return out;
}

teig_schur_opts schur_opts(const SchurOptions& o, const TiledMatrix& h) {
    teig_schur_opts c;
    teig_schur_opts_default(&c);
    c.deflation = o.deflation == DeflationCondition::norm_stable ? 1 : 0;
    c.shift_count = (int32_t)o.shift_count;
    c.aed_window = (int32_t)o.aed_window;
    c.small_threshold = (int32_t)o.small_threshold;
    c.iteration_limit = (int64_t)o.iteration_limit;
    c.tile_size = (int64_t)std::min<size_t>(h.tile_size(), 128);  // chase window floor (schur.cpp:869)
    return c;
}

}  // namespace

// ---------------------------------------------------------------------------
// reorder.hpp

std::size_t Selection::selected_rows() const {
    std::size_t r = 0;
    for (std::size_t i = 0; i < blocks.size(); ++i)
        if (flags[i]) r += blocks[i].size;
    return r;
}

Selection select_eigenvalues(const TiledMatrix& s, const std::function<bool(std::complex<double>)>& pred) {
    Selection sel;
    sel.blocks = scan(s);
    sel.flags.reserve(sel.blocks.size());
    for (const auto& b : sel.blocks) {
        const bool up = pred(b.eigenvalue);
        if (b.size == 2 && pred(std::conj(b.eigenvalue)) != up)
            throw std::invalid_argument("selection predicate splits a conjugate pair");
        sel.flags.push_back(up);
    }
    return sel;
}

Selection select_eigenvalues(const TiledMatrix& s, const std::vector<bool>& flags) {
    Selection sel;
    sel.blocks = scan(s);
    if (flags.size() != sel.blocks.size()) throw std::invalid_argument("selection flag count must equal block count");
    sel.flags = flags;
    return sel;
}

Selection select_fraction(const TiledMatrix& s, double fraction, std::uint64_t seed) {
    if (fraction < 0.0 || fraction > 1.0) throw std::invalid_argument("selection fraction must be in [0, 1]");
    Selection sel;
    sel.blocks = scan(s);
    std::vector<uint8_t> f(std::max<size_t>(sel.blocks.size(), 1), 0);
    teig_check(teig_select_fraction((int64_t)sel.blocks.size(), fraction, seed, f.data()), "select_fraction");
    sel.flags.assign(sel.blocks.size(), false);
    for (size_t i = 0; i < sel.blocks.size(); ++i) sel.flags[i] = f[i] != 0;
    return sel;
}

Selection select_by_name(const TiledMatrix& s, const std::string& name, std::size_t k) {
    if (name == "left-half-plane") return select_eigenvalues(s, [](std::complex<double> z) { return z.real() < 0.0; });
    if (name == "inside-unit-disk") return select_eigenvalues(s, [](std::complex<double> z) { return std::abs(z) < 1.0; });
    if (name == "largest-magnitude-k") {
        Selection sel;
        sel.blocks = scan(s);
        std::vector<size_t> idx(sel.blocks.size());
        for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
        std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) {
            return std::abs(sel.blocks[a].eigenvalue) > std::abs(sel.blocks[b].eigenvalue);
        });
        sel.flags.assign(sel.blocks.size(), false);
        for (size_t i = 0; i < std::min(k, idx.size()); ++i) sel.flags[idx[i]] = true;
        return sel;
    }
    throw std::invalid_argument("unknown selection predicate: " + name);
}

WindowReorderOutcome window_reorder(DenseMatrix& w, const std::vector<std::size_t>& block_sizes,
                                    const std::vector<bool>& selected, DenseMatrix& acc) {
    const size_t d = w.rows();
    WindowReorderOutcome out;
    acc = DenseMatrix::identity(d);
    const size_t nb = block_sizes.size();
    std::vector<uint8_t> sz(nb), sl(nb);
    size_t rows = 0;
    for (size_t i = 0; i < nb; ++i) {
        rows += block_sizes[i];
        sz[i] = (uint8_t)std::min<size_t>(block_sizes[i], 255);
        sl[i] = i < selected.size() && selected[i] ? 1 : 0;
    }
    // the reference's size check rejects these layouts before any swap
    // (reorder.cpp:132-154); the device kernel needs 1 <= nb <= d as well
    if (nb == 0 || nb > d || rows != d || d == 0) {
        out.executed = false;
        return out;
    }
    for (size_t i = 0; i < nb; ++i)
        if (block_sizes[i] != 1 && block_sizes[i] != 2) {
            out.executed = false;
            return out;
        }
    Stream st;
    DevBuf dw(d * d), da(d * d);
    cuda_check(cudaMemcpyAsync(dw.p, w.data(), d * d * sizeof(double), cudaMemcpyHostToDevice, st.s), "H2D");
    std::vector<uint32_t> order(nb);
    std::vector<uint8_t> stuck(nb);
    int32_t executed = 0;
    teig_check(teig_window_reorder_device((int64_t)d, dw.p, (int64_t)d, (int64_t)nb, sz.data(), sl.data(), da.p,
                                          order.data(), stuck.data(), &executed, st.s),
               "window_reorder");
    out.executed = executed != 0;
    if (!out.executed) return out;
    cuda_check(cudaMemcpyAsync(w.data(), dw.p, d * d * sizeof(double), cudaMemcpyDeviceToHost, st.s), "D2H");
    cuda_check(cudaMemcpyAsync(acc.data(), da.p, d * d * sizeof(double), cudaMemcpyDeviceToHost, st.s), "D2H");
    cuda_check(cudaStreamSynchronize(st.s), "D2H");
    out.order.assign(order.begin(), order.end());
    out.stuck.assign(nb, false);
    for (size_t i = 0; i < nb; ++i) out.stuck[i] = stuck[i] != 0;
    return out;
}

ReorderResult reorder_schur(TiledMatrix s_in, std::optional<TiledMatrix> q_in, const Selection& sel,
                            const ReorderOptions& opts) {
    ReorderResult out{std::move(s_in), std::move(q_in), {}, {}, {}, true};
    TiledMatrix& s = out.s;
    TiledMatrix* q = out.q ? &*out.q : nullptr;
    const size_t n = s.rows();
    if (sel.blocks.size() != sel.flags.size()) throw std::invalid_argument("reorder_schur: malformed selection");
    const size_t nb = sel.blocks.size();
    std::vector<uint8_t> sizes(std::max<size_t>(nb, 1)), flags(std::max<size_t>(nb, 1));
    size_t row = 0;
    for (size_t i = 0; i < nb; ++i) {
        if (sel.blocks[i].start != row) throw std::invalid_argument("reorder_schur: selection does not match s");
        sizes[i] = (uint8_t)sel.blocks[i].size;
        flags[i] = sel.flags[i] ? 1 : 0;
        row += sel.blocks[i].size;
    }
    if (row != n) throw std::invalid_argument("reorder_schur: selection does not match s");
    if (n == 0) return out;
    // window size as the reference picks it (reorder.cpp:221-222); workers and
    // seed are inert (the device path is deterministic: bitwise-identical
    // results for every value, the reference's test_reorder.cpp:202-221)
    teig_reorder_opts o;
    teig_reorder_opts_default(&o);
    o.window_size = (int64_t)std::max<size_t>(opts.window_size ? opts.window_size : s.tile_size(), 8);
    o.strict = opts.strict ? 1 : 0;
    DeviceProblem dp(s, q);
    std::vector<int64_t> perm(std::max<size_t>(nb, 1)), rej(std::max<size_t>(nb, 1));
    const int64_t cap = (int64_t)std::max<size_t>(8 * nb, 1024);
    std::vector<int64_t> plan(3 * cap);
    teig_reorder_info info{};
    const int world = gpu_world(n);
    if (world > 0)
        reorder_multi(dp, world, o, nb, sizes.data(), flags.data(), perm.data(), rej.data(), plan.data(), cap, &info);
    else
        teig_check(teig_reorder_schur_device((int64_t)n, dp.h.p, (int64_t)n, q ? dp.q.p : nullptr, (int64_t)n,
                                             (int64_t)nb, sizes.data(), flags.data(), &o, perm.data(), rej.data(),
                                             plan.data(), cap, &info, dp.st.s),
                   "reorder_schur");
    dp.back(s, q);
    out.permutation.assign(nb, 0);
    for (size_t i = 0; i < nb; ++i) out.permutation[i] = (size_t)perm[i];
    for (int64_t i = 0; i < info.n_rejected; ++i) out.rejected_blocks.push_back((size_t)rej[i]);
    for (int64_t i = 0; i < std::min(info.n_windows, cap); ++i)
        out.plan.push_back({(size_t)plan[3 * i], (size_t)plan[3 * i + 1], (size_t)plan[3 * i + 2]});
    out.clean = info.clean != 0;
    return out;
}

// ---------------------------------------------------------------------------
// schur.hpp

bool deflation_check(double spike_mag, double block_diag_abs_sum, DeflationCondition cond, double window_frob_norm) {
    return teig_deflation_check(spike_mag, block_diag_abs_sum, cond == DeflationCondition::norm_stable ? 1 : 0,
                                window_frob_norm) != 0;
}

AedResult aed_step(TiledMatrix& h, TiledMatrix* q, std::size_t l, std::size_t ihi, std::size_t window,
                   const SchurOptions& opts) {
    if (window < 4) throw std::invalid_argument("aed_step: window must be >= 4");
    const size_t n = h.rows();
    teig_schur_opts o = schur_opts(opts, h);
    DeviceProblem dp(h, q);
    teig_aed_result r{};
    std::vector<double> sh(2 * std::max<size_t>(window, 1));
    teig_check(teig_aed_step_device((int64_t)n, dp.h.p, (int64_t)n, q ? dp.q.p : nullptr, (int64_t)n, (int64_t)l,
                                    (int64_t)ihi, (int64_t)window, &o, &r, sh.data(), dp.st.s),
               "aed_step");
    dp.back(h, q);
    AedResult out;
    out.window = (size_t)r.window;
    out.deflated = (size_t)r.deflated;
    for (int64_t i = 0; i < r.nshifts; ++i) out.shifts.emplace_back(sh[2 * i], sh[2 * i + 1]);
    out.spike_eliminated = r.spike_eliminated != 0;
    out.converged = r.converged != 0;
    out.swap_rejected = r.swap_rejected != 0;
    return out;
}

BulgeChain introduce_bulges(TiledMatrix& h, TiledMatrix* q, std::size_t l, std::size_t ihi,
                            const std::vector<std::complex<double>>& shifts) {
    // the reference's argument checks (schur.cpp:614-626) run first, as there
    if (shifts.size() < 2) throw std::invalid_argument("introduce_bulges: need at least two shifts");
    if (shifts.size() % 2 != 0) throw std::invalid_argument("introduce_bulges: shifts must come in pairs");
    const size_t n = h.rows();
    std::vector<double> sh;
    for (const auto& z : shifts) {
        sh.push_back(z.real());
        sh.push_back(z.imag());
    }
    const size_t nb = shifts.size() / 2;
    std::vector<int64_t> pos(nb);
    DeviceProblem dp(h, q);
    teig_check(teig_introduce_bulges_device((int64_t)n, dp.h.p, (int64_t)n, q ? dp.q.p : nullptr, (int64_t)n,
                                            (int64_t)l, (int64_t)ihi, (int64_t)shifts.size(), sh.data(), pos.data(),
                                            dp.st.s),
               "introduce_bulges");
    dp.back(h, q);
    BulgeChain chain;
    chain.chain_begin = l;
    chain.chain_end = ihi;
    chain.shifts_used = shifts.size();
    for (int64_t p : pos) chain.positions.push_back((size_t)p);  // bottom first (schur.cpp:645)
    return chain;
}

void chase_bulges(TiledMatrix& h, TiledMatrix* q, BulgeChain& chain, std::size_t window_size,
                  const SchurOptions& opts, ChaseTrace* trace) {
    (void)opts;  // workers / seed: inert (deterministic device path)
    if (chain.positions.empty()) return;
    const size_t n = h.rows();
    std::vector<int64_t> pos(chain.positions.begin(), chain.positions.end());
    DeviceProblem dp(h, q);
    int64_t nw = 0;
    teig_check(teig_chase_bulges_device((int64_t)n, dp.h.p, (int64_t)n, q ? dp.q.p : nullptr, (int64_t)n,
                                        (int64_t)chain.chain_end, (int64_t)pos.size(), pos.data(),
                                        (int64_t)window_size, &nw, dp.st.s),
               "chase_bulges");
    dp.back(h, q);
    if (trace) {
        // The executed dependence DAG of the device stream program
        // (schur_driver.cpp): window k -> its left (row-panel) update on the
        // critical-path stream, window k -> window k+1 (overlapping
        // windows, stream order), window k -> its right (column-panel) and
        // factor updates, released onto the second stream by an event.
        std::vector<int64_t> win(3 * std::max<int64_t>(nw, 1));
        const int64_t cnt = teig_plan_chase((int64_t)pos.size(), pos.data(), (int64_t)chain.chain_end,
                                            (int64_t)window_size, win.data(), nw);
        trace->window_tasks.clear();
        trace->edges.clear();
        trace->labels.clear();
        auto add = [&](const std::string& label) {
            trace->labels.push_back(label);
            return trace->labels.size() - 1;
        };
        std::vector<size_t> wid;
        for (int64_t k = 0; k < cnt; ++k) {
            const size_t a = (size_t)win[3 * k], b = a + (size_t)win[3 * k + 1];
            const size_t w = add("schur:chase:W:" + std::to_string(k));
            wid.push_back(w);
            trace->window_tasks.push_back(w);
            if (k > 0) trace->edges.emplace_back(wid[k - 1], w);
            if (b < n) trace->edges.emplace_back(w, add("schur:chase:L:" + std::to_string(k)));
            if (a > 0) trace->edges.emplace_back(w, add("schur:chase:R:" + std::to_string(k)));
            if (q) trace->edges.emplace_back(w, add("schur:chase:Q:" + std::to_string(k)));
        }
    }
    chain.positions.clear();
}

SchurDecomposition schur_reduce(TiledMatrix h_in, std::optional<TiledMatrix> q_in, const SchurOptions& opts) {
    const size_t n = h_in.rows();
    if (h_in.cols() != n) throw std::invalid_argument("schur_reduce: matrix must be square");
    SchurDecomposition out{std::move(h_in), std::move(q_in), {}, 0, true, 0, {}};
    if (n == 0) return out;
    TiledMatrix& h = out.s;
    TiledMatrix* q = out.q ? &*out.q : nullptr;
    teig_schur_opts o = schur_opts(opts, h);
    DeviceProblem dp(h, q);
    std::vector<double> re(n), im(n);
    teig_schur_info info{};
    if (opts.keep_reports) teig_trace_enable(1);
    const int rc = teig_schur_reduce_device((int64_t)n, dp.h.p, (int64_t)n, q ? dp.q.p : nullptr, (int64_t)n, &o,
                                            re.data(), im.data(), &info, dp.st.s);
    if (opts.keep_reports) teig_trace_enable(0);
    teig_check(rc, "schur_reduce");
    dp.back(h, q);
    if (opts.keep_reports) {
        // one ExecutionReport per round (the reference keeps one per round's
        // TaskGraph, schur.hpp:57): the round's kernel launches, worker =
        // stream, device-event times
        const int64_t cnt = teig_trace_task_count();
        char label[128];
        std::string cur;
        for (int64_t i = 0; i < cnt; ++i) {
            int32_t worker = 0;
            int64_t t0 = 0, t1 = 0;
            teig_trace_task(i, label, sizeof label, &worker, &t0, &t1);
            std::string lb(label);
            const std::string round = lb.substr(lb.rfind(':') + 1);
            if (out.round_reports.empty() || round != cur) {
                out.round_reports.emplace_back();
                cur = round;
            }
            out.round_reports.back().tasks.push_back(TaskRecord{lb, (int)worker, t0, t1});
        }
    }
    for (size_t i = 0; i < n; ++i) out.eigenvalues.emplace_back(re[i], im[i]);
    out.sweeps = (size_t)info.sweeps;
    out.converged = info.converged != 0;
    out.converged_trailing = (size_t)info.converged_trailing;
    return out;
}

}  // namespace taskeig
