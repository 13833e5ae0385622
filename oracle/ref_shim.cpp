// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNMODIFIED reference library (taskeig, the
// C++20 re-statement of StarNEig in /root/reference/proj), compiled from its
// own sources by oracle/Makefile into oracle/_ref/libtaskeig_ref.so.  Only
// tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline legs
// may load it; the product (paper_2002_05024_b200/) never does.
//
// Dense interchange through this shim is ROW-MAJOR n x n, exactly the
// reference's own `TiledMatrix::from_dense/to_dense` convention
// (tiled_matrix.cpp:37-73).  Window / accumulator buffers of the window-level
// entry points are COLUMN-MAJOR with ld = rows, the `DenseMatrix` convention
// (dense.hpp:18-55).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <vector>

#include "taskeig/dense.hpp"
#include "taskeig/eigvec.hpp"
#include "taskeig/generate.hpp"
#include "taskeig/hessenberg.hpp"
#include "taskeig/kernels.hpp"
#include "taskeig/philox.hpp"
#include "taskeig/reorder.hpp"
#include "taskeig/schur.hpp"
#include "taskeig/tiled_matrix.hpp"
#include "taskeig/verify.hpp"

using namespace taskeig;

namespace {
thread_local std::string g_err;

std::vector<double> vec(const double* p, std::size_t n) { return std::vector<double>(p, p + n); }

DenseMatrix dense_from(const double* p, std::size_t r, std::size_t c) {
    DenseMatrix m(r, c);
    std::memcpy(m.data(), p, sizeof(double) * r * c);
    return m;
}

Selection make_sel(const TiledMatrix& s, const std::uint8_t* flags, std::size_t nb) {
    std::vector<bool> f(nb);
    for (std::size_t i = 0; i < nb; ++i) f[i] = flags[i] != 0;
    return select_eigenvalues(s, f);
}
} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Philox4x32-10 block function (philox.hpp:27-34).
void ref_philox_round10(const std::uint32_t* ctr, const std::uint32_t* key, std::uint32_t* out) {
    auto r = Philox::round10({ctr[0], ctr[1], ctr[2], ctr[3]}, {key[0], key[1]});
    for (int i = 0; i < 4; ++i) out[i] = r[i];
}

// First `count` uniform_sym draws of Philox(seed) (philox.hpp:54-57).
void ref_philox_uniform_sym(std::uint64_t seed, std::size_t count, double* out) {
    Philox p(seed);
    for (std::size_t i = 0; i < count; ++i) out[i] = p.uniform_sym();
}

// generate(ProblemSpec{kind, n, seed}) (generate.cpp:179-233); row-major out.
int ref_generate(int kind, std::size_t n, std::uint64_t seed, double* out) {
    try {
        ProblemSpec spec;
        spec.kind = static_cast<ProblemKind>(kind);
        spec.n = n;
        spec.seed = seed;
        auto g = generate(spec);
        std::memcpy(out, g.a.data(), sizeof(double) * n * n);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// default_spectrum (generate.cpp:68-91): interleaved (re, im) pairs.
void ref_default_spectrum(std::size_t n, std::uint64_t seed, double* out) {
    auto sp = default_spectrum(n, seed);
    for (std::size_t i = 0; i < sp.size(); ++i) {
        out[2 * i] = sp[i].real();
        out[2 * i + 1] = sp[i].imag();
    }
}

// Block scan + select_fraction (reorder.cpp:21-43, 80-97).  Returns #blocks.
long ref_select_fraction(std::size_t n, const double* s_rm, double fraction,
                         std::uint64_t seed, std::size_t* sizes, std::uint8_t* flags) {
    try {
        auto s = TiledMatrix::from_dense(vec(s_rm, n * n), n, n, default_tile_size(n));
        auto sel = select_fraction(s, fraction, seed);
        for (std::size_t i = 0; i < sel.blocks.size(); ++i) {
            sizes[i] = sel.blocks[i].size;
            flags[i] = sel.flags[i] ? 1 : 0;
        }
        return static_cast<long>(sel.blocks.size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// select_by_name (reorder.cpp:99-122).
long ref_select_by_name(std::size_t n, const double* s_rm, const char* name, std::size_t k,
                        std::size_t* sizes, std::uint8_t* flags) {
    try {
        auto s = TiledMatrix::from_dense(vec(s_rm, n * n), n, n, default_tile_size(n));
        auto sel = select_by_name(s, name, k);
        for (std::size_t i = 0; i < sel.blocks.size(); ++i) {
            sizes[i] = sel.blocks[i].size;
            flags[i] = sel.flags[i] ? 1 : 0;
        }
        return static_cast<long>(sel.blocks.size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// standardize_2x2 (kernels.cpp:126-219).  out = {cs, sn, a, b, c, d,
// l1re, l1im, l2re, l2im}.
void ref_standardize_2x2(double a, double b, double c, double d, double* out) {
    auto r = kernels::standardize_2x2(a, b, c, d);
    const double v[10] = {r.rotation.c, r.rotation.s, r.a, r.b, r.c, r.d,
                          r.lambda1.real(), r.lambda1.imag(), r.lambda2.real(), r.lambda2.imag()};
    std::memcpy(out, v, sizeof v);
}

// swap_adjacent_blocks (kernels.cpp:510-631) on a col-major m x m matrix with
// a col-major ar x m accumulator.  Returns 0 ok, 1 rejected.
int ref_swap_adjacent_blocks(std::size_t m, double* s, std::size_t ar, double* acc,
                             std::size_t pos, std::size_t p, std::size_t q) {
    DenseMatrix sm = dense_from(s, m, m), am = dense_from(acc, ar, m);
    auto st = kernels::swap_adjacent_blocks(sm, am, pos, p, q);
    std::memcpy(s, sm.data(), sizeof(double) * m * m);
    std::memcpy(acc, am.data(), sizeof(double) * ar * m);
    return st == kernels::SwapStatus::ok ? 0 : 1;
}

// window_reorder (reorder.cpp:124-194) on a col-major d x d window.
// Returns 1 executed, 0 layout mismatch.  order/stuck sized nb.
int ref_window_reorder(std::size_t d, double* w, std::size_t nb, const std::size_t* sizes,
                       const std::uint8_t* sel, double* acc, std::size_t* order,
                       std::uint8_t* stuck) {
    DenseMatrix wm = dense_from(w, d, d), am;
    std::vector<std::size_t> bs(sizes, sizes + nb);
    std::vector<bool> sv(nb);
    for (std::size_t i = 0; i < nb; ++i) sv[i] = sel[i] != 0;
    auto out = window_reorder(wm, bs, sv, am);
    std::memcpy(w, wm.data(), sizeof(double) * d * d);
    std::memcpy(acc, am.data(), sizeof(double) * d * d);
    if (!out.executed) return 0;
    for (std::size_t i = 0; i < nb; ++i) {
        order[i] = out.order[i];
        stuck[i] = out.stuck[i] ? 1 : 0;
    }
    return 1;
}

// reorder_schur (reorder.cpp:215-404).  s_rm/q_rm are row-major in/out (q may
// be null: no accumulation).  plan receives 3 size_t per executed window
// (position, extent, moved_blocks) up to plan_cap windows; *n_plan the count.
// perm receives one slot per block; rejected (up to nb) the rejected indices.
// Returns 0 on success (clean flag in *clean), -1 on exception.
int ref_reorder_schur(std::size_t n, std::size_t tile, double* s_rm, double* q_rm,
                      std::size_t nb, const std::uint8_t* flags, std::size_t window_size,
                      std::size_t workers, int strict, std::size_t* perm,
                      std::size_t* rejected, std::size_t* n_rejected, std::size_t* plan,
                      std::size_t plan_cap, std::size_t* n_plan, int* clean, double* seconds) {
    try {
        if (!tile) tile = default_tile_size(n);
        auto s = TiledMatrix::from_dense(vec(s_rm, n * n), n, n, tile);
        std::optional<TiledMatrix> q;
        if (q_rm) q = TiledMatrix::from_dense(vec(q_rm, n * n), n, n, tile);
        auto sel = make_sel(s, flags, nb);
        ReorderOptions o;
        o.window_size = window_size;
        o.workers = workers;
        o.strict = strict != 0;
        const auto t0 = std::chrono::steady_clock::now();
        auto res = reorder_schur(std::move(s), std::move(q), sel, o);
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        auto sd = res.s.to_dense();
        std::memcpy(s_rm, sd.data(), sizeof(double) * n * n);
        if (q_rm) {
            auto qd = res.q->to_dense();
            std::memcpy(q_rm, qd.data(), sizeof(double) * n * n);
        }
        for (std::size_t i = 0; i < res.permutation.size(); ++i) perm[i] = res.permutation[i];
        *n_rejected = res.rejected_blocks.size();
        for (std::size_t i = 0; i < res.rejected_blocks.size(); ++i) rejected[i] = res.rejected_blocks[i];
        *n_plan = res.plan.size();
        for (std::size_t i = 0; i < res.plan.size() && i < plan_cap; ++i) {
            plan[3 * i] = res.plan[i].position;
            plan[3 * i + 1] = res.plan[i].extent;
            plan[3 * i + 2] = res.plan[i].moved_blocks;
        }
        *clean = res.clean ? 1 : 0;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// A resident reorder problem for timing (bench.py's reference arm and
// cpu_baseline): the pristine S is converted to a TiledMatrix ONCE, straight
// from a column-major buffer tile by tile (tiles are column-major,
// tiled_matrix.hpp:27-35); every ref_problem_reorder copies it, builds Q = I
// (TiledMatrix::identity) and times reorder_schur alone -- no per-step
// row-major conversions of the n x n inputs and outputs.
struct RefProblem {
    TiledMatrix s0;
    std::size_t n;
};

void* ref_problem_create(std::size_t n, std::size_t tile, const double* s_cm) {
    try {
        if (!tile) tile = default_tile_size(n);
        auto* p = new RefProblem{TiledMatrix(n, n, tile), n};
        for (std::size_t tj = 0; tj < p->s0.grid_cols(); ++tj)
            for (std::size_t ti = 0; ti < p->s0.grid_rows(); ++ti) {
                Tile& t = p->s0.tile(ti, tj);
                const std::size_t r0 = ti * tile, c0 = tj * tile;
                for (std::size_t j = 0; j < t.cols; ++j)
                    std::memcpy(&t.data[j * t.rows], s_cm + r0 + (c0 + j) * n, sizeof(double) * t.rows);
            }
        return p;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_problem_destroy(void* h) { delete static_cast<RefProblem*>(h); }

int ref_problem_reorder(void* h, std::size_t nb, const std::uint8_t* flags, std::size_t window_size,
                        std::size_t workers, int with_q, double* seconds, std::size_t* n_plan, int* clean) {
    try {
        auto* p = static_cast<RefProblem*>(h);
        TiledMatrix s = p->s0;
        std::optional<TiledMatrix> q;
        if (with_q) q = TiledMatrix::identity(p->n, p->s0.tile_size());
        auto sel = make_sel(s, flags, nb);
        ReorderOptions o;
        o.window_size = window_size;
        o.workers = workers;
        const auto t0 = std::chrono::steady_clock::now();
        auto res = reorder_schur(std::move(s), std::move(q), sel, o);
        const auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
        if (n_plan) *n_plan = res.plan.size();
        if (clean) *clean = res.clean ? 1 : 0;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// backtransform (eigvec.cpp:448-516): y_cm n x k column-major (the
// EigenvectorSet's DenseMatrix convention), q_rm row-major, col_kind per
// column; x_cm receives the renormalised X = Q Y.
int ref_backtransform(std::size_t n, std::size_t k, const double* y_cm, const double* q_rm, const int* col_kind,
                      double* x_cm, std::size_t workers) {
    try {
        EigenvectorSet y;
        y.n = n;
        y.lambdas.assign(k, {0.0, 0.0});
        y.col_kind.assign(col_kind, col_kind + k);
        y.positions.assign(k, 0);
        y.flagged.assign(k, false);
        y.columns = dense_from(y_cm, n, k);
        auto q = TiledMatrix::from_dense(vec(q_rm, n * n), n, n, default_tile_size(n));
        EigvecOptions o;
        o.workers = workers;
        auto x = backtransform(y, q, o);
        std::memcpy(x_cm, x.columns.data(), sizeof(double) * n * k);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// hessenberg_reduce (hessenberg.cpp:185-280): a_rm in -> h_rm, q_rm out.
int ref_hessenberg_reduce(std::size_t n, const double* a_rm, double* h_rm, double* q_rm,
                          std::size_t workers) {
    try {
        HessenbergOptions o;
        o.workers = workers;
        auto r = hessenberg_reduce(TiledMatrix::from_dense(vec(a_rm, n * n), n, n,
                                                           default_tile_size(n)),
                                   true, o);
        auto hd = r.h.to_dense();
        auto qd = r.q->to_dense();
        std::memcpy(h_rm, hd.data(), sizeof(double) * n * n);
        std::memcpy(q_rm, qd.data(), sizeof(double) * n * n);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// schur_reduce (schur.cpp:671-906).  h_rm in/out (-> S), q_rm in/out (may be
// null).  eig receives n (re, im) pairs when converged.  info = {sweeps,
// converged, converged_trailing}.
int ref_schur_reduce(std::size_t n, std::size_t tile, double* h_rm, double* q_rm,
                     std::size_t workers, int deflation, std::size_t shift_count,
                     std::size_t aed_window, std::size_t iteration_limit,
                     std::size_t small_threshold, double* eig, std::size_t* info,
                     double* seconds) {
    try {
        if (!tile) tile = default_tile_size(n);
        auto h = TiledMatrix::from_dense(vec(h_rm, n * n), n, n, tile);
        std::optional<TiledMatrix> q;
        if (q_rm) q = TiledMatrix::from_dense(vec(q_rm, n * n), n, n, tile);
        SchurOptions o;
        o.deflation = deflation ? DeflationCondition::norm_stable : DeflationCondition::classic;
        o.shift_count = shift_count;
        o.aed_window = aed_window;
        o.iteration_limit = iteration_limit;
        if (small_threshold) o.small_threshold = small_threshold;
        o.workers = workers;
        const auto t0 = std::chrono::steady_clock::now();
        auto sd = schur_reduce(std::move(h), std::move(q), o);
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        auto s = sd.s.to_dense();
        std::memcpy(h_rm, s.data(), sizeof(double) * n * n);
        if (q_rm) {
            auto qd = sd.q->to_dense();
            std::memcpy(q_rm, qd.data(), sizeof(double) * n * n);
        }
        for (std::size_t i = 0; i < sd.eigenvalues.size(); ++i) {
            eig[2 * i] = sd.eigenvalues[i].real();
            eig[2 * i + 1] = sd.eigenvalues[i].imag();
        }
        info[0] = sd.sweeps;
        info[1] = sd.converged ? 1 : 0;
        info[2] = sd.converged_trailing;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// small_schur (kernels.cpp:260-381) on a col-major k x k Hessenberg matrix.
int ref_small_schur(std::size_t k, double* h, double* q, std::size_t* sweeps) {
    DenseMatrix hm = dense_from(h, k, k), qm;
    auto r = kernels::small_schur(hm, qm);
    std::memcpy(h, hm.data(), sizeof(double) * k * k);
    std::memcpy(q, qm.data(), sizeof(double) * k * k);
    *sweeps = r.sweeps;
    return r.converged ? 1 : 0;
}

// aed_step (schur.cpp:599-609) on a full row-major n x n h (q may be null).
// out: {window, deflated, spike_eliminated, converged, swap_rejected, nshifts};
// shifts: (re, im) pairs.
int ref_aed_step(std::size_t n, std::size_t tile, double* h_rm, double* q_rm, std::size_t l,
                 std::size_t ihi, std::size_t window, int deflation, std::size_t* out,
                 double* shifts) {
    try {
        if (!tile) tile = default_tile_size(n);
        auto h = TiledMatrix::from_dense(vec(h_rm, n * n), n, n, tile);
        std::optional<TiledMatrix> q;
        if (q_rm) q = TiledMatrix::from_dense(vec(q_rm, n * n), n, n, tile);
        SchurOptions o;
        o.deflation = deflation ? DeflationCondition::norm_stable : DeflationCondition::classic;
        o.workers = 1;
        auto r = aed_step(h, q ? &*q : nullptr, l, ihi, window, o);
        auto hd = h.to_dense();
        std::memcpy(h_rm, hd.data(), sizeof(double) * n * n);
        if (q_rm) {
            auto qd = q->to_dense();
            std::memcpy(q_rm, qd.data(), sizeof(double) * n * n);
        }
        out[0] = r.window;
        out[1] = r.deflated;
        out[2] = r.spike_eliminated;
        out[3] = r.converged;
        out[4] = r.swap_rejected;
        out[5] = r.shifts.size();
        for (std::size_t i = 0; i < r.shifts.size(); ++i) {
            shifts[2 * i] = r.shifts[i].real();
            shifts[2 * i + 1] = r.shifts[i].imag();
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// introduce_bulges + chase_bulges (schur.cpp:611-669): one full windowed
// multishift sweep.  shifts: nshifts (re, im) pairs.
int ref_sweep(std::size_t n, std::size_t tile, double* h_rm, double* q_rm, std::size_t l,
              std::size_t ihi, std::size_t nshifts, const double* shifts,
              std::size_t window_size) {
    try {
        if (!tile) tile = default_tile_size(n);
        auto h = TiledMatrix::from_dense(vec(h_rm, n * n), n, n, tile);
        std::optional<TiledMatrix> q;
        if (q_rm) q = TiledMatrix::from_dense(vec(q_rm, n * n), n, n, tile);
        std::vector<std::complex<double>> sh;
        for (std::size_t i = 0; i < nshifts; ++i) sh.emplace_back(shifts[2 * i], shifts[2 * i + 1]);
        auto chain = introduce_bulges(h, q ? &*q : nullptr, l, ihi, sh);
        SchurOptions o;
        o.workers = 1;
        chase_bulges(h, q ? &*q : nullptr, chain, window_size, o);
        auto hd = h.to_dense();
        std::memcpy(h_rm, hd.data(), sizeof(double) * n * n);
        if (q_rm) {
            auto qd = q->to_dense();
            std::memcpy(q_rm, qd.data(), sizeof(double) * n * n);
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// verify.cpp oracles (row-major).
double ref_similarity_residual(std::size_t n, const double* a, const double* q, const double* s) {
    return verify::similarity_residual(vec(a, n * n), vec(q, n * n), vec(s, n * n), n);
}
double ref_orthogonality_defect(std::size_t n, const double* q) {
    return verify::orthogonality_defect(vec(q, n * n), n);
}
int ref_is_standardized(std::size_t n, const double* s) {
    return verify::is_standardized_quasi_triangular(vec(s, n * n), n) ? 1 : 0;
}

} // extern "C"
