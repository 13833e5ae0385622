// tests/refcpp/test_multi_gpu.cpp -- TEST INFRASTRUCTURE: the C++ drop-in's
// multi-GPU path (TASKEIG_GPUS) against its single-GPU path, through the
// reference's own API and types: reorder_schur of the same Schur form with
// TASKEIG_GPUS unset and set must give bitwise-identical S and Q, the same
// permutation, plan and clean flag.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <cstdlib>

#include "taskeig/generate.hpp"
#include "taskeig/hessenberg.hpp"
#include "taskeig/reorder.hpp"
#include "taskeig/schur.hpp"
#include "taskeig/verify.hpp"

using namespace taskeig;

TEST_CASE("TASKEIG_GPUS multi-GPU reorder equals the single-GPU reorder bit for bit") {
    const std::size_t n = 700;
    ProblemSpec spec;
    spec.kind = ProblemKind::known_spectrum;
    spec.n = n;
    spec.seed = 17;
    auto gen = generate(spec);
    const std::size_t ts = default_tile_size(n);
    auto hr = hessenberg_reduce(TiledMatrix::from_dense(gen.a, n, n, ts), true);
    auto sd = schur_reduce(std::move(hr.h), std::move(hr.q));
    REQUIRE(sd.converged);
    const auto d = sd.s.to_dense();
    const auto qd = sd.q->to_dense();
    auto sel = select_fraction(sd.s, 0.35, 99);
    ReorderOptions o;
    o.window_size = 64;
    unsetenv("TASKEIG_GPUS");
    auto r1 = reorder_schur(TiledMatrix::from_dense(d, n, n, ts), TiledMatrix::from_dense(qd, n, n, ts), sel, o);
    setenv("TASKEIG_GPUS", "8", 1);  // as many as visible, at most 8
    auto r2 = reorder_schur(TiledMatrix::from_dense(d, n, n, ts), TiledMatrix::from_dense(qd, n, n, ts), sel, o);
    unsetenv("TASKEIG_GPUS");
    CHECK(r1.clean);
    CHECK(r2.clean);
    CHECK(r1.permutation == r2.permutation);
    CHECK(r1.plan.size() == r2.plan.size());
    CHECK(r1.s.equals_bitwise(r2.s));
    CHECK(r1.q->equals_bitwise(*r2.q));
    CHECK(verify::similarity_residual(gen.a, r2.q->to_dense(), r2.s.to_dense(), n) <= 32.0 * n * 2.220446049250313e-16);
}
