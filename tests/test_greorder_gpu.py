"""Generalized Schur-pair reordering (S, T) with Q and Z (SURVEY.md 8a a16,
config C5) on the GPU.  The reference has no generalized path; the external
oracle is LAPACK DTGSEN (scipy 1.18.1, scipy-openblas 0.3.31.dev) on the same
input: the same selected-first / relative-order semantics, so the
generalized eigenvalues must agree position by position.

Bars: backward errors ||S_in - Q S Z^T||_F/||S_in||_F, ||T_in - Q T Z^T||_F/||T_in||_F
and orthogonality of Q and Z <= 10 n eps; eigenvalues (alpha/beta) equal to
LAPACK's in diagonal order to relative 1e-10; the selected multiset leads;
T upper triangular, S upper quasi-triangular with the same block count."""
import numpy as np
import pytest

from conftest import EPS

pytestmark = pytest.mark.gpu

TOL_EIG = 1e-10


def _problem(T, O, n, seed_t=7, frac=0.35, sel_seed=99):
    import torch
    s = T.gen_schur_input(n, T.known_spectrum_seed(1))
    t = T.gen_pair_t(n, seed_t)
    sel = T.select_fraction(s, frac, sel_seed)
    return s, t, sel


def _rows(sel, n):
    rows = np.zeros(n, dtype=np.int32)
    for b, f in zip(sel.blocks, sel.flags):
        if f:
            rows[b.start:b.start + b.size] = 1
    return rows


def _check(O, n, S0, T0, S, Tm, Q, Z, sel, ev_ref):
    import torch
    dev = S.device
    back_s = float(torch.linalg.norm(S0 - Q @ S @ Z.t()) / torch.linalg.norm(S0))
    back_t = float(torch.linalg.norm(T0 - Q @ Tm @ Z.t()) / torch.linalg.norm(T0))
    I = torch.eye(n, dtype=torch.float64, device=dev)
    oq = float(torch.linalg.norm(Q.t() @ Q - I))
    oz = float(torch.linalg.norm(Z.t() @ Z - I))
    tol = 10 * n * EPS
    assert back_s <= tol and back_t <= tol and oq <= tol and oz <= tol, (back_s, back_t, oq, oz)
    s, t = S.cpu().numpy(), Tm.cpu().numpy()
    assert np.all(np.tril(t, -1) == 0.0)
    assert np.all(np.tril(s, -2) == 0.0)
    ev = O.pencil_eigenvalues(s, t)
    assert np.all(np.abs(ev - ev_ref) <= TOL_EIG * np.maximum(1.0, np.abs(ev_ref))), np.abs(ev - ev_ref).max()
    e_in = O.pencil_eigenvalues(S0.cpu().numpy(), T0.cpu().numpy())
    want = np.concatenate([e_in[b.start:b.start + b.size] for b, f in zip(sel.blocks, sel.flags) if f] or [[]])
    assert O.match_spectra(ev[:len(want)], want) <= TOL_EIG * max(1.0, np.abs(want).max(initial=1.0))


@pytest.mark.parametrize("n,ws", [(60, 16), (300, 32), (800, 64), (2000, 64)])
def test_greorder_vs_lapack_dtgsen(T, O, cuda, n, ws):
    S0, T0, sel = _problem(T, O, n)
    S, Tm, Q, Z = S0.clone(), T0.clone(), T.identity(n), T.identity(n)
    res = T.greorder_schur(S, Tm, Q, Z, sel, T.ReorderOptions(window_size=ws))
    assert res.clean
    _, _, _, _, ev_ref = O.lapack_tgsen(S0.cpu().numpy(), T0.cpu().numpy(), _rows(sel, n))
    _check(O, n, S0, T0, S, Tm, Q, Z, sel, ev_ref)


def test_greorder_host_entry_and_no_factors(T, O, cuda):
    n = 400
    S0, T0, sel = _problem(T, O, n, seed_t=3, frac=0.5, sel_seed=5)
    r = T.greorder_schur(S0.cpu().numpy(), T0.cpu().numpy(), np.eye(n), np.eye(n), sel,
                         T.ReorderOptions(window_size=32))
    assert r.clean
    _, _, _, _, ev_ref = O.lapack_tgsen(S0.cpu().numpy(), T0.cpu().numpy(), _rows(sel, n))
    import torch
    as_t = lambda a: torch.as_tensor(np.ascontiguousarray(a)).cuda()
    _check(O, n, S0, T0, as_t(r.s), as_t(r.t), as_t(r.q), as_t(r.z), sel, ev_ref)
    S2, T2 = S0.clone(), T0.clone()
    T.greorder_schur(S2, T2, None, None, sel, T.ReorderOptions(window_size=32))
    assert torch.equal(S2, as_t(r.s)) and torch.equal(T2, as_t(r.t))


def test_generator_matches_oracle(T, O, cuda):
    n = 333
    assert np.array_equal(T.gen_pair_t(n, 11).cpu().numpy(), O.pair_t(n, 11))


def test_empty_and_full_selection_are_noops(T, O, cuda):
    import torch
    n = 100
    S0, T0, sel = _problem(T, O, n)
    for flag in (False, True):
        sel2 = T.Selection(sel.blocks, [flag] * len(sel.blocks))
        S, Tm = S0.clone(), T0.clone()
        res = T.greorder_schur(S, Tm, None, None, sel2)
        assert res.clean and res.info["n_windows"] == 0
        assert torch.equal(S, S0) and torch.equal(Tm, T0)
