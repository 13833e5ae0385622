"""Hessenberg reduction on the B200 (csrc/hessenberg.cu) vs the reference's
hessenberg_reduce (hessenberg.cpp:185-280): the same blocked compact-WY
algorithm and reflector convention, so H and Q1 agree entry by entry to
rounding (tolerance 1e-12 ||A||: only the summation orders differ), plus the
backward-error / orthogonality bars (10 n eps), exact zeros below the
subdiagonal, and the reference's golden pipeline fixture (n = 150)."""
import numpy as np
import pytest

from conftest import EPS

pytestmark = pytest.mark.gpu


def _run(T, a_np, **kw):
    import torch
    a = torch.as_tensor(a_np).cuda().t().contiguous().t()
    r = T.hessenberg_reduce(a, True, T.HessenbergOptions(**kw))
    return r.h, r.q, r.info


def _check(T, A, H, Q, n):
    import torch
    At = torch.as_tensor(A).cuda()
    back = float(torch.linalg.norm(At - Q @ H @ Q.t()) / max(float(torch.linalg.norm(At)), 1e-300))
    orth = float(torch.linalg.norm(Q.t() @ Q - torch.eye(n, dtype=torch.float64, device=Q.device)))
    assert back <= 10 * n * EPS and orth <= 10 * n * EPS, (back, orth)
    if n > 2:
        assert float(torch.tril(H, -2).abs().max()) == 0.0


def test_golden_pipeline_n150(T, cuda, golden):
    A = golden["ks150_a"]
    H, Q, _ = _run(T, A)
    n = A.shape[0]
    _check(T, A, H, Q, n)
    scale = np.abs(A).max()
    assert np.abs(H.cpu().numpy() - golden["ks150_h"]).max() <= 1e-12 * scale * n
    assert np.abs(Q.cpu().numpy() - golden["ks150_q"]).max() <= 1e-12 * n


@pytest.mark.parametrize("n,pw", [(1, 0), (2, 0), (3, 0), (5, 0), (40, 0), (150, 0), (257, 16), (500, 0), (1000, 0),
                                  (1300, 64), (1025, 100)])
def test_vs_reference(T, O, cuda, n, pw):
    rng = np.random.default_rng(n)
    A = rng.uniform(-1, 1, (n, n))
    H, Q, info = _run(T, A, panel_width=pw)
    _check(T, A, H, Q, n)
    if O.ref_available() and n <= 1300 and pw in (0,):
        h_ref, q_ref = O.ref_hessenberg_reduce(np.ascontiguousarray(A), workers=0)
        tol = 1e-12 * max(1.0, np.abs(A).max()) * max(1, n) ** 0.5 * 10
        assert np.abs(H.cpu().numpy() - h_ref).max() <= tol
        assert np.abs(Q.cpu().numpy() - q_ref).max() <= tol


def test_feeds_schur_reduce_on_device(T, O, cuda, golden):
    """hessenberg -> schur_reduce without leaving HBM: the known-spectrum
    n = 150 pipeline recovers the true eigenvalues (reference test_schur.cpp
    known-spectrum pipeline, 1e-9)."""
    import torch
    A = golden["ks150_a"]
    n = A.shape[0]
    H, Q, _ = _run(T, A)
    sd = T.schur_reduce(H, Q)
    assert sd.converged
    ev = np.array(sd.eigenvalues)
    assert O.match_spectra(ev, golden["ks150_true"]) <= 1e-9
    At = torch.as_tensor(A).cuda()
    back = float(torch.linalg.norm(At - Q @ H @ Q.t()) / torch.linalg.norm(At))
    assert back <= 10 * n * EPS
