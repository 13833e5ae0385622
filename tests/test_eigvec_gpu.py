"""Eigenvector back-transformation X = Q Y (reference eigvec.cpp:448-516) on
the DMMA GEMM kernel + renormalisation (csrc/backtransform.cu), through the C
ABI: against the reference's own backtransform (golden fixture and, where
oracle/_ref travelled, live), and against an independent fp64 GEMM (torch /
cuBLAS) with the renormalisation restated in numpy, for odd shapes and
leading dimensions.  Tolerance: |x| <= 1 after renormalisation, each entry a
length-n dot product summed in another order -> 4 n eps."""
import numpy as np
import pytest

from conftest import EPS

pytestmark = pytest.mark.gpu


def renorm_np(x, kind):
    """eigvec.cpp:494-512 restated."""
    x = x.copy()
    n, k = x.shape
    j = 0
    for j in range(k):
        if kind[j] == 2:
            continue
        cols = [j, j + 1] if kind[j] == 1 else [j]
        m = np.abs(x[:, cols]).max(axis=1)
        nrm = m.max()
        if nrm == 0.0:
            continue
        arg = int(np.argmax(m))  # first index attaining the maximum
        lead = x[arg, j]
        if kind[j] == 1 and abs(x[arg, j + 1]) > abs(lead):
            lead = x[arg, j + 1]
        x[:, cols] *= (-1.0 if lead < 0 else 1.0) / nrm
    return x


def test_backtransform_equals_reference_golden(T, cuda, golden_r2):
    import torch
    y = torch.as_tensor(golden_r2["bt_y"]).cuda()
    q = torch.as_tensor(golden_r2["bt_q"]).cuda()
    kind = golden_r2["bt_kind"]
    x = T.backtransform(y, q, list(kind)).cpu().numpy()
    want = golden_r2["bt_x"]
    n = y.shape[0]
    assert np.max(np.abs(x - want)) <= 4 * n * EPS


@pytest.mark.parametrize("n,k", [(1, 1), (7, 3), (130, 1), (300, 41), (1000, 129), (2049, 64)])
def test_backtransform_vs_gemm(T, O, cuda, n, k):
    import torch
    g = torch.Generator().manual_seed(n * 1000 + k)
    q, _ = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, generator=g))
    y = torch.rand(n, k, dtype=torch.float64, generator=g) * 2 - 1
    kind = np.zeros(k, dtype=np.int8)
    for j in range(1, k - 1, 4):
        kind[j], kind[j + 1] = 1, 2
    # odd leading dimensions: views into padded buffers
    qd = torch.empty((n, n + 1), dtype=torch.float64, device=cuda).t()[:n, :]
    qd.copy_(q)
    yd = torch.empty((k, n + 5), dtype=torch.float64, device=cuda).t()[:n, :]
    yd.copy_(y)
    x = T.backtransform(yd, qd, list(kind)).cpu().numpy()
    want = renorm_np((q @ y).numpy(), kind)
    assert np.max(np.abs(x - want)) <= 4 * n * EPS
    raw = T.backtransform(yd, qd, None).cpu().numpy()  # no renormalisation: the GEMM alone
    ref = (q @ y).numpy()
    assert np.max(np.abs(raw - ref)) <= 4 * n * EPS * max(1.0, np.abs(ref).max())
    if O.ref_available() and n <= 1000:
        xr = O.ref_backtransform(y.numpy(), q.numpy(), kind.astype(np.int32), workers=1)
        assert np.max(np.abs(x - xr)) <= 4 * n * EPS


def test_backtransform_chains_on_the_device_q(T, O, cuda):
    """Zero-copy chaining: the Q a reorder_schur left in HBM feeds the
    back-transformation directly; for the reordered form's leading
    eigenvectors the result equals the transformed input eigenvectors
    (S Q = Q S_new: x = Q y solves S_in x = lambda x when S_new y = lambda y)."""
    import torch
    n = 600
    s0 = T.gen_schur_input(n, T.known_spectrum_seed(4))
    s = s0.clone()
    q = T.identity(n)
    sel = T.select_fraction(s, 0.35, 3)
    r = T.reorder_schur(s, q, sel, T.ReorderOptions(window_size=64))
    assert r.clean
    # the leading 1x1 block's eigenvector of S_new is e_1
    assert float(s[1, 0]) == 0.0
    y = torch.zeros(n, 1, dtype=torch.float64, device=cuda)
    y[0, 0] = 1.0
    x = T.backtransform(y, q, [0])
    lam = float(s[0, 0])
    resid = float(torch.linalg.norm(s0 @ x - lam * x))
    assert resid <= 10 * n * EPS * float(torch.linalg.norm(s0))


def test_backtransform_errors(T, cuda):
    import torch
    q = torch.eye(5, dtype=torch.float64, device=cuda)
    with pytest.raises(ValueError):
        T.backtransform(torch.zeros(4, 2, dtype=torch.float64, device=cuda), q)
    y = torch.zeros(5, 2, dtype=torch.float64, device=cuda)
    y[0, 0] = float("nan")
    with pytest.raises(T.TaskeigError):
        T.backtransform(y, q, [0, 0])
