"""Rejected swaps on the GPU path (reference reorder.cpp:166-191 stuck blocks,
:372-395 fold/replan), through the C ABI, on the scenarios of
tests/rejection_cases.py: identical 2x2 "twins" whose swap the reference
rejects, planted inside one window, across several groups and in the middle
of a group's window chain.

Bars for every case and window size:
  * the rejected blocks are exactly the selected twins, and the final
    arrangement is the analytically predicted one (selected blocks lead in
    order; each rejected twin sits directly below its unselected twin) --
    the reference's own result wherever its run is well defined (golden
    fixtures from the unmodified reference, tests/golden/rejection_golden.npz);
  * the permutation describes the matrix (positional eigenvalues to 1e-10);
  * backward error and orthogonality <= 10 n eps, standardized form;
  * strict mode raises (reorder.cpp:383-385).
Where the reference livelocks (mid-chain rejection: tests/test_rejection.py)
the GPU driver returns the predicted arrangement."""
import numpy as np
import pytest

import rejection_cases as RC
from conftest import EPS

pytestmark = pytest.mark.gpu


def _run(T, S, sizes, flags, ws, strict=False, overlap=True):
    import torch
    n = S.shape[0]
    s = torch.as_tensor(np.asfortranarray(S)).cuda()
    s = s.t().contiguous().t()  # column-major storage
    q = torch.eye(n, dtype=torch.float64).cuda()
    sel = T.select_eigenvalues(s, [bool(f) for f in flags])
    assert np.array_equal(sel.sizes_array(), sizes)
    r = T.reorder_schur(s, q, sel, T.ReorderOptions(window_size=ws, strict=strict, overlap_factor=overlap))
    return s, q, r


def _check(O, S, sizes, flags, s, q, r):
    import torch
    n = S.shape[0]
    perm, rej = RC.predicted_permutation(S, sizes, flags)
    assert not r.clean
    assert sorted(r.rejected_blocks) == rej
    assert r.permutation == perm.tolist()
    sn = s.cpu().numpy()
    assert RC.consistent(S, sizes, r.permutation, sn, O.read_eigenvalues, tol=1e-10)
    A = torch.as_tensor(S).cuda()
    back = float(torch.linalg.norm(A - q @ s @ q.t()) / torch.linalg.norm(A))
    orth = float(torch.linalg.norm(q.t() @ q - torch.eye(n, dtype=torch.float64, device=q.device)))
    assert back <= 10 * n * EPS and orth <= 10 * n * EPS, (back, orth)
    assert O.is_standardized(sn)
    assert float(torch.tril(s, -2).abs().max()) == 0.0


@pytest.mark.parametrize("name", RC.NAMES)
def test_rejections_match_reference_semantics(T, O, cuda, name):
    S, sizes, flags, ws = RC.case(name)
    s, q, r = _run(T, S, sizes, flags, ws)
    _check(O, S, sizes, flags, s, q, r)
    assert r.info["n_passes"] >= 2  # a deviation forces a replanning pass


@pytest.mark.parametrize("name", RC.REF_WELL_DEFINED)
def test_rejections_equal_reference_golden(T, O, golden_rej, cuda, name):
    S, sizes, flags, ws = RC.case(name)
    assert np.array_equal(golden_rej[f"{name}_S_in"], S)
    s, q, r = _run(T, S, sizes, flags, ws)
    assert r.permutation == golden_rej[f"{name}_perm"].tolist()
    assert r.rejected_blocks == golden_rej[f"{name}_rejected"].tolist()
    assert r.clean == bool(golden_rej[f"{name}_clean"])
    ev = O.read_eigenvalues(s.cpu().numpy())
    er = golden_rej[f"{name}_eig"]
    assert np.all(np.abs(ev - er) <= 1e-10 * np.maximum(1.0, np.abs(er)))


@pytest.mark.parametrize("name", ["multigroup", "midchain", "dense"])
@pytest.mark.parametrize("ws", [16, 48, 96, 128])
def test_rejections_any_window_size(T, O, cuda, name, ws):
    S, sizes, flags, _ = RC.case(name)
    s, q, r = _run(T, S, sizes, flags, ws, overlap=(ws != 48))
    _check(O, S, sizes, flags, s, q, r)


def test_rejection_strict_mode_raises(T, cuda):
    S, sizes, flags, ws = RC.case("multigroup")
    with pytest.raises(RuntimeError):
        _run(T, S, sizes, flags, ws, strict=True)


def test_live_reference_when_available(T, O, cuda):
    """If the compiled reference travelled with the repo (oracle/_ref), compare
    with it live too (well-defined cases)."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    for name in RC.REF_WELL_DEFINED:
        S, sizes, flags, ws = RC.case(name)
        n = S.shape[0]
        s_rm = np.ascontiguousarray(S.copy())
        rr = O.ref_reorder_schur(s_rm, np.ascontiguousarray(np.eye(n)), flags, window_size=ws, workers=1)
        _, _, r = _run(T, S, sizes, flags, ws)
        assert r.permutation == rr["permutation"].tolist()
        assert r.rejected_blocks == rr["rejected"].tolist()
