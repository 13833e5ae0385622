"""Rejected swaps on the CPU side: the oracle and the unmodified reference on
the scenarios of tests/rejection_cases.py (no GPU).

* Where the reference's run is well defined (REF_WELL_DEFINED) the oracle
  equals it bit for bit and both produce the analytically predicted
  arrangement (rejection_cases.predicted_permutation) -- the bar the GPU path
  is held to in tests/test_rejection_gpu.py.
* Where the stuck event happens in the middle of a group's window chain
  (REF_LIVELOCKS) the reference's later windows of that chain run on a stale
  selection mask (their size-only layout check passes, reorder.cpp:132-154),
  its block bookkeeping diverges from its matrix, and from then on the same
  window is planned and fails its layout check forever (reorder.cpp:372-395:
  fold breaks, replan, repeat) -- the reference never returns.  The oracle
  restates that behaviour (bounded here by its max_windows guard).  The GPU
  driver instead skips every window planned after a deviation
  (reorder_driver.cpp fold_outcomes) and returns the predicted arrangement."""
import numpy as np
import pytest

import rejection_cases as RC


@pytest.mark.parametrize("name", RC.REF_WELL_DEFINED)
def test_oracle_equals_reference_on_rejections(O, name, golden_rej):
    S, sizes, flags, ws = RC.case(name)
    n = S.shape[0]
    so = S.copy(order="F")
    qo = np.asfortranarray(np.eye(n))
    ro = O.reorder_schur(so, qo, sizes, flags, ws)
    perm, rej = RC.predicted_permutation(S, sizes, flags)
    assert not ro["clean"]
    assert ro["rejected"].tolist() == rej
    assert np.array_equal(ro["permutation"], perm)
    assert np.array_equal(golden_rej[f"{name}_perm"], perm)
    assert golden_rej[f"{name}_rejected"].tolist() == rej
    assert RC.consistent(S, sizes, ro["permutation"], so, O.read_eigenvalues)
    if O.ref_available():
        s_rm = np.ascontiguousarray(S.copy())
        q_rm = np.ascontiguousarray(np.eye(n))
        r = O.ref_reorder_schur(s_rm, q_rm, flags, window_size=ws, workers=1)
        assert np.array_equal(r["permutation"], ro["permutation"])
        assert r["rejected"].tolist() == ro["rejected"].tolist()
        assert np.array_equal(s_rm, so) and np.array_equal(q_rm, qo)  # bitwise


@pytest.mark.parametrize("name", RC.REF_LIVELOCKS)
def test_reference_livelocks_after_midchain_rejection(O, name):
    S, sizes, flags, ws = RC.case(name)
    n = S.shape[0]
    so = S.copy(order="F")
    ro = O.reorder_schur(so, None, sizes, flags, ws, max_windows=1500)
    assert ro["windows_executed"] >= 1500        # never finished
    tail = ro["plan"][-20:]
    assert (tail == tail[0]).all()               # the same window, planned again and again
    _, rej = RC.predicted_permutation(S, sizes, flags)
    assert sorted(ro["rejected"].tolist()) == rej  # the rejections themselves agree


def test_predicted_arrangement_is_consistent(O):
    for name in RC.NAMES:
        S, sizes, flags, _ = RC.case(name)
        perm, rej = RC.predicted_permutation(S, sizes, flags)
        assert sorted(perm.tolist()) == list(range(len(sizes)))
        assert len(rej) == len(RC.twins(S, sizes, flags)) > 0
