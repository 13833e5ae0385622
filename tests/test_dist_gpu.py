"""Multi-GPU reorder on ONE GPU: every rank of the distributed
algorithm runs in this process (loopback communicator: peer copies instead of
NCCL, identical schedule).  The distributed result must equal the single-GPU
result BIT FOR BIT (same kernels, same per-element update order) and meet the
reference parity bars."""
import numpy as np
import pytest

from conftest import EPS

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,world,ws", [(600, 2, 64), (1500, 3, 128), (2500, 4, 128), (4000, 8, 128)])
def test_loopback_equals_single_gpu(T, O, cuda, n, world, ws):
    import torch
    from paper_2002_05024_b200 import dist as D
    s0 = T.gen_schur_input(n, T.known_spectrum_seed(1))
    sel = T.select_fraction(s0, 0.35, 99)
    s1, q1 = s0.clone(), T.identity(n)
    r1 = T.reorder_schur(s1, q1, sel, T.ReorderOptions(window_size=ws))
    s2, q2 = s0.clone(), T.identity(n)
    r2 = D.reorder_schur_loopback(s2, q2, sel, world, T.ReorderOptions(window_size=ws))
    assert r1.clean and r2.clean and r1.permutation == r2.permutation
    assert r2.info["n_windows"] == r1.info["n_windows"]
    assert torch.equal(s1, s2) and torch.equal(q1, q2)
    back = float(torch.linalg.norm(s0 - q2 @ s2 @ q2.t()) / torch.linalg.norm(s0))
    orth = float(torch.linalg.norm(q2.t() @ q2 - torch.eye(n, dtype=torch.float64, device=cuda)))
    assert back <= 10 * n * EPS and orth <= 10 * n * EPS


def test_loopback_without_q_and_uniform_slabs(T, O, cuda):
    import torch
    from paper_2002_05024_b200 import dist as D
    n, world = 1200, 2
    s0 = T.gen_schur_input(n, T.known_spectrum_seed(2))
    sel = T.select_fraction(s0, 0.5, 7)
    s1 = s0.clone()
    T.reorder_schur(s1, None, sel, T.ReorderOptions(window_size=64))
    s2 = s0.clone()
    cb = np.array([0, 600, 1200])
    rb = np.array([0, 600, 1200])
    D.reorder_schur_loopback(s2, None, sel, world, T.ReorderOptions(window_size=64), cb, rb)
    assert torch.equal(s1, s2)


def test_slab_generators_match_full(T, O, cuda):
    import torch
    from paper_2002_05024_b200 import dist as D
    n = 777
    full = T.gen_schur_input(n, T.known_spectrum_seed(1))
    sl = D.gen_schur_input_slab(n, T.known_spectrum_seed(1), 300, 700)
    assert torch.equal(sl[:, :400], full[:, 300:700])
    q = D.identity_rows_slab(n, 100, 350)
    assert torch.equal(q, torch.eye(n, dtype=torch.float64, device=cuda)[100:350])


@pytest.mark.parametrize("n,world", [(800, 2), (1500, 3), (2000, 4)])
def test_generalized_loopback_equals_single_gpu(T, O, cuda, n, world):
    """The C5 pencil across ranks (S, T column slabs; Q, Z row slabs) equals
    the single-GPU generalized reorder bit for bit."""
    import torch
    from paper_2002_05024_b200 import dist as D
    s0 = T.gen_schur_input(n, T.known_spectrum_seed(1))
    t0 = T.gen_pair_t(n, 7)
    sel = T.select_fraction(s0, 0.35, 99)
    opts = T.ReorderOptions(window_size=64)
    s1, t1, q1, z1 = s0.clone(), t0.clone(), T.identity(n), T.identity(n)
    r1 = T.greorder_schur(s1, t1, q1, z1, sel, opts)
    s2, t2, q2, z2 = s0.clone(), t0.clone(), T.identity(n), T.identity(n)
    perm, rej, clean, info = D.greorder_schur_loopback(s2, t2, q2, z2, sel, world, opts)
    assert r1.clean and clean and perm == r1.permutation
    assert torch.equal(s1, s2) and torch.equal(t1, t2) and torch.equal(q1, q2) and torch.equal(z1, z2)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_loopback_rejections_equal_single_gpu(T, O, cuda, world):
    """Rejected swaps across ranks: the deviation flag rides every owner's
    broadcast segment, later levels skip on every rank, the replan pass runs
    distributed -- the result equals the single-GPU driver's bit for bit and
    the predicted arrangement (tests/rejection_cases.py)."""
    import torch
    import rejection_cases as RC
    from paper_2002_05024_b200 import dist as D
    S, sizes, flags, ws = RC.case("wide")
    n = S.shape[0]
    s0 = torch.as_tensor(S).cuda().t().contiguous().t()
    sel = T.select_eigenvalues(s0, [bool(f) for f in flags])
    s1, q1 = s0.clone(), T.identity(n)
    r1 = T.reorder_schur(s1, q1, sel, T.ReorderOptions(window_size=ws))
    s2, q2 = s0.clone(), T.identity(n)
    r2 = D.reorder_schur_loopback(s2, q2, sel, world, T.ReorderOptions(window_size=ws))
    perm, rej = RC.predicted_permutation(S, sizes, flags)
    assert not r1.clean and not r2.clean
    assert r1.permutation == r2.permutation == perm.tolist()
    assert r1.rejected_blocks == r2.rejected_blocks == rej
    assert torch.equal(s1, s2) and torch.equal(q1, q2)


def test_multi_gpu_entry_single_device(T, O, cuda):
    """The single-process multi-GPU entry (teig_dist_reorder_schur_multi:
    per-device stream pairs, NCCL clique from ncclCommInitAll, grouped
    broadcasts) on the one GPU this box has (world 1): equals the single-GPU
    driver bit for bit.  With more GPUs pass more devices."""
    import torch
    from paper_2002_05024_b200 import dist as D
    if not D.nccl_available():
        pytest.skip("libnccl.so.2 not loadable")
    n = 1500
    s0 = T.gen_schur_input(n, T.known_spectrum_seed(6))
    sel = T.select_fraction(s0, 0.35, 4)
    s1, q1 = s0.clone(), T.identity(n)
    r1 = T.reorder_schur(s1, q1, sel, T.ReorderOptions(window_size=128))
    devs = list(range(torch.cuda.device_count()))[:4]
    s2, q2 = s0.clone(), T.identity(n)
    r2 = D.reorder_schur_multi(s2, q2, sel, devs, T.ReorderOptions(window_size=128))
    assert r1.clean and r2.clean and r1.permutation == r2.permutation
    assert torch.equal(s1, s2) and torch.equal(q1, q2)
