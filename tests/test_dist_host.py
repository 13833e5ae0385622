"""Host-side logic of the multi-GPU reorder on CPU: slab
balancing, the communication schedule, and the NCCL-id exchange over a real
world_size-2 torch.distributed (gloo) group -- the plumbing the NCCL path
uses, exercised without GPUs."""
import os
import socket

import numpy as np
import pytest


def _selection(T, O, n, seed=99, frac=0.35):
    if n <= 12000:
        s = O.schur_input(n, O.known_spectrum_seed(1))
        sizes = O.scan_blocks(s)
    else:  # the synthetic input's block pattern: reals first, then 2x2 blocks
        npairs = n // 4
        sizes = np.array([1] * (n - 2 * npairs) + [2] * npairs, dtype=np.uint8)
    flags = O.select_fraction(len(sizes), frac, seed)
    starts = np.concatenate([[0], np.cumsum(sizes)])
    blocks = [T.Block(int(starts[i]), int(sizes[i]), 0j) for i in range(len(sizes))]
    return T.Selection(blocks, [bool(f) for f in flags])


def _work_profile(T, n, sel, ws):
    win, _, _, _ = T.plan_reorder(n, sel, ws)
    a, b = win[:, 0], win[:, 1]
    d = (b - a).astype(float)
    prof = np.zeros(n + 1)
    np.add.at(prof, b, 2 * d * d)
    dens = np.cumsum(prof)[:n]
    r = np.zeros(n + 1)
    np.add.at(r, a, 2 * d * a)
    np.add.at(r, b, -2 * d * a)
    return dens + np.cumsum(r)[:n], win


@pytest.mark.parametrize("n,world", [(2000, 2), (4000, 4), (10000, 8), (40000, 8)])
def test_balance_equalizes_slab_work(T, O, n, world):
    from paper_2002_05024_b200 import dist as D
    sel = _selection(T, O, n)
    cb, rb = D.balance(n, sel, world, 128)
    assert cb[0] == 0 and cb[-1] == n and np.all(np.diff(cb) >= 256)
    assert rb[0] == 0 and rb[-1] == n and np.all(np.diff(rb) >= 0)
    dens, _ = _work_profile(T, n, sel, 128)
    cw = np.concatenate([[0], np.cumsum(dens)])
    loads = np.array([cw[cb[g + 1]] - cw[cb[g]] for g in range(world)])
    assert loads.max() / loads.mean() <= 1.05


@pytest.mark.parametrize("n,world", [(2000, 2), (10000, 4), (40000, 8)])
def test_schedule_matches_straddling_windows(T, O, n, world):
    from paper_2002_05024_b200 import dist as D
    sel = _selection(T, O, n)
    cb, _ = D.balance(n, sel, world, 128)
    sch = D.schedule(n, sel, world, cb, 128)
    _, win = _work_profile(T, n, sel, 128)
    a, b = win[:, 0], win[:, 1]
    straddles = sum(int(np.sum((a < c) & (b > c))) for c in cb[1:-1])
    # every straddling window: window halo in + halo back (+ panel halo in when a > 0)
    assert np.sum(sch[:, 1] == 0) == straddles and np.sum(sch[:, 1] == 2) == straddles
    for lv, ph, src, dst, r0, r1, c0, c1 in sch:
        assert abs(src - dst) == 1 and c0 == cb[max(src, dst)] and 0 < c1 - c0 < 128
        if ph == 2:
            assert src == dst - 1 and r0 == 0
        else:
            assert src == dst + 1


def _worker(rank, world, port, n, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import paper_2002_05024_b200 as T
        from paper_2002_05024_b200 import dist as D
        from oracle import oracle as O
        sel = _selection(T, O, n)
        obj = [D.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        cb, rb = D.balance(n, sel, world, 128)
        sch = D.schedule(n, sel, world, cb, 128)
        got = [None] * world
        dist.all_gather_object(got, (obj[0], cb.tolist(), rb.tolist(), sch.tolist()))
        q.put((rank, all(g == got[0] for g in got), len(obj[0]), len(sch)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_agrees_on_layout_and_nccl_id():
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 3000, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[1] for r in res) and all(r[2] == 128 for r in res)
