"""Multi-GPU Schur-form reordering over the C ABI
(include/taskeig_b200.h, csrc/dist_reorder.cpp).

S lives in COLUMN SLABS (rank r owns columns [C[r], C[r+1]) plus a 128-column
halo), Q in ROW SLABS (rank r owns rows [R[r], R[r+1])).  Every wavefront's
accumulators are published by their owners (one grouped NCCL broadcast per
owner); windows straddling a slab boundary move their missing columns point
to point.  One process per GPU (``reorder_schur_dist`` with an NCCL
communicator from ``nccl_comm``), all ranks in one process on one GPU each
(``reorder_schur_multi``, ncclCommInitAll), or -- for tests on a single GPU
-- all ranks in one process on one device (``reorder_schur_loopback``).
The distributed result is bitwise identical to ``reorder_schur``.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N
from .reorder import ReorderOptions, ReorderResult, Selection, _stream_ptr

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None

HALO = 128


def _vp(a):
    return a.ctypes.data_as(C.c_void_p)


def balance(n: int, sel: Selection, world: int, window_size: int = 0):
    """Column slabs with equal left+right update flops (from the plan) and
    equal Q row slabs.  Returns (col_bounds, row_bounds), each world+1 long."""
    cb = np.zeros(world + 1, dtype=np.int64)
    rb = np.zeros(world + 1, dtype=np.int64)
    sizes, flags = sel.sizes_array(), sel.flags_array()
    N.check(N.lib().teig_dist_balance(n, len(sizes), _vp(sizes), _vp(flags), window_size, world, _vp(cb), _vp(rb)))
    return cb, rb


def schedule(n: int, sel: Selection, world: int, col_bounds, window_size: int = 0) -> np.ndarray:
    """Host-side communication schedule of the first pass (no device work):
    rows (level, phase, src, dst, r0, r1, c0, c1), phase 0 = window halo in,
    1 = panel halo in, 2 = halo back."""
    sizes, flags = sel.sizes_array(), sel.flags_array()
    cb = np.ascontiguousarray(col_bounds, dtype=np.int64)
    cap = 1024
    while True:
        out = np.zeros(8 * cap, dtype=np.int64)
        k = N.check(N.lib().teig_dist_schedule(n, len(sizes), _vp(sizes), _vp(flags), window_size, world, _vp(cb),
                                               _vp(out), cap))
        if k <= cap:
            return out[:8 * k].reshape(k, 8)
        cap = k


def nccl_available() -> bool:
    return bool(N.lib().teig_nccl_available())


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    N.check(N.lib().teig_nccl_unique_id(buf))
    return bytes(buf)


def nccl_comm(rank: int, world: int, group=None):
    """An NCCL communicator of the library's own (rank 0 creates the unique id,
    torch.distributed broadcasts it -- gloo or nccl backend)."""
    import torch.distributed as dist
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    uid = (C.c_uint8 * 128)(*obj[0])
    comm = C.c_void_p()
    N.check(N.lib().teig_nccl_comm_init(world, rank, uid, C.byref(comm)))
    return comm


def nccl_comm_destroy(comm) -> None:
    N.lib().teig_nccl_comm_destroy(comm)


def s_slab_empty(n: int, c0: int, c1: int, device="cuda"):
    """Column slab of S (n rows x (c1-c0) + halo columns), column-major, ld n."""
    return torch.empty((c1 - c0 + HALO, n), dtype=torch.float64, device=device).t()


def q_slab_empty(n: int, r0: int, r1: int, device="cuda"):
    """Row slab of Q ((r1-r0) rows x n), column-major, ld r1-r0."""
    return torch.empty((n, max(r1 - r0, 1)), dtype=torch.float64, device=device).t()[: r1 - r0]


def gen_schur_input_slab(n: int, fill_seed: int, c0: int, c1: int, device="cuda", stream=None):
    """Columns [c0, c1) of the SURVEY.md 8d synthetic Schur form, in HBM."""
    t = s_slab_empty(n, c0, c1, device)
    N.check(N.lib().teig_gen_schur_input_cols_device(n, t.data_ptr(), n, c0, c1, int(fill_seed) & (2**64 - 1),
                                                     _stream_ptr(stream, t)))
    return t


def identity_rows_slab(n: int, r0: int, r1: int, device="cuda", stream=None):
    t = q_slab_empty(n, r0, r1, device)
    if r1 > r0:
        N.check(N.lib().teig_set_identity_rows_device(n, t.data_ptr(), max(r1 - r0, 1), r0, r1,
                                                      _stream_ptr(stream, t)))
    return t


def _opts(opts: Optional[ReorderOptions]) -> N.ReorderOpts:
    opts = opts or ReorderOptions()
    o = N.ReorderOpts()
    N.lib().teig_reorder_opts_default(C.byref(o))
    o.window_size = int(opts.window_size)
    o.strict = int(bool(opts.strict))
    return o


def _call(n, world, rank, comm, s_slabs, q_slabs, cb, rb, sel, opts, stream_t):
    nb = len(sel.blocks)
    sizes, flags = sel.sizes_array(), sel.flags_array()
    perm = np.zeros(max(nb, 1), dtype=np.int64)
    rej = np.zeros(max(nb, 1), dtype=np.int64)
    info = N.ReorderInfo()
    sp = (C.c_void_p * len(s_slabs))(*[t.data_ptr() for t in s_slabs])
    qp = (C.c_void_p * len(q_slabs))(*[t.data_ptr() for t in q_slabs]) if q_slabs is not None else None
    cb = np.ascontiguousarray(cb, dtype=np.int64)
    rb = np.ascontiguousarray(rb, dtype=np.int64)
    o = _opts(opts)
    rc = N.lib().teig_dist_reorder_schur(n, world, rank, comm, sp, n, qp, _vp(cb), _vp(rb), nb, _vp(sizes),
                                         _vp(flags), C.byref(o), _vp(perm), _vp(rej), C.byref(info),
                                         _stream_ptr(None, stream_t))
    if rc == -1002:
        raise RuntimeError("reorder_schur: swap rejected in strict mode")
    N.check(rc)
    inf = {f: getattr(info, f) for f, _ in N.ReorderInfo._fields_ if f != "pad"}
    return [int(x) for x in perm[:nb]], [int(x) for x in rej[:info.n_rejected]], bool(info.clean), inf


def reorder_schur_dist(s_slab, q_slab, sel: Selection, col_bounds, row_bounds, rank: int, world: int, comm,
                       opts: Optional[ReorderOptions] = None) -> ReorderResult:
    """One rank of the NCCL-distributed reorder (one process per GPU): s_slab
    from ``s_slab_empty``/``gen_schur_input_slab``, q_slab from
    ``q_slab_empty``/``identity_rows_slab`` (or None)."""
    n = s_slab.shape[0]
    perm, rej, clean, inf = _call(n, world, rank, comm, [s_slab], [q_slab] if q_slab is not None else None,
                                  col_bounds, row_bounds, sel, opts, s_slab)
    return ReorderResult(s_slab, q_slab, perm, rej, [], clean, inf)


def reorder_schur_loopback(s, q, sel: Selection, world: int, opts: Optional[ReorderOptions] = None,
                           col_bounds=None, row_bounds=None) -> ReorderResult:
    """All `world` ranks in this process on one device (peer copies instead of
    NCCL): scatters s (and q) into slabs, runs the distributed algorithm,
    gathers the result back into s and q (in place)."""
    n = s.shape[0]
    opts = opts or ReorderOptions()
    if col_bounds is None:
        col_bounds, row_bounds = balance(n, sel, world, opts.window_size)
    cb, rb = list(map(int, col_bounds)), list(map(int, row_bounds))
    ss, qs = [], []
    for r in range(world):
        t = s_slab_empty(n, cb[r], cb[r + 1], s.device)
        t[:, : cb[r + 1] - cb[r]].copy_(s[:, cb[r]:cb[r + 1]])
        ss.append(t)
        if q is not None:
            u = q_slab_empty(n, rb[r], rb[r + 1], s.device)
            if rb[r + 1] > rb[r]:
                u.copy_(q[rb[r]:rb[r + 1], :])
            qs.append(u)
    perm, rej, clean, inf = _call(n, world, 0, None, ss, qs if q is not None else None, cb, rb, sel, opts, s)
    for r in range(world):
        s[:, cb[r]:cb[r + 1]].copy_(ss[r][:, : cb[r + 1] - cb[r]])
        if q is not None and rb[r + 1] > rb[r]:
            q[rb[r]:rb[r + 1], :].copy_(qs[r])
    return ReorderResult(s, q, perm, rej, [], clean, inf)


def reorder_schur_multi(s, q, sel: Selection, devices: Sequence[int], opts: Optional[ReorderOptions] = None,
                        col_bounds=None, row_bounds=None) -> ReorderResult:
    """All ranks in THIS process, rank r on GPU devices[r] (distinct), one
    NCCL clique from ncclCommInitAll (teig_dist_reorder_schur_multi): the
    single-process multi-GPU entry behind the reference's in-process API.
    s (and q) are scattered from their device into slabs on each rank's GPU,
    reordered, and gathered back in place.  Bitwise equal to reorder_schur."""
    n = s.shape[0]
    world = len(devices)
    opts = opts or ReorderOptions()
    if col_bounds is None:
        col_bounds, row_bounds = balance(n, sel, world, opts.window_size)
    cb, rb = list(map(int, col_bounds)), list(map(int, row_bounds))
    ss, qs = [], []
    for r, dev in enumerate(devices):
        d = torch.device("cuda", int(dev))
        t = s_slab_empty(n, cb[r], cb[r + 1], d)
        t[:, : cb[r + 1] - cb[r]].copy_(s[:, cb[r]:cb[r + 1]])
        ss.append(t)
        if q is not None:
            u = q_slab_empty(n, rb[r], rb[r + 1], d)
            if rb[r + 1] > rb[r]:
                u.copy_(q[rb[r]:rb[r + 1], :])
            qs.append(u)
    for dev in devices:
        torch.cuda.synchronize(int(dev))
    nb = len(sel.blocks)
    sizes, flags = sel.sizes_array(), sel.flags_array()
    perm = np.zeros(max(nb, 1), dtype=np.int64)
    rej = np.zeros(max(nb, 1), dtype=np.int64)
    info = N.ReorderInfo()
    sp = (C.c_void_p * world)(*[t.data_ptr() for t in ss])
    qp = (C.c_void_p * world)(*[t.data_ptr() for t in qs]) if q is not None else None
    dv = np.ascontiguousarray(devices, dtype=np.int32)
    cba = np.ascontiguousarray(cb, dtype=np.int64)
    rba = np.ascontiguousarray(rb, dtype=np.int64)
    o = _opts(opts)
    rc = N.lib().teig_dist_reorder_schur_multi(n, world, _vp(dv), sp, n, qp, _vp(cba), _vp(rba), nb, _vp(sizes),
                                               _vp(flags), C.byref(o), _vp(perm), _vp(rej), None, 0, C.byref(info))
    if rc == -1002:
        raise RuntimeError("reorder_schur: swap rejected in strict mode")
    N.check(rc)
    for r in range(world):
        s[:, cb[r]:cb[r + 1]].copy_(ss[r][:, : cb[r + 1] - cb[r]])
        if q is not None and rb[r + 1] > rb[r]:
            q[rb[r]:rb[r + 1], :].copy_(qs[r])
    inf = {f: getattr(info, f) for f, _ in N.ReorderInfo._fields_ if f != "pad"}
    return ReorderResult(s, q, [int(x) for x in perm[:nb]], [int(x) for x in rej[:info.n_rejected]], [],
                         bool(info.clean), inf)


# ---------------------------------------------------------------------------
# generalized pencil (S, T) with Q and Z (config C5) across ranks

def _gcall(n, world, rank, comm, s_slabs, t_slabs, q_slabs, z_slabs, cb, rb, sel, opts, stream_t):
    nb = len(sel.blocks)
    sizes, flags = sel.sizes_array(), sel.flags_array()
    perm = np.zeros(max(nb, 1), dtype=np.int64)
    rej = np.zeros(max(nb, 1), dtype=np.int64)
    info = N.ReorderInfo()
    arr = lambda ts: (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts]) if ts is not None else None
    cb = np.ascontiguousarray(cb, dtype=np.int64)
    rb = np.ascontiguousarray(rb, dtype=np.int64)
    o = _opts(opts)
    rc = N.lib().teig_dist_greorder_schur(n, world, rank, comm, arr(s_slabs), arr(t_slabs), n, arr(q_slabs),
                                          arr(z_slabs), _vp(cb), _vp(rb), nb, _vp(sizes), _vp(flags), C.byref(o),
                                          _vp(perm), _vp(rej), C.byref(info), _stream_ptr(None, stream_t))
    if rc == -1002:
        raise RuntimeError("reorder: swap rejected in strict mode")
    N.check(rc)
    inf = {f: getattr(info, f) for f, _ in N.ReorderInfo._fields_ if f != "pad"}
    return [int(x) for x in perm[:nb]], [int(x) for x in rej[:info.n_rejected]], bool(info.clean), inf


def greorder_schur_dist(s_slab, t_slab, q_slab, z_slab, sel: Selection, col_bounds, row_bounds, rank: int,
                        world: int, comm, opts: Optional[ReorderOptions] = None):
    """One rank of the NCCL-distributed generalized reorder (slabs as for
    reorder_schur_dist; T like S, Z like Q)."""
    n = s_slab.shape[0]
    one = lambda t: [t] if t is not None else None
    return _gcall(n, world, rank, comm, [s_slab], [t_slab], one(q_slab), one(z_slab), col_bounds, row_bounds, sel,
                  opts, s_slab)


def greorder_schur_loopback(s, t, q, z, sel: Selection, world: int, opts: Optional[ReorderOptions] = None,
                            col_bounds=None, row_bounds=None):
    """All ranks of the generalized distributed reorder in this process on one
    device; scatters, runs, gathers back in place.  Returns (perm, rejected,
    clean, info)."""
    n = s.shape[0]
    opts = opts or ReorderOptions(window_size=64)
    if col_bounds is None:
        col_bounds, row_bounds = balance(n, sel, world, opts.window_size or 64)
    cb, rb = list(map(int, col_bounds)), list(map(int, row_bounds))
    ss, ts, qs, zs = [], [], [], []
    for r in range(world):
        for src, dst in ((s, ss), (t, ts)):
            x = s_slab_empty(n, cb[r], cb[r + 1], s.device)
            x[:, : cb[r + 1] - cb[r]].copy_(src[:, cb[r]:cb[r + 1]])
            dst.append(x)
        for src, dst in ((q, qs), (z, zs)):
            if src is None:
                continue
            u = q_slab_empty(n, rb[r], rb[r + 1], s.device)
            if rb[r + 1] > rb[r]:
                u.copy_(src[rb[r]:rb[r + 1], :])
            dst.append(u)
    res = _gcall(n, world, 0, None, ss, ts, qs if q is not None else None, zs if z is not None else None, cb, rb,
                 sel, opts, s)
    for r in range(world):
        s[:, cb[r]:cb[r + 1]].copy_(ss[r][:, : cb[r + 1] - cb[r]])
        t[:, cb[r]:cb[r + 1]].copy_(ts[r][:, : cb[r + 1] - cb[r]])
        if rb[r + 1] > rb[r]:
            if q is not None:
                q[rb[r]:rb[r + 1], :].copy_(qs[r])
            if z is not None:
                z[rb[r]:rb[r + 1], :].copy_(zs[r])
    return res
