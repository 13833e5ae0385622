"""Host-side mirror of the reference's reordering API (reorder.hpp:22-89).

Same names, argument meaning and error behaviour as ``taskeig::`` --
``Selection``, ``select_eigenvalues``, ``select_fraction``,
``select_by_name``, ``window_reorder``, ``ReorderOptions``,
``ReorderResult``, ``reorder_schur`` -- over the B200 C ABI.  Matrices are
torch CUDA float64 tensors (device path) or numpy float64 arrays (host path,
host<->device copies inside the call).  Dense matrices are used in their
logical orientation; internally the library works on column-major storage,
the orientation of the reference's tiles (tiled_matrix.hpp:27-35).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Union

import numpy as np

from . import _native as N

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None


# ---------------------------------------------------------------------------
# selections (reorder.cpp:21-122)

@dataclass
class Block:
    start: int
    size: int
    eigenvalue: complex  # +imag representative for a pair


@dataclass
class Selection:
    blocks: List[Block] = field(default_factory=list)
    flags: List[bool] = field(default_factory=list)

    def selected_rows(self) -> int:
        return sum(b.size for b, f in zip(self.blocks, self.flags) if f)

    def sizes_array(self) -> np.ndarray:
        return np.asarray([b.size for b in self.blocks], dtype=np.uint8)

    def flags_array(self) -> np.ndarray:
        return np.asarray(self.flags, dtype=np.uint8)


def _tridiag(s) -> tuple:
    """(diag, super, sub) of s as numpy float64 arrays."""
    if torch is not None and isinstance(s, torch.Tensor):
        d = torch.diagonal(s, 0).double().cpu().numpy()
        up = torch.diagonal(s, 1).double().cpu().numpy()
        lo = torch.diagonal(s, -1).double().cpu().numpy()
        return d, up, lo
    a = np.asarray(s, dtype=np.float64)
    return np.diagonal(a, 0).copy(), np.diagonal(a, 1).copy(), np.diagonal(a, -1).copy()


def scan_blocks(s) -> List[Block]:
    """Exact-zero subdiagonal block scan (reorder.cpp:21-43)."""
    d, up, lo = _tridiag(s)
    n = len(d)
    blocks = []
    i = 0
    while i < n:
        if i + 1 < n and lo[i] != 0.0:
            im = math.sqrt(abs(up[i])) * math.sqrt(abs(lo[i]))
            blocks.append(Block(i, 2, complex(d[i], im)))
            i += 2
        else:
            blocks.append(Block(i, 1, complex(d[i], 0.0)))
            i += 1
    return blocks


def select_eigenvalues(s, pred: Union[Callable[[complex], bool], Sequence[bool]]) -> Selection:
    """Predicate (evaluated on both members of a pair; disagreement raises
    ``ValueError`` like the reference's std::invalid_argument) or explicit
    per-block flags (count must equal the block count)."""
    blocks = scan_blocks(s)
    if callable(pred):
        flags = []
        for b in blocks:
            up = bool(pred(b.eigenvalue))
            if b.size == 2 and bool(pred(b.eigenvalue.conjugate())) != up:
                raise ValueError("selection predicate splits a conjugate pair")
            flags.append(up)
        return Selection(blocks, flags)
    flags = [bool(f) for f in pred]
    if len(flags) != len(blocks):
        raise ValueError("selection flag count must equal block count")
    return Selection(blocks, flags)


def select_fraction(s, fraction: float, seed: int) -> Selection:
    """Exactly floor(fraction * #blocks) blocks by a seeded shuffle
    (reorder.cpp:80-97); same Philox stream as the reference."""
    if fraction < 0.0 or fraction > 1.0:
        raise ValueError("selection fraction must be in [0, 1]")
    blocks = scan_blocks(s)
    flags = np.zeros(max(len(blocks), 1), dtype=np.uint8)
    N.check(N.lib().teig_select_fraction(len(blocks), float(fraction), int(seed) & (2**64 - 1),
                                         flags.ctypes.data_as(C.c_void_p)))
    return Selection(blocks, [bool(x) for x in flags[:len(blocks)]])


def select_by_name(s, name: str, k: int = 0) -> Selection:
    """Named predicates (reorder.cpp:99-122)."""
    if name == "left-half-plane":
        return select_eigenvalues(s, lambda z: z.real < 0.0)
    if name == "inside-unit-disk":
        return select_eigenvalues(s, lambda z: abs(z) < 1.0)
    if name == "largest-magnitude-k":
        blocks = scan_blocks(s)
        idx = sorted(range(len(blocks)), key=lambda i: -abs(blocks[i].eigenvalue))
        flags = [False] * len(blocks)
        for i in idx[:min(k, len(idx))]:
            flags[i] = True
        return Selection(blocks, flags)
    raise ValueError("unknown selection predicate: " + name)


# ---------------------------------------------------------------------------
# window_reorder (reorder.cpp:124-194)

@dataclass
class WindowReorderOutcome:
    executed: bool = True
    order: List[int] = field(default_factory=list)  # order[new_pos] = old local block
    stuck: List[bool] = field(default_factory=list)


def window_reorder(w, block_sizes: Sequence[int], selected: Sequence[bool], stream=None):
    """Runs the single-CTA window kernel on a d x d CUDA tensor ``w`` (in
    place).  Returns ``(outcome, acc)`` with acc the d x d orthogonal factor."""
    _need_torch_cuda(w)
    d = w.shape[0]
    work, ld, copy_back = _as_colmajor(w)
    acc_t = torch.empty((d, d), dtype=torch.float64, device=w.device)  # column-major view below
    nb = len(block_sizes)
    sizes = np.asarray(block_sizes, dtype=np.uint8)
    sel = np.asarray(selected, dtype=np.uint8)
    order = np.zeros(max(nb, 1), dtype=np.uint32)
    stuck = np.zeros(max(nb, 1), dtype=np.uint8)
    ex = C.c_int32(0)
    N.check(N.lib().teig_window_reorder_device(
        d, work.data_ptr(), ld, nb, sizes.ctypes.data_as(C.c_void_p), sel.ctypes.data_as(C.c_void_p),
        acc_t.data_ptr(), order.ctypes.data_as(C.c_void_p), stuck.ctypes.data_as(C.c_void_p),
        C.byref(ex), _stream_ptr(stream, w)))
    if copy_back:
        w.copy_(work)
    acc = acc_t.t()  # buffer holds acc column-major
    out = WindowReorderOutcome(bool(ex.value), [int(x) for x in order[:nb]], [bool(x) for x in stuck[:nb]])
    return out, acc


# ---------------------------------------------------------------------------
# reorder_schur (reorder.cpp:215-404)

@dataclass
class ReorderOptions:
    window_size: int = 0      # 0: tile size rule (reorder.cpp:221-222)
    workers: int = 0          # accepted for API parity; the GPU scheduler ignores it
    seed: int = 0             # accepted for API parity (scheduler perturbation only)
    strict: bool = False      # raise on rejected swaps instead of recording
    overlap_factor: bool = True
    profile: bool = False     # per-kernel-class CUDA-event timing in ReorderResult.info
    full_factor: bool = False  # update Q over all rows (no skipping of its exactly-zero rows)


@dataclass
class PlanWindow:
    position: int
    extent: int
    moved_blocks: int


@dataclass
class ReorderResult:
    s: object
    q: object
    permutation: List[int]
    rejected_blocks: List[int]
    plan: List[PlanWindow]
    clean: bool
    info: dict


def _need_torch_cuda(t):
    if torch is None or not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("expected a CUDA torch tensor")
    if t.dtype != torch.float64:
        raise TypeError("expected float64")


def _stream_ptr(stream, t):
    if stream is None:
        stream = torch.cuda.current_stream(t.device)
    return C.c_void_p(stream.cuda_stream)


def _as_colmajor(t):
    """(work tensor whose storage is column-major, ld, needs_copy_back)."""
    n0, n1 = t.shape
    if t.stride(0) == 1 and t.stride(1) >= max(n0, 1):
        return t, t.stride(1), False
    work = torch.empty((n1, n0), dtype=t.dtype, device=t.device).t()
    work.copy_(t)
    return work, n0, True


def colmajor_empty(n: int, device="cuda"):
    """An n x n float64 CUDA tensor with column-major storage (ld = n)."""
    return torch.empty((n, n), dtype=torch.float64, device=device).t()


def reorder_schur(s, q, sel: Selection, opts: Optional[ReorderOptions] = None,
                  stream=None) -> ReorderResult:
    """Moves every selected eigenvalue to the leading diagonal blocks; q (if
    given) is updated to q * Q3.  CUDA tensors are updated in place when
    they are column-major; numpy arrays go through the host entry point."""
    opts = opts or ReorderOptions()
    if len(sel.blocks) != len(sel.flags):
        raise ValueError("reorder_schur: malformed selection")
    row = 0
    for b in sel.blocks:
        if b.start != row:
            raise ValueError("reorder_schur: selection does not match s")
        row += b.size
    n = s.shape[0]
    if row != n:
        raise ValueError("reorder_schur: selection does not match s")
    nb = len(sel.blocks)
    sizes = sel.sizes_array()
    flags = sel.flags_array()
    perm = np.zeros(max(nb, 1), dtype=np.int64)
    rej = np.zeros(max(nb, 1), dtype=np.int64)
    cap = max(4 * nb, 1024)
    plan = np.zeros(3 * cap, dtype=np.int64)
    info = N.ReorderInfo()
    o = N.ReorderOpts()
    N.lib().teig_reorder_opts_default(C.byref(o))
    o.window_size = int(opts.window_size)
    o.strict = int(bool(opts.strict))
    o.overlap_factor = int(bool(opts.overlap_factor))
    o.profile = int(bool(opts.profile))
    o.full_factor = int(bool(opts.full_factor))
    vp = lambda a: a.ctypes.data_as(C.c_void_p)
    if torch is not None and isinstance(s, torch.Tensor):
        _need_torch_cuda(s)
        sw, lds, cb_s = _as_colmajor(s)
        if q is not None:
            _need_torch_cuda(q)
            qw, ldq, cb_q = _as_colmajor(q)
        else:
            qw, ldq, cb_q = None, n, False
        rc = N.lib().teig_reorder_schur_device(
            n, sw.data_ptr(), lds, qw.data_ptr() if qw is not None else None, ldq, nb, vp(sizes),
            vp(flags), C.byref(o), vp(perm), vp(rej), vp(plan), cap, C.byref(info),
            _stream_ptr(stream, s))
        if rc == -1002:
            raise RuntimeError("reorder_schur: swap rejected in strict mode")
        N.check(rc)
        if cb_s:
            s.copy_(sw)
        if cb_q:
            q.copy_(qw)
        s_out, q_out = s, q
    else:
        sf = np.asfortranarray(np.array(s, dtype=np.float64, copy=True))
        qf = np.asfortranarray(np.array(q, dtype=np.float64, copy=True)) if q is not None else None
        rc = N.lib().teig_reorder_schur_host(
            n, vp(sf), n, vp(qf) if qf is not None else None, n, nb, vp(sizes), vp(flags),
            C.byref(o), vp(perm), vp(rej), vp(plan), cap, C.byref(info), None)
        if rc == -1002:
            raise RuntimeError("reorder_schur: swap rejected in strict mode")
        N.check(rc)
        s_out, q_out = sf, qf
    k = min(info.n_windows, cap)
    pl = [PlanWindow(int(plan[3 * i]), int(plan[3 * i + 1]), int(plan[3 * i + 2])) for i in range(k)]
    inf = {f: getattr(info, f) for f, _ in N.ReorderInfo._fields_ if f != "pad"}
    return ReorderResult(s_out, q_out, [int(x) for x in perm[:nb]],
                         [int(x) for x in rej[:info.n_rejected]], pl, bool(info.clean), inf)


def reorder_schur_host_buffers(s_buf: np.ndarray, q_buf: Optional[np.ndarray], n: int, sel: Selection,
                               opts: Optional[ReorderOptions] = None) -> dict:
    """Reorders HOST buffers holding S and Q COLUMN-MAJOR with ld = n (e.g. a
    C-ordered array of S^T, or pinned memory) in place through the C ABI's
    host entry point; host<->device copies happen inside the call."""
    opts = opts or ReorderOptions()
    assert s_buf.dtype == np.float64 and s_buf.size == n * n and s_buf.flags.contiguous
    nb = len(sel.blocks)
    sizes, flags = sel.sizes_array(), sel.flags_array()
    perm = np.zeros(max(nb, 1), dtype=np.int64)
    rej = np.zeros(max(nb, 1), dtype=np.int64)
    info = N.ReorderInfo()
    o = N.ReorderOpts()
    N.lib().teig_reorder_opts_default(C.byref(o))
    o.window_size = int(opts.window_size)
    o.strict = int(bool(opts.strict))
    o.overlap_factor = int(bool(opts.overlap_factor))
    vp = lambda a: a.ctypes.data_as(C.c_void_p)
    N.check(N.lib().teig_reorder_schur_host(n, vp(s_buf), n, vp(q_buf) if q_buf is not None else None, n, nb,
                                            vp(sizes), vp(flags), C.byref(o), vp(perm), vp(rej), None, 0,
                                            C.byref(info), None))
    return {f: getattr(info, f) for f, _ in N.ReorderInfo._fields_ if f != "pad"}


def apply_window_updates(s, q, a: int, qw, stream=None) -> None:
    """Synchronous L/R/Q propagation of a window similarity
    (window_tasks.cpp:89-102) on CUDA tensors; qw is the d x d accumulator."""
    _need_torch_cuda(s)
    n = s.shape[0]
    d = qw.shape[0]
    sw, lds, cb_s = _as_colmajor(s)
    qq, ldq, cb_q = (_as_colmajor(q) if q is not None else (None, n, False))
    qwc = qw.t().contiguous()  # column-major d x d, ld d
    N.check(N.lib().teig_apply_window_updates_device(
        n, sw.data_ptr(), lds, qq.data_ptr() if qq is not None else None, ldq, a, d, qwc.data_ptr(),
        _stream_ptr(stream, s)))
    if cb_s:
        s.copy_(sw)
    if cb_q:
        q.copy_(qq)


def gen_schur_input(n: int, fill_seed: int, device="cuda", stream=None):
    """Synthetic Schur form of SURVEY.md 8d generated in HBM (column-major)."""
    t = colmajor_empty(n, device)
    N.check(N.lib().teig_gen_schur_input_device(n, t.data_ptr(), n, int(fill_seed) & (2**64 - 1),
                                                _stream_ptr(stream, t)))
    return t


def gen_hessenberg(n: int, seed: int, device="cuda", stream=None):
    t = colmajor_empty(n, device)
    N.check(N.lib().teig_gen_hessenberg_device(n, t.data_ptr(), n, int(seed) & (2**64 - 1),
                                               _stream_ptr(stream, t)))
    return t


def identity(n: int, device="cuda", stream=None):
    t = colmajor_empty(n, device)
    N.check(N.lib().teig_set_identity_device(n, t.data_ptr(), n, _stream_ptr(stream, t)))
    return t


def known_spectrum_seed(seed: int) -> int:
    """Fill seed generate() derives for known_spectrum (generate.cpp:184)."""
    return (seed * 0x9E3779B97F4A7C15 + 1) & (2**64 - 1)


def scan_blocks_device(s, stream=None) -> np.ndarray:
    _need_torch_cuda(s)
    sw, lds, _ = _as_colmajor(s)
    n = s.shape[0]
    sizes = np.zeros(n, dtype=np.uint8)
    nb = N.check(N.lib().teig_scan_blocks_device(n, sw.data_ptr(), lds, sizes.ctypes.data_as(C.c_void_p),
                                                 _stream_ptr(stream, s)))
    return sizes[:nb].copy()


def plan_reorder(n: int, sel: Selection, window_size: int = 0):
    """Host planner of the GPU scheduler (no device work).  Returns
    (windows int64[k, 5] of (wtop, wbot, count, group, level), n_levels,
    n_groups, update flops with Q)."""
    sizes, flags = sel.sizes_array(), sel.flags_array()
    nb = len(sizes)
    cap = max(64, 2 * nb)
    while True:
        win = np.zeros(5 * cap, dtype=np.int64)
        nl, ng, fl = C.c_int64(0), C.c_int64(0), C.c_double(0)
        k = N.check(N.lib().teig_plan_reorder(n, nb, sizes.ctypes.data_as(C.c_void_p),
                                              flags.ctypes.data_as(C.c_void_p), window_size,
                                              win.ctypes.data_as(C.c_void_p), cap, C.byref(nl),
                                              C.byref(ng), C.byref(fl)))
        if k <= cap:
            return win[:5 * k].reshape(k, 5), nl.value, ng.value, fl.value
        cap = k


# ---------------------------------------------------------------------------
# generalized Schur-pair reordering (S, T) with Q and Z

@dataclass
class GReorderResult:
    s: object
    t: object
    q: object
    z: object
    permutation: List[int]
    rejected_blocks: List[int]
    clean: bool
    info: dict


def greorder_schur(s, t, q, z, sel: Selection, opts: Optional[ReorderOptions] = None,
                   stream=None) -> GReorderResult:
    """Moves the selected generalized eigenvalues of the pencil (S, T) to the
    leading blocks: (S, T) <- Qs^T (S, T) Zs, q <- q Qs, z <- z Zs (LAPACK
    DTGSEN semantics on the reference's reorder planner).  S upper
    quasi-triangular with the block structure of `sel`, T upper triangular.
    CUDA tensors are updated in place (column-major), numpy arrays through
    the host entry point (copies returned)."""
    opts = opts or ReorderOptions()
    n = s.shape[0]
    row = 0
    for b in sel.blocks:
        if b.start != row:
            raise ValueError("reorder: selection does not match (S, T)")
        row += b.size
    if row != n or len(sel.flags) != len(sel.blocks):
        raise ValueError("reorder: selection does not match (S, T)")
    nb = len(sel.blocks)
    sizes, flags = sel.sizes_array(), sel.flags_array()
    perm = np.zeros(max(nb, 1), dtype=np.int64)
    rej = np.zeros(max(nb, 1), dtype=np.int64)
    info = N.ReorderInfo()
    o = N.ReorderOpts()
    N.lib().teig_reorder_opts_default(C.byref(o))
    o.window_size = int(opts.window_size)
    o.strict = int(bool(opts.strict))
    vp = lambda a: a.ctypes.data_as(C.c_void_p)
    if torch is not None and isinstance(s, torch.Tensor):
        mats = []
        for m in (s, t, q, z):
            if m is None:
                mats.append((None, n, False))
            else:
                _need_torch_cuda(m)
                mats.append(_as_colmajor(m))
        ptr = lambda k: mats[k][0].data_ptr() if mats[k][0] is not None else None
        rc = N.lib().teig_greorder_schur_device(n, ptr(0), mats[0][1], ptr(1), mats[1][1], ptr(2), mats[2][1], ptr(3),
                                                mats[3][1], nb, vp(sizes), vp(flags), C.byref(o), vp(perm), vp(rej),
                                                C.byref(info), _stream_ptr(stream, s))
        if rc == -1002:
            raise RuntimeError("reorder: swap rejected in strict mode")
        N.check(rc)
        for m, (w, _, cb) in zip((s, t, q, z), mats):
            if cb:
                m.copy_(w)
        outs = (s, t, q, z)
    else:
        hs = [np.asfortranarray(np.array(m, dtype=np.float64, copy=True)) if m is not None else None for m in (s, t, q, z)]
        p = lambda a: vp(a) if a is not None else None
        rc = N.lib().teig_greorder_schur_host(n, p(hs[0]), n, p(hs[1]), n, p(hs[2]), n, p(hs[3]), n, nb, vp(sizes),
                                              vp(flags), C.byref(o), vp(perm), vp(rej), C.byref(info), None)
        if rc == -1002:
            raise RuntimeError("reorder: swap rejected in strict mode")
        N.check(rc)
        outs = tuple(hs)
    inf = {f: getattr(info, f) for f, _ in N.ReorderInfo._fields_ if f != "pad"}
    return GReorderResult(*outs, [int(x) for x in perm[:nb]], [int(x) for x in rej[:info.n_rejected]],
                          bool(info.clean), inf)


def gen_pair_t(n: int, seed: int, device="cuda", stream=None):
    """The C5 input T in HBM, column-major."""
    tt = colmajor_empty(n, device)
    N.check(N.lib().teig_gen_pair_t_device(n, tt.data_ptr(), n, int(seed) & (2**64 - 1), _stream_ptr(stream, tt)))
    return tt
