"""Host-side mirror of the reference's Schur-reduction API (schur.hpp:18-95).

Same names, argument meaning and error behaviour as ``taskeig::`` --
``DeflationCondition``, ``SchurOptions``, ``AedResult``, ``BulgeChain``,
``SchurDecomposition``, ``deflation_check``, ``aed_step``,
``introduce_bulges``, ``chase_bulges``, ``schur_reduce`` and
``kernels::small_schur`` -- over the B200 C ABI (include/taskeig_b200.h).
Matrices are torch CUDA float64 tensors (updated in place when stored
column-major, the orientation of the reference's tiles) or, for
``schur_reduce``, numpy arrays (host entry point, copies inside the call).
There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N
from .reorder import _as_colmajor, _need_torch_cuda, _stream_ptr

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None


class DeflationCondition(enum.IntEnum):  # schur.hpp:18
    classic = 0
    norm_stable = 1


@dataclass
class SchurOptions:  # schur.hpp:20-29
    deflation: DeflationCondition = DeflationCondition.norm_stable
    shift_count: int = 0       # 0: max(4, round-to-even(active/16)), cap 64
    aed_window: int = 0        # 0: 3m/2
    iteration_limit: int = 0   # 0: 30 n total sweeps
    small_threshold: int = 64
    workers: int = 0           # accepted for API parity; the GPU path ignores it
    seed: int = 0              # accepted for API parity
    keep_reports: bool = False  # the call's execution trace in SchurDecomposition.info['round_reports'] (JSON)
    tile_size: int = 0         # chase window; 0 = default_tile_size(n) (the TiledMatrix tile)
    profile: bool = False      # CUDA-event time per kernel class in SchurDecomposition.info


@dataclass
class AedResult:  # schur.hpp:32-39
    window: int = 0
    deflated: int = 0
    shifts: List[complex] = field(default_factory=list)
    spike_eliminated: bool = False
    converged: bool = True
    swap_rejected: bool = False


@dataclass
class BulgeChain:  # schur.hpp:43-48
    positions: List[int] = field(default_factory=list)  # bottom-most first
    shifts_used: int = 0
    chain_begin: int = 0
    chain_end: int = 0


@dataclass
class SchurDecomposition:  # schur.hpp:50-58
    s: object
    q: object
    eigenvalues: List[complex]
    sweeps: int
    converged: bool
    converged_trailing: int
    info: dict


def _opts(opts: Optional[SchurOptions]) -> N.SchurOpts:
    opts = opts or SchurOptions()
    o = N.SchurOpts()
    N.lib().teig_schur_opts_default(C.byref(o))
    o.deflation = int(opts.deflation)
    o.shift_count = int(opts.shift_count)
    o.aed_window = int(opts.aed_window)
    o.small_threshold = int(opts.small_threshold)
    o.iteration_limit = int(opts.iteration_limit)
    o.tile_size = int(opts.tile_size)
    o.profile = int(bool(opts.profile))
    return o


def deflation_check(spike_mag: float, block_diag_abs_sum: float, cond: DeflationCondition,
                    window_frob_norm: float) -> bool:
    """classic: |s| <= max(eps * sum|diag|, safmin); norm-stable: |s| <= eps ||W||_F
    (schur.cpp:406-411)."""
    return bool(N.lib().teig_deflation_check(float(spike_mag), float(block_diag_abs_sum), int(cond),
                                             float(window_frob_norm)))


def _dev_mats(h, q):
    _need_torch_cuda(h)
    hw, ldh, cb_h = _as_colmajor(h)
    if q is not None:
        _need_torch_cuda(q)
        qw, ldq, cb_q = _as_colmajor(q)
    else:
        qw, ldq, cb_q = None, h.shape[0], False
    return hw, ldh, cb_h, qw, ldq, cb_q


def _copy_back(h, hw, cb_h, q, qw, cb_q):
    if cb_h:
        h.copy_(hw)
    if cb_q:
        q.copy_(qw)


def _vp(a):
    return a.ctypes.data_as(C.c_void_p)


def schur_reduce(h, q=None, opts: Optional[SchurOptions] = None, stream=None) -> SchurDecomposition:
    """Multishift QR with aggressive early deflation: reduces the upper
    Hessenberg h to standardized real Schur form; q (if given) becomes q * Z
    (schur.hpp:91-95).  CUDA tensors are reduced in place (when column-major);
    numpy arrays go through the host entry point and are returned as copies."""
    n = h.shape[0]
    if h.shape[1] != n:
        raise ValueError("schur_reduce: matrix must be square")
    o = _opts(opts)
    info = N.SchurInfo()
    re = np.zeros(n)
    im = np.zeros(n)
    keep = bool(opts is not None and opts.keep_reports)
    if keep:  # SchurOptions::keep_reports: the call's execution trace
        N.trace_enable(True)
    try:
        s_out, q_out = _schur_call(h, q, n, o, re, im, info, stream)
    finally:
        if keep:
            N.trace_enable(False)
    conv = bool(info.converged)
    eig = [complex(a, b) for a, b in zip(re, im)] if conv else []
    inf = {f: getattr(info, f) for f, _ in N.SchurInfo._fields_ if f != "pad"}
    if keep:
        inf["round_reports"] = N.trace_json()
    return SchurDecomposition(s_out, q_out, eig, int(info.sweeps), conv, int(info.converged_trailing), inf)


def _schur_call(h, q, n, o, re, im, info, stream):
    if torch is not None and isinstance(h, torch.Tensor):
        hw, ldh, cb_h, qw, ldq, cb_q = _dev_mats(h, q)
        N.check(N.lib().teig_schur_reduce_device(n, hw.data_ptr(), ldh, qw.data_ptr() if qw is not None else None,
                                                 ldq, C.byref(o), _vp(re), _vp(im), C.byref(info),
                                                 _stream_ptr(stream, h)))
        _copy_back(h, hw, cb_h, q, qw, cb_q)
        s_out, q_out = h, q
    else:
        hf = np.asfortranarray(np.array(h, dtype=np.float64, copy=True))
        qf = np.asfortranarray(np.array(q, dtype=np.float64, copy=True)) if q is not None else None
        N.check(N.lib().teig_schur_reduce_host(n, _vp(hf), n, _vp(qf) if qf is not None else None, n, C.byref(o),
                                               _vp(re), _vp(im), C.byref(info), None))
        s_out, q_out = hf, qf
    return s_out, q_out


def aed_step(h, q, l: int, ihi: int, window: int, opts: Optional[SchurOptions] = None,
             stream=None) -> AedResult:
    """One AED step on the trailing window of the active range [l, ihi)
    (schur.hpp:66-69), window task + off-window updates, in place."""
    if window < 4:
        raise ValueError("aed_step: window must be >= 4")
    n = h.shape[0]
    hw, ldh, cb_h, qw, ldq, cb_q = _dev_mats(h, q)
    o = _opts(opts)
    r = N.AedResultC()
    sh = np.zeros(2 * max(window, 1) + 4)
    N.check(N.lib().teig_aed_step_device(n, hw.data_ptr(), ldh, qw.data_ptr() if qw is not None else None, ldq,
                                         int(l), int(ihi), int(window), C.byref(o), C.byref(r), _vp(sh),
                                         _stream_ptr(stream, h)))
    _copy_back(h, hw, cb_h, q, qw, cb_q)
    k = int(r.nshifts)
    return AedResult(int(r.window), int(r.deflated), [complex(sh[2 * i], sh[2 * i + 1]) for i in range(k)],
                     bool(r.spike_eliminated), bool(r.converged), bool(r.swap_rejected))


def introduce_bulges(h, q, l: int, ihi: int, shifts: Sequence[complex], stream=None) -> BulgeChain:
    """Plants len(shifts)/2 bulges at the top of [l, ihi) (schur.hpp:71-75);
    raises ValueError on malformed shift lists like the reference."""
    shifts = [complex(z) for z in shifts]
    if len(shifts) < 2:
        raise ValueError("introduce_bulges: need at least two shifts")
    if len(shifts) % 2:
        raise ValueError("introduce_bulges: shifts must come in pairs")
    for j in range(0, len(shifts) - 1, 2):
        s1, s2 = shifts[j], shifts[j + 1]
        if s1.imag != 0.0 and (s1.real != s2.real or s1.imag != -s2.imag):
            raise ValueError("introduce_bulges: shift pair not conjugate")
    nb = len(shifts) // 2
    if l + 3 * nb + 2 > ihi:
        raise ValueError("introduce_bulges: too many shifts for range")
    n = h.shape[0]
    hw, ldh, cb_h, qw, ldq, cb_q = _dev_mats(h, q)
    sh = np.zeros(2 * len(shifts))
    sh[0::2] = [z.real for z in shifts]
    sh[1::2] = [z.imag for z in shifts]
    pos = np.zeros(nb, dtype=np.int64)
    N.check(N.lib().teig_introduce_bulges_device(n, hw.data_ptr(), ldh, qw.data_ptr() if qw is not None else None,
                                                 ldq, int(l), int(ihi), len(shifts), _vp(sh), _vp(pos),
                                                 _stream_ptr(stream, h)))
    _copy_back(h, hw, cb_h, q, qw, cb_q)
    return BulgeChain([int(p) for p in pos], len(shifts), int(l), int(ihi))


def chase_bulges(h, q, chain: BulgeChain, window_size: int, opts: Optional[SchurOptions] = None,
                 stream=None) -> int:
    """Chases every bulge of the chain off the bottom of the active range with
    windows of max(window_size, 3nb+6) rows and their off-window updates
    (schur.hpp:85-89).  Empties chain.positions; returns the window count."""
    if not chain.positions:
        return 0
    n = h.shape[0]
    hw, ldh, cb_h, qw, ldq, cb_q = _dev_mats(h, q)
    pos = np.asarray(chain.positions, dtype=np.int64)
    nw = C.c_int64(0)
    N.check(N.lib().teig_chase_bulges_device(n, hw.data_ptr(), ldh, qw.data_ptr() if qw is not None else None,
                                             ldq, int(chain.chain_end), len(pos), _vp(pos), int(window_size),
                                             C.byref(nw), _stream_ptr(stream, h)))
    _copy_back(h, hw, cb_h, q, qw, cb_q)
    chain.positions = []
    return int(nw.value)


def small_schur(h, stream=None):
    """kernels::small_schur (kernels.hpp:93) on a k x k CUDA tensor in place.
    Returns (converged, q) with q the k x k similarity."""
    _need_torch_cuda(h)
    k = h.shape[0]
    hw, ldh, cb_h = _as_colmajor(h)
    qt = torch.empty((k, k), dtype=torch.float64, device=h.device)
    conv = C.c_int32(0)
    N.check(N.lib().teig_small_schur_device(k, hw.data_ptr(), ldh, qt.data_ptr(), C.byref(conv),
                                            _stream_ptr(stream, h)))
    if cb_h:
        h.copy_(hw)
    return bool(conv.value), qt.t()


def schur_reduce_host_buffers(h_buf: np.ndarray, q_buf: Optional[np.ndarray], n: int,
                              opts: Optional[SchurOptions] = None) -> dict:
    """Reduces HOST buffers holding H and Q COLUMN-MAJOR with ld = n (e.g. a
    C-ordered array of H^T) in place through the C ABI's host entry point;
    host<->device copies happen inside the call."""
    assert h_buf.dtype == np.float64 and h_buf.size == n * n and h_buf.flags.contiguous
    o = _opts(opts)
    info = N.SchurInfo()
    N.check(N.lib().teig_schur_reduce_host(n, _vp(h_buf), n, _vp(q_buf) if q_buf is not None else None, n,
                                           C.byref(o), None, None, C.byref(info), None))
    return {f: getattr(info, f) for f, _ in N.SchurInfo._fields_ if f != "pad"}
