"""Hessenberg reduction on the device (mirror of ``taskeig::hessenberg_reduce``,
reference hessenberg.hpp / hessenberg.cpp:185-280): the reference's blocked
compact-WY algorithm (csrc/hessenberg.cu) -- per-column reductions and the
panel GEMV on all SMs, the trailing / top-right / Q1 updates as FP64
tensor-core GEMMs -- feeding ``schur_reduce`` without leaving HBM."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

from . import _native as N
from .reorder import _as_colmajor, _need_torch_cuda, _stream_ptr, colmajor_empty


class HessenbergInfo(C.Structure):
    _fields_ = [("panels", C.c_int64), ("launches", C.c_int64), ("flops", C.c_double),
                ("panel_width", C.c_int64)]


@dataclass
class HessenbergOptions:  # hessenberg.hpp:57-61
    workers: int = 0       # accepted for API parity; the device path is deterministic
    panel_width: int = 0   # 0: min(tile, 64) as the reference; values above 64 run at 64
    seed: int = 0          # accepted for API parity


@dataclass
class HessenbergResult:  # hessenberg.hpp:63-67
    h: object
    q: object
    info: dict


def hessenberg_reduce(a, accumulate_q: bool = True, opts: Optional[HessenbergOptions] = None,
                      stream=None) -> HessenbergResult:
    """Reduces the square CUDA float64 tensor ``a`` in place to upper
    Hessenberg form H = Q1^T A Q1 (exact zeros below the subdiagonal); returns
    H (= a) and, when accumulate_q, Q1 as a new column-major tensor."""
    _need_torch_cuda(a)
    n = a.shape[0]
    if a.shape[1] != n:
        raise ValueError("hessenberg_reduce: matrix must be square")
    opts = opts or HessenbergOptions()
    aw, lda, cb = _as_colmajor(a)
    q = colmajor_empty(n, a.device) if accumulate_q else None
    info = HessenbergInfo()
    N.check(N.lib().teig_hessenberg_reduce_device(n, aw.data_ptr(), lda, q.data_ptr() if q is not None else None, n,
                                                  int(opts.panel_width), C.byref(info), _stream_ptr(stream, a)))
    if cb:
        a.copy_(aw)
    return HessenbergResult(a, q, {f: getattr(info, f) for f, _ in HessenbergInfo._fields_})
