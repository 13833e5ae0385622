"""Eigenvector back-transformation on the device (mirror of
``taskeig::backtransform``, reference eigvec.hpp:88-89 / eigvec.cpp:448-516).

X = Q Y with the orthogonal factor a ``reorder_schur`` / ``schur_reduce`` call
left in HBM (no host round trip between the phases), on the FP64 tensor pipe
(csrc/backtransform.cu), then each real column and each complex pair scaled
to unit max-norm with a positive lead entry -- the reference's convention.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import _native as N
from .reorder import _as_colmajor, _need_torch_cuda, _stream_ptr

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None


def backtransform(y, q, col_kind: Optional[Sequence[int]] = None, stream=None):
    """Returns X = Q Y (n x k CUDA float64 tensor, column-major), renormalised
    per ``col_kind`` (0 real, 1 real part of a pair, 2 imaginary part; None:
    no renormalisation).  Raises ``ValueError`` on a dimension mismatch (the
    reference's std::invalid_argument) and ``TaskeigError`` on a non-finite
    result (its assert_finite)."""
    _need_torch_cuda(y)
    _need_torch_cuda(q)
    n, k = y.shape
    if q.shape[0] != n or q.shape[1] != n:
        raise ValueError("backtransform: dimension mismatch")
    if col_kind is not None and len(col_kind) != k:
        raise ValueError("backtransform: one col_kind per column")
    x = torch.empty((k, n), dtype=torch.float64, device=y.device).t()
    if k == 0:
        return x
    qw, ldq, _ = _as_colmajor(q)
    yw, ldy, _ = _as_colmajor(y)
    kind = None if col_kind is None else np.ascontiguousarray(col_kind, dtype=np.int8)
    N.check(N.lib().teig_backtransform_device(
        n, k, qw.data_ptr(), ldq, yw.data_ptr(), ldy, x.data_ptr(), n,
        kind.ctypes.data_as(C.c_void_p) if kind is not None else None, _stream_ptr(stream, y)))
    return x
