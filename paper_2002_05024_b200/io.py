"""Matrix files in the reference's formats (mirror of taskeig's
write_matrix_file / read_matrix_file, reference io.hpp / io.cpp:37-121),
through the C ABI (csrc/io.cpp): "teig" (binary, row-major float64) and
"matrixmarket" (array real general, column by column, 17 digits).  Arrays are
row-major numpy float64 (the reference's DenseBuffer); errors raise
``TaskeigError`` (the reference's std::runtime_error / invalid_argument)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N


def write_matrix_file(path: str, a, fmt: str = "teig") -> None:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if a.ndim != 2:
        raise ValueError("write_matrix_file: a 2-D array is required")
    N.check(N.lib().teig_write_matrix_file(str(path).encode(), fmt.encode(), a.shape[0], a.shape[1],
                                           a.ctypes.data_as(C.c_void_p)))


def read_matrix_file(path: str, fmt: str = "teig") -> np.ndarray:
    r, c = C.c_int64(0), C.c_int64(0)
    N.check(N.lib().teig_read_matrix_file(str(path).encode(), fmt.encode(), C.byref(r), C.byref(c), None, 0))
    a = np.empty((r.value, c.value), dtype=np.float64)
    N.check(N.lib().teig_read_matrix_file(str(path).encode(), fmt.encode(), C.byref(r), C.byref(c),
                                          a.ctypes.data_as(C.c_void_p), a.size))
    return a
