"""ctypes binding of the in-tree C ABI (include/taskeig_b200.h).

The product path is the CUDA library ``_lib/libtaskeig_b200.so``; there is
no CPU fallback.  Importing this module on a machine without the built
library raises immediately, and every call that fails on the device raises
``TaskeigError`` carrying the library's message.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TEIG_LIB_PATH") or os.path.join(HERE, "_lib", "libtaskeig_b200.so")
CSRC = os.path.join(HERE, "csrc")


class TaskeigError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"taskeig_b200 error {code}: {msg}")
        self.code = code


def build(verbose: bool = False) -> str:
    """Compile the sm_100a library in-tree (nvcc cross-compiles without a GPU)."""
    cmd = ["make", "-C", CSRC, "-j8"]
    if not verbose:
        cmd.insert(1, "-s")
    subprocess.run(cmd, check=True)
    return LIB_PATH


class ReorderOpts(C.Structure):
    _fields_ = [("window_size", C.c_int64), ("strict", C.c_int32), ("overlap_factor", C.c_int32),
                ("profile", C.c_int32), ("full_factor", C.c_int32)]


class ReorderInfo(C.Structure):
    _fields_ = [("n_windows", C.c_int64), ("n_levels", C.c_int64), ("n_passes", C.c_int64),
                ("n_groups", C.c_int64), ("n_rejected", C.c_int64), ("clean", C.c_int32),
                ("pad", C.c_int32), ("update_flops", C.c_double), ("update_bytes", C.c_double),
                ("plan_ms", C.c_double), ("n_launches", C.c_int64), ("ms_window", C.c_double),
                ("ms_left", C.c_double), ("ms_right", C.c_double), ("ms_factor", C.c_double),
                ("flops_left", C.c_double), ("flops_right", C.c_double), ("flops_factor", C.c_double),
                ("flops_factor_exec", C.c_double), ("flops_dmma", C.c_double)]


class SchurOpts(C.Structure):
    _fields_ = [("deflation", C.c_int32), ("shift_count", C.c_int32), ("aed_window", C.c_int32),
                ("small_threshold", C.c_int32), ("iteration_limit", C.c_int64), ("tile_size", C.c_int64),
                ("profile", C.c_int32), ("pad", C.c_int32)]


class SchurInfo(C.Structure):
    _fields_ = [("sweeps", C.c_int64), ("rounds", C.c_int64), ("aed_windows", C.c_int64),
                ("chase_windows", C.c_int64), ("converged_trailing", C.c_int64), ("n_launches", C.c_int64),
                ("converged", C.c_int32), ("pad", C.c_int32), ("update_flops", C.c_double),
                ("ms_window", C.c_double), ("ms_update", C.c_double), ("ms_total_host", C.c_double)]


class AedResultC(C.Structure):
    _fields_ = [("window", C.c_int64), ("deflated", C.c_int64), ("nshifts", C.c_int64),
                ("spike_eliminated", C.c_int32), ("converged", C.c_int32), ("swap_rejected", C.c_int32),
                ("pad", C.c_int32)]


_P = C.c_void_p
_I64 = C.c_int64

# symbol -> (restype, argtypes); the test suite checks that every symbol
# declared in include/taskeig_b200.h is exported.
SIGNATURES = {
    "teig_last_error": (C.c_char_p, []),
    "teig_version": (C.c_int, []),
    "teig_reorder_opts_default": (None, [_P]),
    "teig_reorder_schur_device": (C.c_int, [_I64, _P, _I64, _P, _I64, _I64, _P, _P, _P, _P, _P, _P,
                                            _I64, _P, _P]),
    "teig_release_host_staging": (None, []),
    "teig_set_memory_retention": (None, [C.c_int32]),
    "teig_memory_retention": (C.c_int32, []),
    "teig_release_memory": (None, []),
    "teig_host_transfer_bytes": (None, [C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "teig_trace_enable": (None, [C.c_int32]),
    "teig_trace_json": (C.c_int64, [C.c_char_p, C.c_int64]),
    "teig_trace_task_count": (C.c_int64, []),
    "teig_trace_task": (C.c_int, [_I64, C.c_char_p, _I64, _P, _P, _P]),
    "teig_reorder_schur_host": (C.c_int, [_I64, _P, _I64, _P, _I64, _I64, _P, _P, _P, _P, _P, _P,
                                          _I64, _P, _P]),
    "teig_scan_blocks_device": (C.c_int64, [_I64, _P, _I64, _P, _P]),
    "teig_select_fraction": (C.c_int, [_I64, C.c_double, C.c_uint64, _P]),
    "teig_plan_reorder": (C.c_int64, [_I64, _I64, _P, _P, _I64, _P, _I64, _P, _P, _P]),
    "teig_window_reorder_device": (C.c_int, [_I64, _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P]),
    "teig_apply_window_updates_device": (C.c_int, [_I64, _P, _I64, _P, _I64, _I64, _I64, _P, _P]),
    "teig_update_panel_device": (C.c_int, [C.c_int32, _I64, _P, _I64, _P, _I64, _I64, _I64, _I64, _I64, _P]),
    "teig_gen_schur_input_device": (C.c_int, [_I64, _P, _I64, C.c_uint64, _P]),
    "teig_gen_hessenberg_device": (C.c_int, [_I64, _P, _I64, C.c_uint64, _P]),
    "teig_set_identity_device": (C.c_int, [_I64, _P, _I64, _P]),
    "teig_schur_opts_default": (None, [_P]),
    "teig_schur_reduce_device": (C.c_int, [_I64, _P, _I64, _P, _I64, _P, _P, _P, _P, _P]),
    "teig_schur_reduce_host": (C.c_int, [_I64, _P, _I64, _P, _I64, _P, _P, _P, _P, _P]),
    "teig_aed_step_device": (C.c_int, [_I64, _P, _I64, _P, _I64, _I64, _I64, _I64, _P, _P, _P, _P]),
    "teig_introduce_bulges_device": (C.c_int, [_I64, _P, _I64, _P, _I64, _I64, _I64, _I64, _P, _P, _P]),
    "teig_chase_bulges_device": (C.c_int, [_I64, _P, _I64, _P, _I64, _I64, _I64, _P, _I64, _P, _P]),
    "teig_small_schur_device": (C.c_int, [_I64, _P, _I64, _P, _P, _P]),
    "teig_plan_chase": (C.c_int64, [_I64, _P, _I64, _I64, _P, _I64]),
    "teig_backtransform_device": (C.c_int, [_I64, _I64, _P, _I64, _P, _I64, _P, _I64, _P, _P]),
    "teig_hessenberg_reduce_device": (C.c_int, [_I64, _P, _I64, _P, _I64, _I64, _P, _P]),
    "teig_write_matrix_file": (C.c_int, [C.c_char_p, C.c_char_p, _I64, _I64, _P]),
    "teig_read_matrix_file": (C.c_int, [C.c_char_p, C.c_char_p, _P, _P, _P, _I64]),
    "teig_deflation_check": (C.c_int, [C.c_double, C.c_double, C.c_int32, C.c_double]),
    "teig_greorder_schur_device": (C.c_int, [_I64, _P, _I64, _P, _I64, _P, _I64, _P, _I64, _I64, _P, _P, _P, _P,
                                             _P, _P, _P]),
    "teig_greorder_schur_host": (C.c_int, [_I64, _P, _I64, _P, _I64, _P, _I64, _P, _I64, _I64, _P, _P, _P, _P,
                                           _P, _P, _P]),
    "teig_gen_pair_t_device": (C.c_int, [_I64, _P, _I64, C.c_uint64, _P]),
    "teig_dist_balance": (C.c_int, [_I64, _I64, _P, _P, _I64, C.c_int32, _P, _P]),
    "teig_dist_schedule": (C.c_int64, [_I64, _I64, _P, _P, _I64, C.c_int32, _P, _P, _I64]),
    "teig_dist_reorder_schur": (C.c_int, [_I64, C.c_int32, C.c_int32, _P, _P, _I64, _P, _P, _P, _I64, _P, _P, _P,
                                          _P, _P, _P, _P]),
    "teig_dist_greorder_schur": (C.c_int, [_I64, C.c_int32, C.c_int32, _P, _P, _P, _I64, _P, _P, _P, _P, _I64, _P,
                                           _P, _P, _P, _P, _P, _P]),
    "teig_dist_reorder_schur_multi": (C.c_int, [_I64, C.c_int32, _P, _P, _I64, _P, _P, _P, _I64, _P, _P, _P, _P, _P,
                                                _P, _I64, _P]),
    "teig_nccl_available": (C.c_int, []),
    "teig_nccl_unique_id": (C.c_int, [_P]),
    "teig_nccl_comm_init": (C.c_int, [C.c_int32, C.c_int32, _P, _P]),
    "teig_nccl_comm_destroy": (C.c_int, [_P]),
    "teig_gen_schur_input_cols_device": (C.c_int, [_I64, _P, _I64, _I64, _I64, C.c_uint64, _P]),
    "teig_set_identity_rows_device": (C.c_int, [_I64, _P, _I64, _I64, _I64, _P]),
}

_lib = None


def lib():
    """Load the native library (built in-tree).  Raises if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> int:
    if rc < 0:
        raise TaskeigError(rc, lib().teig_last_error().decode(errors="replace"))
    return rc


def set_memory_retention(on: bool) -> None:
    """Keep the library's device pool and host-path staging between calls
    (teig_set_memory_retention; off by default)."""
    lib().teig_set_memory_retention(1 if on else 0)


def memory_retention() -> bool:
    return bool(lib().teig_memory_retention())


def host_transfer_bytes():
    """(h2d, d2h) bytes of this thread's last host-entry-point reorder call."""
    a, b = C.c_int64(0), C.c_int64(0)
    lib().teig_host_transfer_bytes(C.byref(a), C.byref(b))
    return int(a.value), int(b.value)


def release_memory() -> None:
    """Return the library's cached device memory (staging + pools, every device)."""
    lib().teig_release_memory()


def trace_enable(on: bool = True) -> None:
    """Record an execution trace of the reorder calls made on this thread."""
    lib().teig_trace_enable(1 if on else 0)


def trace_json() -> str:
    """The last traced call's trace (JSON: tasks, stalls, windows)."""
    n = lib().teig_trace_json(None, 0)
    buf = C.create_string_buffer(n + 1)
    lib().teig_trace_json(buf, n + 1)
    return buf.value.decode()
