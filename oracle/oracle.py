"""oracle/oracle.py -- TEST INFRASTRUCTURE ONLY.

ctypes views of
  * ``oracle/_build/libteig_oracle.so`` -- the plain-C restatement of the
    reference's reorder path (``teig_oracle.c``), and
  * ``oracle/_ref/libtaskeig_ref.so``   -- the UNMODIFIED reference
    (``/root/reference/proj/src``) compiled from its own sources by
    ``oracle/Makefile`` plus our extern "C" shim (``ref_shim.cpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module; the
product package never does.  Parity of the restatement against the reference
is pinned by ``tests/test_oracle.py`` (bit-for-bit) and by the golden
fixtures in ``tests/golden/``.

Matrices handed to the restatement are numpy arrays in FORTRAN order
(column-major, ``ld = rows``); the reference shim takes row-major arrays,
its own ``from_dense``/``to_dense`` convention (tiled_matrix.cpp:37-73).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libteig_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtaskeig_ref.so")

_P = C.c_void_p
_SZ = C.c_size_t
_U64 = C.c_uint64
_D = C.c_double


def build(ref: bool = True) -> None:
    """Compile the restatement (and the reference when its sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)


def _ptr(a):
    return a.ctypes.data_as(_P) if a is not None else None


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        L = C.CDLL(ORACLE_SO)
        L.teo_philox_round10.argtypes = [_P, _P, _P]
        L.teo_philox_round10.restype = None
        L.teo_schur_input.argtypes = [_SZ, _U64, _P, _SZ]
        L.teo_schur_input.restype = None
        L.teo_known_spectrum_seed.argtypes = [_U64]
        L.teo_known_spectrum_seed.restype = _U64
        L.teo_hessenberg_random.argtypes = [_SZ, _U64, _P, _SZ]
        L.teo_hessenberg_random.restype = None
        L.teo_scan_blocks.argtypes = [_SZ, _P, _SZ, _P]
        L.teo_scan_blocks.restype = _SZ
        L.teo_select_fraction.argtypes = [_SZ, _D, _U64, _P]
        L.teo_select_fraction.restype = None
        L.teo_standardize_2x2.argtypes = [_D, _D, _D, _D, _P]
        L.teo_standardize_2x2.restype = None
        L.teo_swap_adjacent_blocks.argtypes = [_SZ, _P, _SZ, _P, _SZ, _SZ, _SZ]
        L.teo_swap_adjacent_blocks.restype = C.c_int
        L.teo_window_reorder.argtypes = [_SZ, _P, _SZ, _P, _P, _P, _P, _P]
        L.teo_window_reorder.restype = C.c_int
        L.teo_reorder_schur.argtypes = [_SZ, _P, _SZ, _P, _SZ, _SZ, _P, _P, _SZ, _P, _P, _P,
                                        _P, _SZ, _P, _P, C.c_long]
        L.teo_reorder_schur.restype = C.c_long
        L.teo_similarity_residual.argtypes = [_SZ, _P, _SZ, _P, _SZ, _P, _SZ]
        L.teo_similarity_residual.restype = _D
        L.teo_orthogonality_defect.argtypes = [_SZ, _P, _SZ]
        L.teo_orthogonality_defect.restype = _D
        L.teo_is_standardized.argtypes = [_SZ, _P, _SZ]
        L.teo_is_standardized.restype = C.c_int
        L.teo_read_eigenvalues.argtypes = [_SZ, _P, _SZ, _P, _P]
        L.teo_read_eigenvalues.restype = None
        L.teo_plan_reorder.argtypes = [_SZ, _P, _P, _SZ, _P]
        L.teo_plan_reorder.restype = C.c_int
        L.teo_plan_free.argtypes = [_P]
        L.teo_plan_free.restype = None
        L.teo_plan_flops.argtypes = [_P, _SZ, C.c_int]
        L.teo_plan_flops.restype = _D
        L.teo_pair_t.argtypes = [_SZ, _U64, _P, _SZ]
        L.teo_pair_t.restype = None
        L.teo_small_schur.argtypes = [_SZ, _P, _P, _P]
        L.teo_small_schur.restype = C.c_int
        L.teo_deflation_check.argtypes = [_D, _D, C.c_int, _D]
        L.teo_deflation_check.restype = C.c_int
        L.teo_aed_step.argtypes = [_SZ, _P, _SZ, _P, _SZ, _SZ, _SZ, _SZ, _P, _P, _P]
        L.teo_aed_step.restype = C.c_int
        L.teo_sweep.argtypes = [_SZ, _P, _SZ, _P, _SZ, _SZ, _SZ, _SZ, _P, _SZ]
        L.teo_sweep.restype = C.c_int
        L.teo_schur_reduce.argtypes = [_SZ, _P, _SZ, _P, _SZ, _SZ, _P, _P, _P]
        L.teo_schur_reduce.restype = C.c_int
        _lib = L
    return _lib


class SchurOpts(C.Structure):
    """teo_schur_opts == SchurOptions (schur.hpp:20-29)."""
    _fields_ = [("deflation", C.c_int), ("shift_count", _SZ), ("aed_window", _SZ),
                ("iteration_limit", _SZ), ("small_threshold", _SZ)]


class AedOut(C.Structure):
    _fields_ = [("window", _SZ), ("deflated", _SZ), ("nshifts", _SZ), ("spike_eliminated", C.c_int),
                ("converged", C.c_int), ("swap_rejected", C.c_int), ("newbeta", _D)]


class SchurInfo(C.Structure):
    _fields_ = [("sweeps", _SZ), ("rounds", _SZ), ("converged_trailing", _SZ), ("converged", C.c_int)]


def schur_opts(deflation=1, shift_count=0, aed_window=0, iteration_limit=0, small_threshold=64):
    return SchurOpts(deflation, shift_count, aed_window, iteration_limit, small_threshold)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError("oracle/_ref/libtaskeig_ref.so not built (make -C oracle ref)")
        R = C.CDLL(REF_SO)
        R.ref_last_error.restype = C.c_char_p
        R.ref_philox_round10.argtypes = [_P, _P, _P]
        R.ref_philox_uniform_sym.argtypes = [_U64, _SZ, _P]
        R.ref_generate.argtypes = [C.c_int, _SZ, _U64, _P]
        R.ref_generate.restype = C.c_int
        R.ref_default_spectrum.argtypes = [_SZ, _U64, _P]
        R.ref_select_fraction.argtypes = [_SZ, _P, _D, _U64, _P, _P]
        R.ref_select_fraction.restype = C.c_long
        R.ref_select_by_name.argtypes = [_SZ, _P, C.c_char_p, _SZ, _P, _P]
        R.ref_select_by_name.restype = C.c_long
        R.ref_standardize_2x2.argtypes = [_D, _D, _D, _D, _P]
        R.ref_swap_adjacent_blocks.argtypes = [_SZ, _P, _SZ, _P, _SZ, _SZ, _SZ]
        R.ref_swap_adjacent_blocks.restype = C.c_int
        R.ref_window_reorder.argtypes = [_SZ, _P, _SZ, _P, _P, _P, _P, _P]
        R.ref_window_reorder.restype = C.c_int
        R.ref_reorder_schur.argtypes = [_SZ, _SZ, _P, _P, _SZ, _P, _SZ, _SZ, C.c_int, _P, _P,
                                        _P, _P, _SZ, _P, _P, _P]
        R.ref_reorder_schur.restype = C.c_int
        R.ref_problem_create.argtypes = [_SZ, _SZ, _P]
        R.ref_problem_create.restype = C.c_void_p
        R.ref_problem_destroy.argtypes = [C.c_void_p]
        R.ref_problem_reorder.argtypes = [C.c_void_p, _SZ, _P, _SZ, _SZ, C.c_int, _P, _P, _P]
        R.ref_problem_reorder.restype = C.c_int
        R.ref_backtransform.argtypes = [_SZ, _SZ, _P, _P, _P, _P, _SZ]
        R.ref_backtransform.restype = C.c_int
        R.ref_hessenberg_reduce.argtypes = [_SZ, _P, _P, _P, _SZ]
        R.ref_hessenberg_reduce.restype = C.c_int
        R.ref_schur_reduce.argtypes = [_SZ, _SZ, _P, _P, _SZ, C.c_int, _SZ, _SZ, _SZ, _SZ, _P,
                                       _P, _P]
        R.ref_schur_reduce.restype = C.c_int
        R.ref_small_schur.argtypes = [_SZ, _P, _P, _P]
        R.ref_small_schur.restype = C.c_int
        R.ref_aed_step.argtypes = [_SZ, _SZ, _P, _P, _SZ, _SZ, _SZ, C.c_int, _P, _P]
        R.ref_aed_step.restype = C.c_int
        R.ref_sweep.argtypes = [_SZ, _SZ, _P, _P, _SZ, _SZ, _SZ, _P, _SZ]
        R.ref_sweep.restype = C.c_int
        R.ref_similarity_residual.argtypes = [_SZ, _P, _P, _P]
        R.ref_similarity_residual.restype = _D
        R.ref_orthogonality_defect.argtypes = [_SZ, _P]
        R.ref_orthogonality_defect.restype = _D
        R.ref_is_standardized.argtypes = [_SZ, _P]
        R.ref_is_standardized.restype = C.c_int
        _ref = R
    return _ref


def _chk_ref(rc):
    if rc != 0:
        raise RuntimeError("reference: " + ref().ref_last_error().decode())


# --------------------------------------------------------------------------
# restatement (column-major)

def philox_round10(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    lib().teo_philox_round10(_ptr(c), _ptr(k), _ptr(o))
    return [int(x) for x in o]


def known_spectrum_seed(seed: int) -> int:
    return int(lib().teo_known_spectrum_seed(seed))


def schur_input(n: int, fill_seed: int) -> np.ndarray:
    """Synthetic standardized Schur form, column-major."""
    s = np.zeros((n, n), dtype=np.float64, order="F")
    lib().teo_schur_input(n, fill_seed, _ptr(s), n)
    return s


def hessenberg_random(n: int, seed: int) -> np.ndarray:
    h = np.zeros((n, n), dtype=np.float64, order="F")
    lib().teo_hessenberg_random(n, seed, _ptr(h), n)
    return h


def scan_blocks(s: np.ndarray) -> np.ndarray:
    s = np.asfortranarray(s)
    n = s.shape[0]
    sizes = np.zeros(n, dtype=np.uint8)
    nb = lib().teo_scan_blocks(n, _ptr(s), n, _ptr(sizes))
    return sizes[:nb].copy()


def select_fraction(nb: int, fraction: float, seed: int) -> np.ndarray:
    flags = np.zeros(max(nb, 1), dtype=np.uint8)
    lib().teo_select_fraction(nb, fraction, seed, _ptr(flags))
    return flags[:nb].copy()


def standardize_2x2(a, b, c, d):
    o = np.zeros(10)
    lib().teo_standardize_2x2(a, b, c, d, _ptr(o))
    return o


def swap_adjacent_blocks(s: np.ndarray, acc: np.ndarray, pos: int, p: int, q: int) -> int:
    assert s.flags.f_contiguous and acc.flags.f_contiguous
    return lib().teo_swap_adjacent_blocks(s.shape[0], _ptr(s), acc.shape[0], _ptr(acc), pos, p, q)


def window_reorder(w: np.ndarray, sizes, sel):
    """In place on the Fortran-ordered window; returns (executed, acc, order, stuck)."""
    assert w.flags.f_contiguous
    d = w.shape[0]
    sizes = np.asarray(sizes, dtype=np.uint8)
    sel = np.asarray(sel, dtype=np.uint8)
    nb = len(sizes)
    acc = np.zeros((d, d), order="F")
    order = np.zeros(max(nb, 1), dtype=np.uint32)
    stuck = np.zeros(max(nb, 1), dtype=np.uint8)
    ex = lib().teo_window_reorder(d, _ptr(w), nb, _ptr(sizes), _ptr(sel), _ptr(acc), _ptr(order),
                                  _ptr(stuck))
    return bool(ex), acc, order[:nb].copy(), stuck[:nb].astype(bool)


class _Window(C.Structure):
    _fields_ = [("wtop", _SZ), ("wbot", _SZ), ("first_block", _SZ), ("count", _SZ),
                ("group", _SZ), ("sizes_off", _SZ)]


class _Plan(C.Structure):
    _fields_ = [("n_windows", _SZ), ("cap_windows", _SZ), ("windows", C.POINTER(_Window)),
                ("n_entries", _SZ), ("cap_entries", _SZ), ("sizes", C.POINTER(C.c_uint8)),
                ("sel", C.POINTER(C.c_uint8)), ("n_groups", _SZ)]


def plan_reorder(sizes, flags, ws: int, n: int | None = None):
    """Planner bookkeeping only.  Returns (windows ndarray[k, 5] of
    (wtop, wbot, first_block, count, group), flops F_ref with Q, n_groups)."""
    sizes = np.asarray(sizes, dtype=np.uint8)
    flags = np.asarray(flags, dtype=np.uint8)
    pl = _Plan()
    rc = lib().teo_plan_reorder(len(sizes), _ptr(sizes), _ptr(flags), ws, C.byref(pl))
    if rc:
        raise RuntimeError("plan failed")
    k = pl.n_windows
    out = np.zeros((k, 5), dtype=np.int64)
    for i in range(k):
        w = pl.windows[i]
        out[i] = (w.wtop, w.wbot, w.first_block, w.count, w.group)
    if n is None:
        n = int(sizes.sum())
    fl = lib().teo_plan_flops(C.byref(pl), n, 1)
    ng = pl.n_groups
    lib().teo_plan_free(C.byref(pl))
    return out, fl, ng


def reorder_schur(s: np.ndarray, q: np.ndarray | None, sizes, flags, ws: int,
                  max_windows: int = 0):
    """Serial CPU reorder (in place on Fortran arrays)."""
    n = s.shape[0]
    assert s.flags.f_contiguous and (q is None or q.flags.f_contiguous)
    sizes = np.asarray(sizes, dtype=np.uint8)
    flags = np.asarray(flags, dtype=np.uint8)
    nb = len(sizes)
    perm = np.zeros(max(nb, 1), dtype=np.uintp)
    rej = np.zeros(max(nb, 1), dtype=np.uintp)
    nrej = _SZ(0)
    cap = 1 << 20
    plan = np.zeros(3 * cap, dtype=np.uintp)
    nplan = _SZ(0)
    clean = C.c_int(0)
    ex = lib().teo_reorder_schur(n, _ptr(s), n, _ptr(q), n, nb, _ptr(sizes), _ptr(flags), ws,
                                 _ptr(perm), _ptr(rej), C.byref(nrej), _ptr(plan), cap,
                                 C.byref(nplan), C.byref(clean), max_windows)
    if ex < 0:
        raise ValueError("reorder_schur: selection does not match s")
    k = min(nplan.value, cap)
    return dict(permutation=perm[:nb].astype(np.int64), rejected=rej[:nrej.value].astype(np.int64),
                plan=plan[:3 * k].reshape(k, 3).astype(np.int64), clean=bool(clean.value),
                windows_executed=int(ex))


def similarity_residual(a, q, s) -> float:
    a, q, s = (np.asfortranarray(x) for x in (a, q, s))
    n = a.shape[0]
    return lib().teo_similarity_residual(n, _ptr(a), n, _ptr(q), n, _ptr(s), n)


def orthogonality_defect(q) -> float:
    q = np.asfortranarray(q)
    return lib().teo_orthogonality_defect(q.shape[0], _ptr(q), q.shape[0])


def is_standardized(s) -> bool:
    s = np.asfortranarray(s)
    return bool(lib().teo_is_standardized(s.shape[0], _ptr(s), s.shape[0]))


def read_eigenvalues(s) -> np.ndarray:
    s = np.asfortranarray(s)
    n = s.shape[0]
    re = np.zeros(n)
    im = np.zeros(n)
    lib().teo_read_eigenvalues(n, _ptr(s), n, _ptr(re), _ptr(im))
    return re + 1j * im


def match_spectra(a, b) -> float:
    """Greedy minimal-distance matching (verify.cpp:132-153)."""
    a = list(np.asarray(a, dtype=complex))
    b = list(np.asarray(b, dtype=complex))
    if len(a) != len(b):
        return float("inf")
    worst = 0.0
    while a:
        A = np.asarray(a)[:, None]
        B = np.asarray(b)[None, :]
        dmat = np.abs(A - B)
        i, j = np.unravel_index(np.argmin(dmat), dmat.shape)
        worst = max(worst, float(dmat[i, j]))
        a.pop(i)
        b.pop(j)
    return worst


# --------------------------------------------------------------------------
# the unmodified reference (row-major interchange)

def ref_philox_round10(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    ref().ref_philox_round10(_ptr(c), _ptr(k), _ptr(o))
    return [int(x) for x in o]


def ref_generate(kind: int, n: int, seed: int) -> np.ndarray:
    """Row-major generate(); kind as ProblemKind (0 random, 1 known, 4 hess)."""
    out = np.zeros((n, n))
    _chk_ref(ref().ref_generate(kind, n, seed, _ptr(out)))
    return out


def ref_select_fraction(s_rm: np.ndarray, fraction: float, seed: int):
    s_rm = np.ascontiguousarray(s_rm)
    n = s_rm.shape[0]
    sizes = np.zeros(n, dtype=np.uintp)
    flags = np.zeros(n, dtype=np.uint8)
    nb = ref().ref_select_fraction(n, _ptr(s_rm), fraction, seed, _ptr(sizes), _ptr(flags))
    if nb < 0:
        raise RuntimeError(ref().ref_last_error().decode())
    return sizes[:nb].astype(np.uint8), flags[:nb].copy()


def ref_select_by_name(s_rm, name: str, k: int = 0):
    s_rm = np.ascontiguousarray(s_rm)
    n = s_rm.shape[0]
    sizes = np.zeros(n, dtype=np.uintp)
    flags = np.zeros(n, dtype=np.uint8)
    nb = ref().ref_select_by_name(n, _ptr(s_rm), name.encode(), k, _ptr(sizes), _ptr(flags))
    if nb < 0:
        raise RuntimeError(ref().ref_last_error().decode())
    return sizes[:nb].astype(np.uint8), flags[:nb].copy()


def ref_standardize_2x2(a, b, c, d):
    o = np.zeros(10)
    ref().ref_standardize_2x2(a, b, c, d, _ptr(o))
    return o


def ref_swap_adjacent_blocks(s, acc, pos, p, q) -> int:
    assert s.flags.f_contiguous and acc.flags.f_contiguous
    return ref().ref_swap_adjacent_blocks(s.shape[0], _ptr(s), acc.shape[0], _ptr(acc), pos, p, q)


def ref_window_reorder(w, sizes, sel):
    assert w.flags.f_contiguous
    d = w.shape[0]
    sz = np.asarray(sizes, dtype=np.uintp)
    sl = np.asarray(sel, dtype=np.uint8)
    nb = len(sz)
    acc = np.zeros((d, d), order="F")
    order = np.zeros(max(nb, 1), dtype=np.uintp)
    stuck = np.zeros(max(nb, 1), dtype=np.uint8)
    ex = ref().ref_window_reorder(d, _ptr(w), nb, _ptr(sz), _ptr(sl), _ptr(acc), _ptr(order),
                                  _ptr(stuck))
    return bool(ex), acc, order[:nb].astype(np.int64), stuck[:nb].astype(bool)


def ref_reorder_schur(s_rm, q_rm, flags, window_size=0, workers=0, tile=0, strict=False):
    """Runs the reference reorder_schur in place on row-major arrays."""
    n = s_rm.shape[0]
    assert s_rm.flags.c_contiguous and (q_rm is None or q_rm.flags.c_contiguous)
    flags = np.asarray(flags, dtype=np.uint8)
    nb = len(flags)
    perm = np.zeros(max(nb, 1), dtype=np.uintp)
    rej = np.zeros(max(nb, 1), dtype=np.uintp)
    nrej = _SZ(0)
    cap = 1 << 20
    plan = np.zeros(3 * cap, dtype=np.uintp)
    nplan = _SZ(0)
    clean = C.c_int(0)
    secs = C.c_double(0)
    _chk_ref(ref().ref_reorder_schur(n, tile, _ptr(s_rm), _ptr(q_rm), nb, _ptr(flags), window_size,
                                     workers, int(strict), _ptr(perm), _ptr(rej), C.byref(nrej),
                                     _ptr(plan), cap, C.byref(nplan), C.byref(clean),
                                     C.byref(secs)))
    k = min(nplan.value, cap)
    return dict(permutation=perm[:nb].astype(np.int64), rejected=rej[:nrej.value].astype(np.int64),
                plan=plan[:3 * k].reshape(k, 3).astype(np.int64), clean=bool(clean.value),
                seconds=secs.value)


class RefProblem:
    """A reorder problem resident in the reference's TiledMatrix form (built
    once from a column-major S); run() times reorder_schur alone."""

    def __init__(self, s_cm: np.ndarray, tile: int = 0):
        assert s_cm.flags.f_contiguous
        self.n = s_cm.shape[0]
        self.h = ref().ref_problem_create(self.n, tile, _ptr(s_cm))
        if not self.h:
            raise RuntimeError("reference: " + ref().ref_last_error().decode())

    def run(self, flags, window_size=0, workers=0, with_q=True):
        flags = np.asarray(flags, dtype=np.uint8)
        secs = C.c_double(0)
        nplan = _SZ(0)
        clean = C.c_int(0)
        _chk_ref(ref().ref_problem_reorder(self.h, len(flags), _ptr(flags), window_size, workers,
                                           int(with_q), C.byref(secs), C.byref(nplan), C.byref(clean)))
        return dict(seconds=secs.value, n_plan=nplan.value, clean=bool(clean.value))

    def close(self):
        if self.h:
            ref().ref_problem_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ref_backtransform(y_cm: np.ndarray, q_rm: np.ndarray, col_kind, workers=0) -> np.ndarray:
    """The reference's backtransform: X = Q Y, renormalised per column / pair."""
    n, k = y_cm.shape
    y_cm = np.asfortranarray(y_cm, dtype=np.float64)
    q_rm = np.ascontiguousarray(q_rm, dtype=np.float64)
    kind = np.ascontiguousarray(col_kind, dtype=np.int32)
    x = np.zeros((n, k), order="F")
    _chk_ref(ref().ref_backtransform(n, k, _ptr(y_cm), _ptr(q_rm), _ptr(kind), _ptr(x), workers))
    return x


REF_IO_TOOL = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref", "ref_io_tool")


def ref_io_convert(in_fmt: str, src: str, out_fmt: str, dst: str) -> None:
    """The reference's read_matrix_file(src, in_fmt) -> write_matrix_file(dst,
    ., out_fmt), in a subprocess (oracle/ref_io_tool.cpp)."""
    r = subprocess.run([REF_IO_TOOL, "convert", in_fmt, src, out_fmt, dst], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("reference io: " + r.stderr.strip())


def ref_hessenberg_reduce(a_rm, workers=0):
    n = a_rm.shape[0]
    a_rm = np.ascontiguousarray(a_rm)
    h = np.zeros((n, n))
    q = np.zeros((n, n))
    _chk_ref(ref().ref_hessenberg_reduce(n, _ptr(a_rm), _ptr(h), _ptr(q), workers))
    return h, q


def ref_schur_reduce(h_rm, q_rm=None, workers=0, deflation=1, shift_count=0, aed_window=0,
                     iteration_limit=0, small_threshold=0, tile=0):
    n = h_rm.shape[0]
    assert h_rm.flags.c_contiguous
    eig = np.zeros(2 * n)
    info = np.zeros(3, dtype=np.uintp)
    secs = C.c_double(0)
    _chk_ref(ref().ref_schur_reduce(n, tile, _ptr(h_rm), _ptr(q_rm), workers, deflation,
                                    shift_count, aed_window, iteration_limit, small_threshold,
                                    _ptr(eig), _ptr(info), C.byref(secs)))
    return dict(eigenvalues=eig[0::2] + 1j * eig[1::2], sweeps=int(info[0]),
                converged=bool(info[1]), converged_trailing=int(info[2]), seconds=secs.value)


def ref_small_schur(h):
    assert h.flags.f_contiguous
    k = h.shape[0]
    q = np.zeros((k, k), order="F")
    sw = _SZ(0)
    ok = ref().ref_small_schur(k, _ptr(h), _ptr(q), C.byref(sw))
    return bool(ok), q, sw.value


def ref_aed_step(h_rm, q_rm, l, ihi, window, deflation=1, tile=0):
    n = h_rm.shape[0]
    out = np.zeros(6, dtype=np.uintp)
    sh = np.zeros(2 * n)
    _chk_ref(ref().ref_aed_step(n, tile, _ptr(h_rm), _ptr(q_rm), l, ihi, window, deflation,
                                _ptr(out), _ptr(sh)))
    ns = int(out[5])
    return dict(window=int(out[0]), deflated=int(out[1]), spike_eliminated=bool(out[2]),
                converged=bool(out[3]), swap_rejected=bool(out[4]),
                shifts=sh[0:2 * ns:2] + 1j * sh[1:2 * ns:2])


def ref_sweep(h_rm, q_rm, l, ihi, shifts, window_size, tile=0):
    n = h_rm.shape[0]
    sh = np.zeros(2 * len(shifts))
    sh[0::2] = np.real(shifts)
    sh[1::2] = np.imag(shifts)
    _chk_ref(ref().ref_sweep(n, tile, _ptr(h_rm), _ptr(q_rm), l, ihi, len(shifts), _ptr(sh),
                             window_size))


def ref_similarity_residual(a_rm, q_rm, s_rm) -> float:
    a_rm, q_rm, s_rm = (np.ascontiguousarray(x) for x in (a_rm, q_rm, s_rm))
    return ref().ref_similarity_residual(a_rm.shape[0], _ptr(a_rm), _ptr(q_rm), _ptr(s_rm))


def ref_orthogonality_defect(q_rm) -> float:
    q_rm = np.ascontiguousarray(q_rm)
    return ref().ref_orthogonality_defect(q_rm.shape[0], _ptr(q_rm))


# --------------------------------------------------------------------------
# Schur reduction path (restatement of schur.cpp / kernels.cpp:223-381)

def small_schur(h: np.ndarray):
    """small_schur on a Fortran k x k array in place; returns (ok, q, sweeps)."""
    assert h.flags.f_contiguous
    k = h.shape[0]
    q = np.zeros((k, k), order="F")
    sw = _SZ(0)
    ok = lib().teo_small_schur(k, _ptr(h), _ptr(q), C.byref(sw))
    return bool(ok), q, sw.value


def deflation_check(spike, diag_sum, norm_stable, wnorm) -> bool:
    return bool(lib().teo_deflation_check(spike, diag_sum, int(norm_stable), wnorm))


def aed_step(h: np.ndarray, q, l, ihi, window, **opts):
    """aed_step (schur.cpp:599-609) on Fortran arrays in place."""
    n = h.shape[0]
    assert h.flags.f_contiguous and (q is None or q.flags.f_contiguous)
    o = schur_opts(**opts)
    r = AedOut()
    sh = np.zeros(2 * n + 4)
    rc = lib().teo_aed_step(n, _ptr(h), n, _ptr(q), n, l, ihi, window, C.byref(o), C.byref(r), _ptr(sh))
    if rc:
        raise ValueError("aed_step: bad arguments")
    ns = r.nshifts
    return dict(window=r.window, deflated=r.deflated, spike_eliminated=bool(r.spike_eliminated),
                converged=bool(r.converged), swap_rejected=bool(r.swap_rejected),
                shifts=sh[0:2 * ns:2] + 1j * sh[1:2 * ns:2])


def sweep(h: np.ndarray, q, l, ihi, shifts, window_size):
    """introduce_bulges + chase_bulges (schur.cpp:611-669) in place."""
    n = h.shape[0]
    sh = np.zeros(2 * len(shifts))
    sh[0::2] = np.real(shifts)
    sh[1::2] = np.imag(shifts)
    if lib().teo_sweep(n, _ptr(h), n, _ptr(q), n, l, ihi, len(shifts), _ptr(sh), window_size):
        raise ValueError("sweep: bad arguments")


def schur_reduce(h: np.ndarray, q=None, tile=0, **opts):
    """Serial schur_reduce (schur.cpp:671-906) in place on Fortran arrays."""
    n = h.shape[0]
    assert h.flags.f_contiguous and (q is None or q.flags.f_contiguous)
    o = schur_opts(**opts)
    info = SchurInfo()
    eig = np.zeros(2 * n)
    lib().teo_schur_reduce(n, _ptr(h), n, _ptr(q), n, tile, C.byref(o), _ptr(eig), C.byref(info))
    return dict(eigenvalues=eig[:n] + 1j * eig[n:], sweeps=info.sweeps, converged=bool(info.converged),
                converged_trailing=info.converged_trailing)


def ref_default_spectrum(n: int, seed: int) -> np.ndarray:
    """default_spectrum (generate.cpp:68-91) from the reference."""
    out = np.zeros(2 * n)
    ref().ref_default_spectrum(n, seed, _ptr(out))
    return out[0::2] + 1j * out[1::2]


# --------------------------------------------------------------------------
# C5 (generalized pair): the input T and the external oracle, LAPACK DTGSEN
# (scipy 1.18.1 / scipy-openblas 0.3.31.dev; the reference has no
# generalized path -- SURVEY.md 8c "C5: parity unpinned by the reference")

def pair_t(n: int, seed: int) -> np.ndarray:
    t = np.zeros((n, n), order="F")
    lib().teo_pair_t(n, seed, _ptr(t), n)
    return t


def lapack_tgsen(s, t, row_select):
    """DTGSEN (ijob=0): reorders the pencil so the selected eigenvalues lead,
    keeping the relative order inside both groups.  Returns (S, T, Q, Z,
    eigenvalues alpha/beta in diagonal order)."""
    from scipy.linalg import lapack
    n = s.shape[0]
    q = np.eye(n, order="F")
    z = np.eye(n, order="F")
    a, b, ar, ai, be, qs, zs, m, pl, pr, dif, info = lapack.dtgsen(
        np.asarray(row_select, dtype=np.int32), np.asfortranarray(s), np.asfortranarray(t), q, z, ijob=0)
    if info != 0:
        raise RuntimeError(f"dtgsen info={info}")
    return a, b, qs, zs, (ar + 1j * ai) / be


def pencil_eigenvalues(s, t) -> np.ndarray:
    """Generalized eigenvalues of the quasi-triangular pencil's diagonal
    blocks, in diagonal order (2x2 blocks: roots of det(S_b - l T_b))."""
    n = s.shape[0]
    out = np.zeros(n, dtype=complex)
    i = 0
    while i < n:
        if i + 1 < n and s[i + 1, i] != 0.0:
            A = s[i:i + 2, i:i + 2]
            B = t[i:i + 2, i:i + 2]
            c2 = B[0, 0] * B[1, 1] - B[0, 1] * B[1, 0]
            c1 = -(A[0, 0] * B[1, 1] + A[1, 1] * B[0, 0] - A[0, 1] * B[1, 0] - A[1, 0] * B[0, 1])
            c0 = A[0, 0] * A[1, 1] - A[0, 1] * A[1, 0]
            r = np.roots([c2, c1, c0])
            r = sorted(r, key=lambda z: -z.imag)
            out[i], out[i + 1] = r[0], r[1]
            i += 2
        else:
            out[i] = s[i, i] / t[i, i]
            i += 1
    return out
