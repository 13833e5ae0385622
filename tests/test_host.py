"""CPU tests of the product's host side: the C ABI library loads and exports
every declared symbol, the host planner/scheduler matches the reference's
plan, selections mirror the reference, argument validation (no GPU needed)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "taskeig_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(teig_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol(T):
    from paper_2002_05024_b200 import _native as N
    syms = header_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(N.lib(), s), s
        assert s in N.SIGNATURES, f"{s} declared but not bound"


def test_library_is_sm100a_only(T):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", T._native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_select_fraction_matches_reference(T, O, golden):
    s = O.schur_input(2000, O.known_spectrum_seed(1))
    sel = T.select_fraction(s, 0.35, 99)
    assert np.array_equal(sel.flags_array(), golden["sel2000_flags"])
    assert sum(sel.flags) == int(0.35 * len(sel.blocks))


@pytest.mark.parametrize("n", [150, 300])
def test_planner_matches_reference_plan(T, O, golden, n):
    s = golden[f"ro{n}_in"]
    sel = T.select_eigenvalues(s, list(golden[f"ro{n}_flags"].astype(bool)))
    win, nl, ng, fl = T.plan_reorder(n, sel, int(golden[f"ro{n}_ws"]))
    ref_plan = golden[f"ro{n}_plan"]  # (position, extent, moved_blocks) per window
    assert len(win) == len(ref_plan)
    assert np.array_equal(win[:, 0], ref_plan[:, 0])
    assert np.array_equal(win[:, 1] - win[:, 0], ref_plan[:, 1])
    assert np.array_equal(win[:, 2], ref_plan[:, 2])


@pytest.mark.parametrize("n,ws", [(2000, 64), (2000, 128), (4000, 64)])
def test_planner_matches_oracle_and_levels_are_valid(T, O, n, ws):
    s = O.schur_input(n, O.known_spectrum_seed(1))
    sel = T.select_fraction(s, 0.35, 99)
    win, nl, ng, fl = T.plan_reorder(n, sel, ws)
    pl, fl2, ng2 = O.plan_reorder(sel.sizes_array(), sel.flags_array(), ws, n)
    assert np.array_equal(win[:, :2], pl[:, :2]) and ng == ng2 and fl == fl2
    # wavefront levels: disjoint inside a level; overlapping windows keep plan order
    lv = win[:, 4]
    assert lv.max() + 1 == nl
    last = np.full(n, -1)
    for (a, b, _, _, l) in win:
        assert last[a:b].max() < l
        last[a:b] = l
    for L in range(nl):
        w = win[lv == L]
        w = w[np.argsort(w[:, 0])]
        assert np.all(w[1:, 0] >= w[:-1, 1])
    # chains pipeline: far fewer wavefronts than windows
    assert nl < len(win) / 4


def test_selection_api_errors(T):
    s = np.array([[1.0, 2.0], [-2.0, 1.0]])  # test_reorder.cpp:43-49
    with pytest.raises(ValueError):
        T.select_eigenvalues(s, lambda z: z.imag > 0.0)
    d = np.array([[-1.0, 0.5], [0.0, 2.0]])  # test_reorder.cpp:32-41
    sel = T.select_eigenvalues(d, lambda z: z.real > 0.0)
    assert sel.flags == [False, True] and sel.blocks[0].eigenvalue == complex(-1.0, 0.0)
    with pytest.raises(ValueError):
        T.select_eigenvalues(d, [True])
    with pytest.raises(ValueError):
        T.select_fraction(d, 1.5, 0)
    with pytest.raises(ValueError):
        T.select_by_name(d, "nope")
    n = 100
    dd = np.diag(1.0 + np.arange(n))
    sel = T.select_fraction(dd, 0.35, 7)  # test_reorder.cpp:51-64
    assert sum(sel.flags) == 35
    assert sel.flags == T.select_fraction(dd, 0.35, 7).flags
    assert sel.flags != T.select_fraction(dd, 0.35, 8).flags


def test_c_abi_argument_validation_without_gpu(T):
    from paper_2002_05024_b200 import _native as N
    L = N.lib()
    sizes = np.ones(3, dtype=np.uint8)
    flags = np.zeros(3, dtype=np.uint8)
    vp = lambda a: a.ctypes.data_as(C.c_void_p)
    assert L.teig_reorder_schur_device(0, None, 0, None, 0, 0, None, None, None, None, None, None, 0,
                                       None, None) == -1
    dummy = C.c_void_p(16)
    assert L.teig_reorder_schur_device(3, dummy, 2, None, 3, 3, vp(sizes), vp(flags), None, None, None,
                                       None, 0, None, None) == -3
    bad = np.array([1, 3, 1], dtype=np.uint8)
    assert L.teig_reorder_schur_device(5, dummy, 5, None, 5, 3, vp(bad), vp(flags), None, None, None,
                                       None, 0, None, None) == -8
    assert L.teig_reorder_schur_device(4, dummy, 4, None, 4, 3, vp(sizes), vp(flags), None, None, None,
                                       None, 0, None, None) == -8
    # window sizes beyond one CTA's shared memory run at 128 (the reference takes
    # any size): the planner shows the clamp without a device
    n = 2000
    sz = np.ones(n, dtype=np.uint8)
    fl = (np.arange(n) % 3 == 0).astype(np.uint8)
    w1 = np.zeros(5 * 100000, dtype=np.int64)
    w2 = np.zeros(5 * 100000, dtype=np.int64)
    k1 = L.teig_plan_reorder(n, n, vp(sz), vp(fl), 256, vp(w1), 100000, None, None, None)
    k2 = L.teig_plan_reorder(n, n, vp(sz), vp(fl), 128, vp(w2), 100000, None, None, None)
    assert k1 == k2 > 0 and np.array_equal(w1[:5 * k1], w2[:5 * k2])
    # python mirror validates the selection before touching the device
    sel = T.select_eigenvalues(np.diag([1.0, 2.0, 3.0]), [True, False, False])
    sel.blocks[1].start = 5
    with pytest.raises(ValueError):
        T.reorder_schur(np.diag([1.0, 2.0, 3.0]), None, sel)


def test_schur_and_pair_c_abi_validation_without_gpu(T):
    """Argument checks of the Schur / generalized / per-step entry points run
    before any device work and return the LAPACK-style codes the C++ layer
    maps onto the reference's exceptions (schur.cpp:601, 614-626)."""
    from paper_2002_05024_b200 import _native as N
    L = N.lib()
    dummy = C.c_void_p(16)
    o = N.SchurOpts()
    L.teig_schur_opts_default(C.byref(o))
    assert o.deflation == 1 and o.small_threshold == 64
    assert L.teig_schur_reduce_device(0, dummy, 1, None, 1, None, None, None, None, None) == -1
    assert L.teig_schur_reduce_device(4, None, 4, None, 4, None, None, None, None, None) == -2
    assert L.teig_schur_reduce_device(4, dummy, 3, None, 4, None, None, None, None, None) == -3
    o.deflation = 3
    assert L.teig_schur_reduce_device(200, dummy, 200, None, 200, C.byref(o), None, None, None, None) == -7
    # aed_step: window < 4 is invalid (schur.cpp:601)
    assert L.teig_aed_step_device(50, dummy, 50, None, 50, 0, 50, 3, None, None, None, None) == -8
    # introduce_bulges: the reference's std::invalid_argument cases (schur.cpp:614-626)
    sh = np.array([1.0, 0.0], dtype=np.float64)
    vp = lambda a: a.ctypes.data_as(C.c_void_p)
    assert L.teig_introduce_bulges_device(12, dummy, 12, None, 12, 0, 12, 1, vp(sh), None, None) == -8
    sh3 = np.array([1.0, 0.0, 2.0, 0.0, 3.0, 0.0], dtype=np.float64)
    assert L.teig_introduce_bulges_device(12, dummy, 12, None, 12, 0, 12, 3, vp(sh3), None, None) == -8
    nc = np.array([1.0, 2.0, 1.0, 2.0], dtype=np.float64)  # (1+2i, 1+2i): not conjugate
    assert L.teig_introduce_bulges_device(12, dummy, 12, None, 12, 0, 12, 2, vp(nc), None, None) == -8
    many = np.zeros(2 * 8)
    assert L.teig_introduce_bulges_device(12, dummy, 12, None, 12, 0, 12, 8, vp(many), None, None) == -8
    # chase_bulges: positions must be the introduced chain (bottom first, 3 apart)
    pos = np.array([10, 5], dtype=np.int64)
    assert L.teig_chase_bulges_device(20, dummy, 20, None, 20, 20, 2, vp(pos), 16, None, None) == -8
    assert L.teig_small_schur_device(200, dummy, 200, dummy, None, None) == -1001
    # generalized pair: window <= 64, selection must match
    sizes = np.ones(3, dtype=np.uint8)
    flags = np.zeros(3, dtype=np.uint8)
    ro = N.ReorderOpts()
    L.teig_reorder_opts_default(C.byref(ro))
    assert L.teig_greorder_schur_device(4, dummy, 4, dummy, 4, None, 4, None, 4, 3, vp(sizes), vp(flags),
                                        None, None, None, None, None) == -8
    assert L.teig_greorder_schur_device(3, dummy, 3, None, 3, None, 3, None, 3, 3, vp(sizes), vp(flags),
                                        None, None, None, None, None) == -2


def test_deflation_check_c_abi(T):
    eps = 2.220446049250313e-16
    assert T.deflation_check(0.0, 1.0, T.DeflationCondition.classic, 1.0)
    assert not T.deflation_check(1.0, 1.0, T.DeflationCondition.norm_stable, 1.0)
    assert T.deflation_check(0.9 * eps, 1e-3, T.DeflationCondition.norm_stable, 1.0)
    assert not T.deflation_check(0.9 * eps, 1e-3, T.DeflationCondition.classic, 1.0)


def test_python_mirror_errors(T):
    import numpy as np
    with pytest.raises(ValueError):
        T.schur_reduce(np.zeros((3, 4)))
    with pytest.raises(ValueError):
        T.introduce_bulges(np.zeros((12, 12)), None, 0, 12, [1.0])
    with pytest.raises(ValueError):
        T.aed_step(np.zeros((12, 12)), None, 0, 12, 3)
