"""The reference's OWN C++ tests and the C++ drop-in (CPU side, no GPU).

tests/refcpp builds proj/tests/test_reorder.cpp and test_schur.cpp (compiled
in place from the reference tree, unmodified) twice:
  *_ref   linked with every reference object -- pins tests/refcpp/doctest.h
          (the stand-in for the reference's absent vendored doctest) against
          the unmodified reference: every case passes here;
  *_b200  linked with the reference objects MINUS reorder.o / schur.o, plus
          the C++ adapter (paper_2002_05024_b200/cxx) and libtaskeig_b200.so
          -- the drop-in; run on the GPU by tests/test_refcpp_gpu.py.
Both need the reference tree (present in the build container only); on a
machine without it the prebuilt binaries travel with the snapshot."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "tests", "refcpp", "_build")
ADAPTER = os.path.join(ROOT, "paper_2002_05024_b200", "_lib", "taskeig_adapter.o")
REF_TREE = "/root/reference/proj"

# the 12 symbols of reorder.o + schur.o the adapter replaces
REPLACED = [
    "taskeig::reorder_schur(", "taskeig::select_by_name(", "taskeig::window_reorder(", "taskeig::select_fraction(",
    "taskeig::select_eigenvalues(taskeig::TiledMatrix const&, std::vector<bool",
    "taskeig::select_eigenvalues(taskeig::TiledMatrix const&, std::function<bool",
    "taskeig::Selection::selected_rows() const", "taskeig::chase_bulges(", "taskeig::schur_reduce(",
    "taskeig::deflation_check(", "taskeig::introduce_bulges(", "taskeig::aed_step(",
]


def _ensure_built(target):
    if os.path.isdir(REF_TREE):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "refcpp"), target], check=True)


def test_adapter_defines_every_replaced_symbol():
    if not os.path.exists(ADAPTER):
        if not os.path.isdir(REF_TREE):
            pytest.skip("adapter not built and no reference headers here")
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2002_05024_b200", "cxx")], check=True)
    out = subprocess.run(["nm", "-C", "--defined-only", ADAPTER], capture_output=True, text=True, check=True).stdout
    defined = [l.split(" T ", 1)[1] for l in out.splitlines() if " T " in l]
    for sym in REPLACED:
        assert any(d.startswith(sym) for d in defined), sym


@pytest.mark.parametrize("name", ["reorder", "schur"])
def test_reference_tests_pass_on_the_reference_with_the_doctest_standin(name):
    exe = os.path.join(BUILD, f"test_{name}_ref")
    if not os.path.exists(exe):
        if not os.path.isdir(REF_TREE):
            pytest.skip("reference tree absent")
        _ensure_built("ref")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "failed: 0" in r.stdout
