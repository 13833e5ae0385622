"""The reference's OWN tests, unmodified (proj/tests/test_reorder.cpp and
test_schur.cpp), run against the C++ drop-in on the B200: the reference's
reorder.o and schur.o replaced by paper_2002_05024_b200/cxx/taskeig_adapter.cpp
over libtaskeig_b200.so (tests/refcpp/Makefile).  Every case must pass:
KATs, pipelines, determinism across worker counts, the Fig-5 chain shape, the
chase dependence shape, non-convergence reporting."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "tests", "refcpp", "_build")


@pytest.mark.parametrize("name", ["reorder", "schur", "multi_gpu"])
def test_reference_suite_through_the_dropin(cuda, name):
    exe = os.path.join(BUILD, f"test_{name}_b200")
    if not os.path.exists(exe):
        pytest.fail(f"{exe} missing: build it in the build container (make -C tests/refcpp)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=1200)
    print(r.stdout)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    assert "failed: 0" in r.stdout
