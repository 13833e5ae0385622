import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

EPS = 2.220446049250313e-16


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(ROOT, "tests", "golden", "reference_golden.npz"))


@pytest.fixture(scope="session")
def O():
    from oracle import oracle
    oracle.lib()
    return oracle


@pytest.fixture(scope="session")
def T():
    import paper_2002_05024_b200 as T
    T.lib()  # raises if the native library is missing -- there is no fallback
    return T


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test collected on a machine without CUDA (run with -m 'not gpu' here)")
    return torch.device("cuda", 0)


@pytest.fixture(scope="session")
def golden_rej():
    return np.load(os.path.join(ROOT, "tests", "golden", "rejection_golden.npz"))


@pytest.fixture(scope="session")
def golden_r2():
    return np.load(os.path.join(ROOT, "tests", "golden", "r2_golden.npz"))
