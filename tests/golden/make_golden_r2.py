#!/usr/bin/env python3
"""Round-2 golden fixtures from the UNMODIFIED reference (oracle/_ref):
tests/golden/r2_golden.npz.  Run in the build container.

  * backtransform (eigvec.cpp:448-516): X of random Y (n=300, k=41, mixed
    real columns and complex pairs) and a random orthogonal Q.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle import oracle as O  # noqa: E402


def bt_case(n=300, k=41, seed=5):
    rng = np.random.default_rng(seed)
    y = np.asfortranarray(rng.uniform(-1, 1, (n, k)))
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    kind = np.zeros(k, dtype=np.int32)
    j = 3
    while j + 1 < k:  # pairs at 3,4 / 8,9 / ...
        kind[j], kind[j + 1] = 1, 2
        j += 5
    return y, q, kind


def main():
    if not O.ref_available():
        O.build(ref=True)
    g = {}
    y, q, kind = bt_case()
    g["bt_y"], g["bt_q"], g["bt_kind"] = y, q, kind
    g["bt_x"] = O.ref_backtransform(y, q, kind, workers=1)
    np.savez_compressed(os.path.join(HERE, "r2_golden.npz"), **g)
    print("wrote", sorted(g))


if __name__ == "__main__":
    main()
