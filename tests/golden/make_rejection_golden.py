#!/usr/bin/env python3
"""Generates tests/golden/rejection_golden.npz from the UNMODIFIED reference
(oracle/_ref/libtaskeig_ref.so) on the rejection scenarios of
tests/rejection_cases.py whose reference run is well defined (it terminates
and its bookkeeping describes its matrix): permutation, rejected_blocks,
clean and the output's eigenvalue read-off.  Run in the build container."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
sys.path.insert(0, os.path.join(HERE, ".."))
from oracle import oracle as O  # noqa: E402
import rejection_cases as RC  # noqa: E402


def main():
    if not O.ref_available():
        O.build(ref=True)
    g = {}
    for name in RC.REF_WELL_DEFINED:
        S, sizes, flags, ws = RC.case(name)
        n = S.shape[0]
        s_rm = np.ascontiguousarray(S.copy())
        q_rm = np.ascontiguousarray(np.eye(n))
        r = O.ref_reorder_schur(s_rm, q_rm, flags, window_size=ws, workers=1)
        assert RC.consistent(S, sizes, r["permutation"], s_rm, O.read_eigenvalues)
        g[f"{name}_perm"] = r["permutation"]
        g[f"{name}_rejected"] = r["rejected"]
        g[f"{name}_clean"] = np.array(r["clean"])
        g[f"{name}_eig"] = O.read_eigenvalues(s_rm)
        g[f"{name}_S_in"] = S
    np.savez_compressed(os.path.join(HERE, "rejection_golden.npz"), **g)
    print("wrote", sorted(g))


if __name__ == "__main__":
    main()
