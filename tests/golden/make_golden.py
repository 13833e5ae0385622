#!/usr/bin/env python3
"""Generates tests/golden/reference_golden.npz from the UNMODIFIED reference
(oracle/_ref/libtaskeig_ref.so, built from /root/reference/proj/src by
oracle/Makefile).  Run in the build container (where /root/reference
exists); the committed .npz travels to the GPU box, the reference does not.

Contents (all from the reference itself):
  * Philox4x32-10 block outputs (test_generators.cpp:12-21 inputs)
  * standardize_2x2 on the 400 random blocks of test_kernels.cpp:106-110
  * swap_adjacent_blocks on the 200 random windows of test_kernels.cpp:292-339
  * window_reorder on the [1, 2x2, 1] window of test_reorder.cpp:66-99
  * reorder_schur of the SURVEY.md 8d synthetic Schur form, n=150 ws=24 and
    n=300 ws=64, with Q: S, Q, permutation, plan
  * select_fraction flags of the n=2000 synthetic input (seed 99)
  * schur_reduce of generate(hessenberg_random, n=80, seed=3): eigenvalues
  * the Schur path: small_schur (k=30), aed_step (n=100, w=16, both
    deflation conditions), a windowed sweep (n=64, 6 shifts, window 16),
    the perfect-shift problem (n=24) and the known-spectrum pipeline
    (n=150: A, hessenberg_reduce's H and Q, true spectrum, eigenvalues),
    schur_reduce eigenvalues of generate(hessenberg_random, 300, 1)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
from oracle import oracle as O  # noqa: E402


def philox_uniform_sym(seed, count):
    """Draws from the reference's Philox stream (via the shim)."""
    import ctypes as C
    out = np.zeros(count)
    O.ref().ref_philox_uniform_sym(seed, count, out.ctypes.data_as(C.c_void_p))
    return out


def main():
    if not O.ref_available():
        O.build(ref=True)
    g = {}
    kat_in = [([0, 0, 0, 0], [0, 0]),
              ([0xffffffff] * 4, [0xffffffff] * 2),
              ([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0xa4093822, 0x299f31d0])]
    g["philox_ctr"] = np.array([k[0] for k in kat_in], dtype=np.uint32)
    g["philox_key"] = np.array([k[1] for k in kat_in], dtype=np.uint32)
    g["philox_out"] = np.array([O.ref_philox_round10(c, k) for c, k in kat_in], dtype=np.uint32)

    # standardize_2x2 inputs: Philox(seed*13+5), four uniform_sym draws
    ins, outs = [], []
    for seed in range(400):
        a, b, c, d = philox_uniform_sym(seed * 13 + 5, 4)
        ins.append([a, b, c, d])
        outs.append(O.ref_standardize_2x2(a, b, c, d))
    g["std2_in"] = np.array(ins)
    g["std2_out"] = np.array(outs)

    # swap windows (test_kernels.cpp:292-339 construction, re-drawn here with
    # numpy so the fixture is self-contained; the reference does the swap)
    rng = np.random.default_rng(31337)
    sw_in, sw_out, sw_acc, sw_pq, sw_st = [], [], [], [], []
    for _ in range(200):
        p, q = int(rng.integers(1, 3)), int(rng.integers(1, 3))
        dd = p + q
        s = np.zeros((4, 4))
        def put(at, sz):
            if sz == 1:
                s[at, at] = 2.0 * rng.uniform(-1, 1)
            else:
                re, im = rng.uniform(-1, 1), 0.2 + rng.uniform(0, 1)
                s[at, at] = re; s[at + 1, at + 1] = re; s[at, at + 1] = im; s[at + 1, at] = -im
        put(0, p); put(p, q)
        for j in range(p, dd):
            for i in range(p):
                s[i, j] = rng.uniform(-1, 1)
        w = np.asfortranarray(s[:dd, :dd].copy())
        acc = np.asfortranarray(np.eye(dd))
        st = O.ref_swap_adjacent_blocks(w, acc, 0, p, q)
        sw_in.append(s.copy())
        o = np.zeros((4, 4)); o[:dd, :dd] = w
        a = np.zeros((4, 4)); a[:dd, :dd] = acc
        sw_out.append(o); sw_acc.append(a); sw_pq.append([p, q]); sw_st.append(st)
    g["swap_in"] = np.array(sw_in); g["swap_out"] = np.array(sw_out); g["swap_acc"] = np.array(sw_acc)
    g["swap_pq"] = np.array(sw_pq); g["swap_status"] = np.array(sw_st)

    # window_reorder example of test_reorder.cpp:66-99
    w = np.zeros((4, 4), order="F")
    w[0, 0] = 4.0; w[1, 1] = 1.0; w[1, 2] = 2.0; w[2, 1] = -2.0; w[2, 2] = 1.0
    w[0, 1] = 0.3; w[0, 2] = -0.1; w[0, 3] = 0.9; w[1, 3] = 0.2; w[2, 3] = -0.5; w[3, 3] = 7.0
    g["wr_in"] = w.copy()
    ex, acc, order, stuck = O.ref_window_reorder(w, [1, 2, 1], [0, 0, 1])
    g["wr_out"] = w.copy(); g["wr_acc"] = acc; g["wr_order"] = order; g["wr_executed"] = np.array(ex)

    # full reorders
    for n, ws in ((150, 24), (300, 64)):
        s = O.schur_input(n, O.known_spectrum_seed(1))
        sizes = O.scan_blocks(s)
        flags = O.select_fraction(len(sizes), 0.35, 99)
        s_rm = np.ascontiguousarray(s)
        q_rm = np.eye(n)
        r = O.ref_reorder_schur(s_rm, q_rm, flags, window_size=ws, workers=1)
        g[f"ro{n}_in"] = s
        g[f"ro{n}_flags"] = flags
        g[f"ro{n}_ws"] = np.array(ws)
        g[f"ro{n}_s"] = s_rm
        g[f"ro{n}_q"] = q_rm
        g[f"ro{n}_perm"] = r["permutation"]
        g[f"ro{n}_plan"] = r["plan"]
        g[f"ro{n}_clean"] = np.array(r["clean"])

    s = O.schur_input(2000, O.known_spectrum_seed(1))
    _, flags = O.ref_select_fraction(np.ascontiguousarray(s), 0.35, 99)
    g["sel2000_flags"] = flags

    h = O.ref_generate(4, 80, 3)
    g["hess80"] = h
    hh = h.copy()
    r = O.ref_schur_reduce(hh, None, workers=1)
    g["hess80_eig"] = r["eigenvalues"]
    g["hess80_s"] = hh
    # Schur path (schur.cpp / kernels.cpp:260-381), all from the reference
    h = np.asfortranarray(O.ref_generate(4, 30, 5))
    g["ss30_in"] = h.copy()
    ok, q, sw = O.ref_small_schur(h)
    g["ss30_s"], g["ss30_q"], g["ss30_sweeps"] = h, q, np.array(sw)
    h = O.ref_generate(4, 100, 13)
    g["aed100_in"] = h.copy()
    for cond in (0, 1):
        hh, qq = h.copy(), np.eye(100)
        r = O.ref_aed_step(hh, qq, 0, 100, 16, deflation=cond, tile=32)
        g[f"aed100_c{cond}_s"], g[f"aed100_c{cond}_q"] = hh, qq
        g[f"aed100_c{cond}_deflated"] = np.array(r["deflated"])
        g[f"aed100_c{cond}_shifts"] = np.asarray(r["shifts"], dtype=complex)
    h = O.ref_generate(4, 64, 37)
    g["sw64_in"] = h.copy()
    sh = np.array([0.2 * j + 1j * (1.0 + j) for j in range(3) for _ in (0,)])
    shifts = []
    for z in sh:
        shifts += [z, np.conj(z)]
    hh, qq = h.copy(), np.eye(64)
    O.ref_sweep(hh, qq, 0, 64, shifts, 16, tile=8)
    g["sw64_shifts"] = np.asarray(shifts)
    g["sw64_s"], g["sw64_q"] = hh, qq
    # perfect-shift problem (test_schur.cpp:238-257): Hessenberg form + shifts
    a = O.ref_generate(3, 24, 3)
    hr, _ = O.ref_hessenberg_reduce(a)
    sp = O.ref_default_spectrum(24, 3)
    z = next(x for x in sp if x.imag > 0)
    g["ps24_a"], g["ps24_h"], g["ps24_shifts"] = a, hr, np.array([z, np.conj(z)])
    # known-spectrum pipeline n=150 (test_schur.cpp:281-301): A, its
    # Hessenberg form and Q, the true spectrum, the reference's eigenvalues
    a = O.ref_generate(1, 150, 17)
    hr, qr = O.ref_hessenberg_reduce(a)
    g["ks150_a"], g["ks150_h"], g["ks150_q"] = a, hr, qr
    g["ks150_true"] = O.ref_default_spectrum(150, 17)
    hh, qq = hr.copy(), qr.copy()
    r = O.ref_schur_reduce(hh, qq, workers=1)
    g["ks150_eig"] = r["eigenvalues"]
    # schur_reduce of random Hessenberg n=300 (seed 1): eigenvalues
    h = O.ref_generate(4, 300, 1)
    hh = h.copy()
    r = O.ref_schur_reduce(hh, None, workers=1)
    g["hess300_eig"] = r["eigenvalues"]
    g["hess300_sweeps"] = np.array(r["sweeps"])
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **g)
    print("wrote", os.path.join(HERE, "reference_golden.npz"), sorted(g))


if __name__ == "__main__":
    main()
