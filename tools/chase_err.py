"""Forward difference of the GPU windowed chase vs the serial (reference-order)
restatement, for sizing the parity tolerance."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import paper_2002_05024_b200 as T
from oracle import oracle as O
from test_schur_gpu import dev, residuals
for n, seed, nsh, ws in [(12, 31, 2, 6), (64, 37, 6, 16), (300, 4, 16, 32), (700, 5, 64, 128), (700, 5, 8, 128)]:
    d = O.hessenberg_random(n, seed)
    rng = np.random.default_rng(seed)
    shifts = []
    for _ in range(nsh // 2):
        z = complex(rng.uniform(-1, 1), rng.uniform(0.1, 1))
        shifts += [z, z.conjugate()]
    h, q = dev(d), dev(np.eye(n))
    chain = T.introduce_bulges(h, q, 0, n, shifts)
    T.chase_bulges(h, q, chain, ws)
    ho, qo = np.asfortranarray(d.copy()), np.asfortranarray(np.eye(n))
    O.sweep(ho, qo, 0, n, shifts, ws)
    hn = h.cpu().numpy()
    b1, o1 = residuals(d, q, hn)
    b2, o2 = residuals(d, qo, ho)
    print(n, nsh, "dH/|H|", np.abs(hn - ho).max() / np.linalg.norm(d), "dQ", np.abs(q.cpu().numpy() - qo).max(),
          "back gpu/serial", b1, b2, "orth", o1, o2)
