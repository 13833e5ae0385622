"""Loopback distributed reorder vs single GPU at one size (debug helper)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2002_05024_b200 as T  # noqa: E402
from paper_2002_05024_b200 import dist as D  # noqa: E402

n, world = int(sys.argv[1]), int(sys.argv[2])
s0 = T.gen_schur_input(n, T.known_spectrum_seed(1))
sel = T.select_fraction(s0, 0.35, 99)
s1, q1 = s0.clone(), T.identity(n)
T.reorder_schur(s1, q1, sel, T.ReorderOptions(window_size=128))
s2, q2 = s0.clone(), T.identity(n)
D.reorder_schur_loopback(s2, q2, sel, world, T.ReorderOptions(window_size=128))
print("bitwise", torch.equal(s1, s2), torch.equal(q1, q2))
