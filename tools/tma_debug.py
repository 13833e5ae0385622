"""Small reorder run through the TMA update kernels (debug helper)."""
import sys

import os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2002_05024_b200 as T

n = int(sys.argv[1]) if len(sys.argv) > 1 else 600
s0 = T.gen_schur_input(n, T.known_spectrum_seed(1))
sel = T.select_fraction(s0, 0.35, 99)
s1, q1 = s0.clone(), T.identity(n)
r = T.reorder_schur(s1, q1, sel, T.ReorderOptions(window_size=128))
torch.cuda.synchronize()
back = float(torch.linalg.norm(s0 - q1 @ s1 @ q1.t()) / torch.linalg.norm(s0))
print("n", n, "clean", r.clean, "backward", back)
