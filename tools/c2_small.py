"""One standard reorder (window 128, Q accumulated, 35 % selected) at a given n,
for launch lists / profiles.  Usage: python tools/c2_small.py [n]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2002_05024_b200 as T  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
dev = torch.device("cuda", 0)
S = T.gen_schur_input(n, T.known_spectrum_seed(1), device=dev)
sel = T.select_fraction(S, 0.35, 99)
r = T.reorder_schur(S, T.identity(n, dev), sel, T.ReorderOptions(window_size=128))
torch.cuda.synchronize()
print("clean", r.clean, r.info["n_windows"], r.info["n_levels"])
