"""One generalized (S, T) reorder with Q and Z (the C5 construction) at a given
n, for launch lists / profiles."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2002_05024_b200 as T  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8000
dev = torch.device("cuda", 0)
S = T.gen_schur_input(n, T.known_spectrum_seed(1), device=dev)
Tm = T.gen_pair_t(n, 7, device=dev)
sel = T.select_fraction(S, 0.35, 99)
r = T.greorder_schur(S, Tm, T.identity(n, dev), T.identity(n, dev), sel, T.ReorderOptions(window_size=64))
torch.cuda.synchronize()
print("clean", r.clean, r.info["n_windows"], r.info["n_levels"])
