"""Small generalized reorders (several seeds / fractions) for compute-sanitizer
runs of the generalized window kernel."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2002_05024_b200 as T  # noqa: E402

dev = torch.device("cuda", 0)
for n, seed, frac in [(200, 1, 0.35), (130, 3, 0.5), (64, 5, 0.6)]:
    s = T.gen_schur_input(n, T.known_spectrum_seed(seed), device=dev)
    t = T.gen_pair_t(n, 7, device=dev)
    sel = T.select_fraction(s, frac, 99)
    g = T.greorder_schur(s, t, T.identity(n, dev), T.identity(n, dev), sel, T.ReorderOptions(window_size=64))
    torch.cuda.synchronize()
    print("greorder", n, g.clean, flush=True)
