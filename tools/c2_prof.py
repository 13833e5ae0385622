import sys, torch
sys.path.insert(0, ".")
import paper_2002_05024_b200 as T
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
dev = torch.device("cuda", 0)
S0 = T.gen_schur_input(n, T.known_spectrum_seed(1), device=dev)
sel = T.select_fraction(S0, 0.35, 99)
for prof in (False, True):
    S, Q = S0.clone(), T.identity(n, dev)
    r = T.reorder_schur(S, Q, sel, T.ReorderOptions(window_size=128, profile=prof, overlap_factor=not prof))
    i = r.info
    print(prof, {k: round(i[k], 2) for k in ("ms_window", "ms_left", "ms_right", "ms_factor", "n_levels", "n_windows")})
