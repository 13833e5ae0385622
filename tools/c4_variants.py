"""A/B of the reorder step's scheduling options at one size (CUDA events,
3 warm-up + 3 timed steps each): profile events on/off, factor overlap on/off,
priority streams on/off (TEIG_NO_PRIO must be set in the environment)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, ".")
import paper_2002_05024_b200 as T  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
T.set_memory_retention(True)
dev = torch.device("cuda", 0)
S0 = T.gen_schur_input(n, T.known_spectrum_seed(1), device=dev)
sel = T.select_fraction(S0, 0.35, 99)
S = T.colmajor_empty(n, dev)
Q = T.colmajor_empty(n, dev)
I = T.identity(n, dev)
tag = "noprio" if os.environ.get("TEIG_NO_PRIO") == "1" else "prio"
for name, opts in (("default", T.ReorderOptions()), ("profile", T.ReorderOptions(profile=True)),
                   ("no-overlap", T.ReorderOptions(overlap_factor=False)),
                   ("full-factor", T.ReorderOptions(full_factor=True))):
    ms = []
    for k in range(6):
        S.copy_(S0)
        Q.copy_(I)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        T.reorder_schur(S, Q, sel, opts)
        e1.record()
        torch.cuda.synchronize()
        if k >= 3:
            ms.append(e0.elapsed_time(e1))
    print(f"n={n} {tag} {name}: {statistics.mean(ms):.1f} ms {[round(x, 1) for x in ms]}", flush=True)
