"""Time the C5 generalized reorder (n, window 64, Q and Z) with CUDA events;
prints per-call ms.  Usage: python tools/c5_time.py [n] [calls]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2002_05024_b200 as T  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda", 0)
S0 = T.gen_schur_input(n, T.known_spectrum_seed(1), device=dev)
T0 = T.gen_pair_t(n, 7, device=dev)
sel = T.select_fraction(S0, 0.35, 99)
for c in range(calls):
    S, Tm = S0.clone(), T0.clone()
    Q, Z = T.identity(n, dev), T.identity(n, dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = T.greorder_schur(S, Tm, Q, Z, sel, T.ReorderOptions(window_size=64))
    e1.record()
    torch.cuda.synchronize()
    print(f"call {c}: {e0.elapsed_time(e1):.1f} ms clean={r.clean}", flush=True)
