"""Time reorder_schur (Q accumulated, 35 % selected, window 128) with CUDA
events, with and without the look-ahead schedule.
Usage: python tools/reorder_time.py [n] [calls]"""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2002_05024_b200 as T  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = torch.device("cuda", 0)
S0 = T.gen_schur_input(n, T.known_spectrum_seed(1), device=dev)
sel = T.select_fraction(S0, 0.35, 99)
S = T.colmajor_empty(n, dev)
Q0 = T.identity(n, dev)
Q = T.colmajor_empty(n, dev)
T.set_memory_retention(True)
for la in ("0", "1", "0", "1"):
    os.environ["TEIG_NO_LOOKAHEAD"] = la
    ms = []
    for c in range(calls):
        S.copy_(S0)
        Q.copy_(Q0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = T.reorder_schur(S, Q, sel, T.ReorderOptions(window_size=128))
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    print(f"n={n} lookahead={'off' if la == '1' else 'on'}: " + " ".join(f"{m:.1f}" for m in ms) + " ms", flush=True)
