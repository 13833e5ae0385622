"""Time the host entry point (pinned host S, Q) at n with TEIG_HOST_PROF=1
breakdowns; checks the result against the device path.
Usage: TEIG_HOST_PROF=1 python tools/host_time.py [n] [calls]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2002_05024_b200 as T  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda", 0)
S0 = T.gen_schur_input(n, T.known_spectrum_seed(1), device=dev)
sel = T.select_fraction(S0, 0.35, 99)
T.set_memory_retention(True)
Sd, Qd = S0.clone(), T.identity(n, dev)
T.reorder_schur(Sd, Qd, sel, T.ReorderOptions(window_size=128))
Sh = torch.empty((n, n), dtype=torch.float64).pin_memory()
Qh = torch.empty((n, n), dtype=torch.float64).pin_memory()
for c in range(calls):
    Sh.copy_(S0.t().cpu())
    Qh.copy_(torch.eye(n, dtype=torch.float64))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    T.reorder.reorder_schur_host_buffers(Sh.numpy(), Qh.numpy(), n, sel, T.ReorderOptions(window_size=128))
    t1 = time.perf_counter()
    ok = torch.equal(Sh.to(dev).t(), Sd) and torch.equal(Qh.to(dev).t(), Qd)
    print(f"call {c}: {1e3 * (t1 - t0):.1f} ms, equals the device result: {ok}", flush=True)
