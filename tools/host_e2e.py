"""Time the host entry point (pinned buffers) phase by phase: TEIG_HOST_PROF=1."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2002_05024_b200 as T  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
s0 = T.gen_schur_input(n, T.known_spectrum_seed(1))
sel = T.select_fraction(s0, 0.35, 99)
Sh = torch.empty((n, n), dtype=torch.float64).pin_memory()
Qh = torch.empty((n, n), dtype=torch.float64).pin_memory()
for k in range(int(os.environ.get("CALLS", "3"))):
    Sh.copy_(s0.t())
    Qh.zero_()
    Qh.diagonal().fill_(1.0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    info = T.reorder.reorder_schur_host_buffers(Sh.numpy(), Qh.numpy(), n, sel, T.ReorderOptions())
    print(f"call {k}: {time.perf_counter() - t0:.3f} s plan_ms {info['plan_ms']:.1f} passes {info['n_passes']}",
          flush=True)
S, Q = T.colmajor_empty(n), T.colmajor_empty(n)
I = T.identity(n)
for k in range(int(os.environ.get("CALLS", "3"))):
    S.copy_(s0)
    Q.copy_(I)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = T.reorder_schur(S, Q, sel, T.ReorderOptions())
    torch.cuda.synchronize()
    print(f"device call {k}: {time.perf_counter() - t0:.3f} s plan_ms {r.info['plan_ms']:.1f}", flush=True)
d = torch.empty(n * n, dtype=torch.float64, device="cuda")
h = Sh.view(-1)
for name, f in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{name} {n * n * 8 / 1e9:.2f} GB in {dt * 1e3:.1f} ms = {n * n * 8 / dt / 1e9:.1f} GB/s")
