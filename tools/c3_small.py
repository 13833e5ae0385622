"""One schur_reduce (Q accumulated) of generate(hessenberg_random, n, seed 1)
with event timing; for profiles.  Usage: python tools/c3_small.py [n] [calls]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2002_05024_b200 as T  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 1
dev = torch.device("cuda", 0)
H0 = T.gen_hessenberg(n, 1, device=dev)
for c in range(calls):
    H = T.colmajor_empty(n, dev)
    H.copy_(H0)
    Q = T.identity(n, dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = T.schur_reduce(H, Q, T.SchurOptions(profile=True))
    e1.record()
    torch.cuda.synchronize()
    i = r.info
    print(f"call {c}: {e0.elapsed_time(e1):.1f} ms sweeps={i.get('sweeps')} window_ms={i.get('ms_window'):.1f} "
          f"update_ms={i.get('ms_update'):.1f}", flush=True)
