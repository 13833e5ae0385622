"""Time schur_reduce on the device (C3 workload shape) and check residuals.
usage: python tools/schur_time.py n [profile]"""
import sys
import time

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2002_05024_b200 as T  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
prof = len(sys.argv) > 2 and sys.argv[2] == "1"
h = T.gen_hessenberg(n, 1)
h0 = h.clone()
q = T.identity(n)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t = time.time()
e0.record()
res = T.schur_reduce(h, q, T.SchurOptions(profile=prof))
e1.record()
torch.cuda.synchronize()
wall = time.time() - t
R = h0 - q @ h @ q.t()
back = float(torch.linalg.norm(R) / torch.linalg.norm(h0))
orth = float(torch.linalg.norm(q.t() @ q - torch.eye(n, dtype=torch.float64, device="cuda")))
print(f"n={n} converged={res.converged} sweeps={res.sweeps} wall={wall:.3f}s event={e0.elapsed_time(e1)/1e3:.3f}s "
      f"backward={back:.2e} orth={orth:.2e} tol={10*n*2.22e-16:.2e}")
print({k: v for k, v in res.info.items()})
