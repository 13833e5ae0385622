"""Times the device Hessenberg reduction (with Q1) at a given n, CUDA events."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2002_05024_b200 as T  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
g = torch.Generator(device="cuda").manual_seed(1)
A0 = (torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1).t().contiguous().t()
for rep in range(2):
    A = A0.clone()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = T.hessenberg_reduce(A, True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"n={n} rep={rep} {ms:.1f} ms  panels={r.info['panels']} launches={r.info['launches']} "
          f"flops={r.info['flops']:.3g} -> {r.info['flops'] / ms / 1e9:.2f} TF/s")
Q = r.q
back = float(torch.linalg.norm(A0 - Q @ A @ Q.t()) / torch.linalg.norm(A0))
orth = float(torch.linalg.norm(Q.t() @ Q - torch.eye(n, dtype=torch.float64, device="cuda")))
print(f"backward {back:.3e} orth {orth:.3e} bound {10 * n * 2.22e-16:.3e}")
