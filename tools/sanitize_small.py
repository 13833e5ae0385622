"""Small runs of every kernel family, for compute-sanitizer (racecheck /
synccheck / memcheck): window_reorder + bulk-copy and cp.async DMMA updates
(reorder with ws 64 and 128), the AED / small-solve and chase windows
(schur_reduce), the generalized window kernel, the Hessenberg column kernels
and DMMA GEMMs, the back-transformation."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2002_05024_b200 as T  # noqa: E402

dev = torch.device("cuda", 0)
for n, ws in ((300, 64), (520, 128)):
    s = T.gen_schur_input(n, T.known_spectrum_seed(1), device=dev)
    q = T.identity(n, dev)
    sel = T.select_fraction(s, 0.35, 99)
    r = T.reorder_schur(s, q, sel, T.ReorderOptions(window_size=ws))
    print("reorder", n, ws, r.clean, flush=True)
h = T.gen_hessenberg(200, 1, device=dev)
q = T.identity(200, dev)
sd = T.schur_reduce(h, q)
print("schur", sd.converged, flush=True)
s = T.gen_schur_input(260, T.known_spectrum_seed(1), device=dev)
t = T.gen_pair_t(260, 7, device=dev)
sel = T.select_fraction(s, 0.35, 99)
g = T.greorder_schur(s, t, T.identity(260, dev), T.identity(260, dev), sel, T.ReorderOptions(window_size=64))
print("greorder", g.clean, flush=True)
a = torch.rand(300, 300, dtype=torch.float64, device=dev).t().contiguous().t()
hr = T.hessenberg_reduce(a, True)
print("hessenberg", hr.info["panels"], flush=True)
y = torch.rand(300, 17, dtype=torch.float64, device=dev)
x = T.backtransform(y, hr.q, [0] * 17)
torch.cuda.synchronize()
print("backtransform ok", flush=True)
