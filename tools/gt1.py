import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2002_05024_b200 as T
from oracle import oracle as O
dev = 'cuda'
# 1. generator parity
for n in [10, 101, 500]:
    s_gpu = T.gen_schur_input(n, T.known_spectrum_seed(1)).cpu().numpy()
    s_cpu = O.schur_input(n, O.known_spectrum_seed(1))
    print("gen", n, np.array_equal(s_gpu, s_cpu))
    h_gpu = T.gen_hessenberg(n, 1).cpu().numpy()
    h_cpu = O.hessenberg_random(n, 1)
    print("hess", n, np.array_equal(h_gpu, h_cpu))
# 2. window reorder parity vs oracle on a window
rng = np.random.default_rng(0)
for n in [200, 1000, 2000]:
    S0 = O.schur_input(n, O.known_spectrum_seed(1))
    sizes = O.scan_blocks(S0); flags = O.select_fraction(len(sizes), 0.35, 99)
    Sc = S0.copy(order='F'); Qc = np.asfortranarray(np.eye(n))
    t = time.time(); ro = O.reorder_schur(Sc, Qc, sizes, flags, 64); tc = time.time() - t
    S = T.gen_schur_input(n, T.known_spectrum_seed(1)); Q = T.identity(n)
    sel = T.select_fraction(S, 0.35, 99)
    assert (sel.flags_array() == flags).all()
    torch.cuda.synchronize()
    t = time.time(); res = T.reorder_schur(S, Q, sel, T.ReorderOptions(window_size=64)); torch.cuda.synchronize(); tg = time.time() - t
    Sg = S.cpu().numpy(); Qg = Q.cpu().numpy()
    print(n, "cpu %.2fs gpu %.3fs" % (tc, tg), res.clean, res.info['n_windows'], res.info['n_levels'], "perm eq", res.permutation == list(ro['permutation']),
          "maxdiff S", np.abs(Sg - Sc).max(), "Q", np.abs(Qg - Qc).max())
    ev_g = O.read_eigenvalues(Sg); ev_c = O.read_eigenvalues(Sc)
    print("   eig maxrel", np.max(np.abs(ev_g - ev_c) / np.maximum(1, np.abs(ev_c))), "std", O.is_standardized(Sg))
    Sd = torch.from_numpy(S0).to(dev); Qd = torch.from_numpy(Qg).to(dev); Sgd = torch.from_numpy(Sg).to(dev)
    R = Sd - Qd @ Sgd @ Qd.T
    print("   resid", (torch.linalg.norm(R) / torch.linalg.norm(Sd)).item(), "orth", torch.linalg.norm(Qd.T @ Qd - torch.eye(n, device=dev, dtype=torch.float64)).item(), "10neps", 10*n*2.2e-16)
