import sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_2002_05024_b200 as T
n = int(sys.argv[1]); out = sys.argv[2]
dev = torch.device("cuda", 0)
H = T.gen_hessenberg(n, 1, device=dev); Q = T.identity(n, dev)
r = T.schur_reduce(H, Q)
np.save(out + "_h.npy", H.cpu().numpy()); np.save(out + "_q.npy", Q.cpu().numpy())
print("done", r.info.get("sweeps"))
