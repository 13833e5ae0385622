import sys, time, torch
sys.path.insert(0, ".")
import paper_2002_05024_b200 as T
n = 10000
dev = torch.device("cuda", 0)
S0 = T.gen_schur_input(n, T.known_spectrum_seed(1), device=dev)
sel = T.select_fraction(S0, 0.35, 99)
T.set_memory_retention(True)
S = T.colmajor_empty(n, dev); Q = T.colmajor_empty(n, dev); Q0 = T.identity(n, dev)
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    S.copy_(S0); Q.copy_(Q0); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    r = T.reorder_schur(S, Q, sel, T.ReorderOptions(window_size=128))
    e1.record(); t1 = time.perf_counter(); torch.cuda.synchronize()
    print(f"call {it}: events {e0.elapsed_time(e1):.1f} ms, host wall {1e3*(t1-t0):.1f} ms, plan_ms {r.info['plan_ms']:.2f}")
