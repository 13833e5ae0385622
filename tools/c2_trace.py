"""Timeline of one C2 reorder (look-ahead schedule) from the library's trace:
per level, when the window kernel starts/ends and what sits between
consecutive window kernels.  Usage: python tools/c2_trace.py [n]"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2002_05024_b200 as T  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
dev = torch.device("cuda", 0)
S0 = T.gen_schur_input(n, T.known_spectrum_seed(1), device=dev)
sel = T.select_fraction(S0, 0.35, 99)
for it in range(2):
    S, Q = S0.clone(), T.identity(n, dev)
    T.trace_enable(it == 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    T.reorder_schur(S, Q, sel, T.ReorderOptions(window_size=128))
    e1.record()
    torch.cuda.synchronize()
    print("call", it, "ms", e0.elapsed_time(e1))
tr = json.loads(T.trace_json())
tasks = tr["tasks"]
win = {}
other = {}
for t in tasks:
    lab = t["label"]  # reorder:W:p0:l12
    parts = lab.split(":")
    cls, lvl = parts[1], int(parts[3][1:])
    if cls == "W":
        win[lvl] = (t["start_ns"], t["end_ns"])
    else:
        other.setdefault((cls, lvl, t["worker"]), []).append((t["start_ns"], t["end_ns"]))
L = sorted(win)
busy = sum(e - s for s, e in win.values())
span = win[L[-1]][1] - win[L[0]][0]
gaps = [win[L[i + 1]][0] - win[L[i]][1] for i in range(len(L) - 1)]
print(f"levels {len(L)}: window kernels {busy / 1e6:.1f} ms of a {span / 1e6:.1f} ms span; "
      f"gaps between consecutive windows: total {sum(gaps) / 1e6:.1f} ms, median {sorted(gaps)[len(gaps) // 2] / 1e3:.1f} us")
for lv in L[:3] + L[len(L) // 2:len(L) // 2 + 3]:
    s0 = win[lv][0]
    items = [("W", 0, win[lv][0], win[lv][1])]
    for (c, l2, w), v in other.items():
        if l2 in (lv, lv - 1):
            for a, b in v:
                items.append((f"{c}{l2}", w, a, b))
    items.sort(key=lambda x: x[2])
    print(f"level {lv}: " + "  ".join(f"{c}/w{w} {(a - s0) / 1e3:.0f}..{(b - s0) / 1e3:.0f}us" for c, w, a, b in items))
