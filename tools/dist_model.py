#!/usr/bin/env python3
"""Per-level critical-path model of the distributed reorder.

From the planner's windows and wavefront levels (teig_plan_reorder, the same
plan the drivers run), count every rank's update flops per level for
  * the shipped layout: S in column slabs (p_r = 1, p_c = p), balanced by
    teig_dist_balance; L updates spread over the ranks owning columns >= b,
    the R update of a window on the owner of column a;
  * 2-D block grids p_r x p_c (S blocks, R spread over the p_r process rows
    of a window's block column, L over the p_c process columns of its block
    row), boundaries chosen for equal work in each direction;
Q updates (half the flops) are row slabs over all p ranks in every layout and
run on a second stream.  Model of the step time in "flop units" (divide by
one GPU's update rate):
  critical = sum over levels of max over ranks of S-update flops  (levels are
             barriers for the window kernels: the S panel updates of level L
             gate level L+1's windows)
  per_rank = max over ranks of all its flops (S + Q)              (throughput)
  model    = max(critical, per_rank);  ideal = total / p.
Prints one JSON line per layout."""
import ctypes as C
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2002_05024_b200 import _native as N  # noqa: E402


def plan(n, ws, frac=0.35, seed=99):
    npairs = n // 4
    nreal = n - 2 * npairs
    sizes = np.array([1] * nreal + [2] * npairs, dtype=np.uint8)
    flags = np.zeros(len(sizes), dtype=np.uint8)
    vp = lambda a: a.ctypes.data_as(C.c_void_p)
    N.check(N.lib().teig_select_fraction(len(sizes), frac, seed, vp(flags)))
    cap = 400000
    win = np.zeros(5 * cap, dtype=np.int64)
    k = N.lib().teig_plan_reorder(n, len(sizes), vp(sizes), vp(flags), ws, vp(win), cap, None, None, None)
    return sizes, flags, win[:5 * k].reshape(k, 5)  # wtop, wbot, count, group, level


def balanced_bounds(weights, parts):
    """Boundaries splitting a 1-D work profile into `parts` equal pieces."""
    cum = np.concatenate([[0.0], np.cumsum(weights)])
    tot = cum[-1]
    b = [0]
    for g in range(1, parts):
        b.append(int(np.searchsorted(cum, tot * g / parts)))
    b.append(len(weights))
    return np.array(b)


def model(n, W, pr, pc, colb=None):
    a = W[:, 0].astype(np.int64)
    b = W[:, 1].astype(np.int64)
    lv = W[:, 4].astype(np.int64)
    d = (b - a).astype(np.float64)
    f2 = 2 * d * d
    nl = int(lv.max()) + 1
    p = pr * pc
    # column work profile (L: 2d^2 per column >= b; R: 2d^2 a spread over [a, b))
    colw = np.zeros(n + 1)
    np.add.at(colw, b, f2)
    colw = np.cumsum(colw)[:n]
    rr = np.zeros(n + 1)
    np.add.at(rr, a, f2 * a / d)
    np.add.at(rr, b, -f2 * a / d)
    colw += np.cumsum(rr)[:n]
    # row work profile: L rows [a, b) carry 2d (n - b) each; R rows [0, a) 2d^2 each
    roww = np.zeros(n + 1)
    np.add.at(roww, a, 2 * d * (n - b))
    np.add.at(roww, b, -2 * d * (n - b))
    rw = np.cumsum(roww)[:n]
    acc = np.zeros(n + 1)
    np.add.at(acc, a, f2)  # rows < a get 2d^2: suffix sums
    rw += np.cumsum(acc[::-1])[::-1][1:n + 1]
    Cb = colb if colb is not None else balanced_bounds(colw, pc)
    Rb = balanced_bounds(rw, pr) if pr > 1 else np.array([0, n])
    S = np.zeros((nl, pr, pc))
    for k in range(len(W)):
        ak, bk, L, w2 = a[k], b[k], lv[k], f2[k]
        ia = np.searchsorted(Rb, ak, side="right") - 1
        ja = np.searchsorted(Cb, ak, side="right") - 1
        # L: rows [a, b) (process row ia), columns [b, n) split by column blocks
        for j in range(pc):
            cols = max(0, Cb[j + 1] - max(Cb[j], bk))
            S[L, ia, j] += w2 * cols
        # R: rows [0, a) split by row blocks, process column ja
        for i in range(pr):
            rows = max(0, min(Rb[i + 1], ak) - Rb[i])
            S[L, i, ja] += w2 * rows
    Qtot = float((f2 * n).sum())
    Sr = S.reshape(nl, p)
    critical = float(Sr.max(axis=1).sum())
    per_rank = float((Sr.sum(axis=0) + Qtot / p).max())
    total = float(Sr.sum() + Qtot)
    return {"layout": f"{pr}x{pc}", "n": n, "ranks": p, "levels": nl, "total_flops": total,
            "ideal": total / p, "critical": critical, "per_rank": per_rank,
            "model": max(critical, per_rank), "efficiency": total / p / max(critical, per_rank)}


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
    ws = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    sizes, flags, W = plan(n, ws)
    for p, grids in ((1, [(1, 1)]), (2, [(1, 2), (2, 1)]), (4, [(1, 4), (2, 2)]), (8, [(1, 8), (2, 4), (4, 2)])):
        for pr, pc in grids:
            colb = None
            if pr == 1 and pc > 1:  # the shipped balancer
                cb = np.zeros(pc + 1, dtype=np.int64)
                rb = np.zeros(pc + 1, dtype=np.int64)
                vp = lambda x: x.ctypes.data_as(C.c_void_p)
                N.check(N.lib().teig_dist_balance(n, len(sizes), vp(sizes), vp(flags), ws, pc, vp(cb), vp(rb)))
                colb = cb
            r = model(n, W, pr, pc, colb)
            print(json.dumps({k: (round(v, 4) if isinstance(v, float) and v < 10 else v) for k, v in r.items()}))


if __name__ == "__main__":
    main()
