#!/usr/bin/env python3
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv).

usage: launch_summary.py launches.csv [header comment...]
Prints per-kernel launches, total ms, mean us and the share of this
library's kernels (namespace teig::) in the summed teig kernel time.
ncu times are cold-cache and serialised: compare SHARES, not absolutes."""
import csv
import sys
from collections import defaultdict


def main(path, note=""):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    unit_i = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        u = r[unit_i] if unit_i is not None else "ns"
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(u, 1e-6)
        name = r[ki]
        tot[name] += v * scale
        cnt[name] += 1
    teig = sum(v for k, v in tot.items() if k.startswith("teig::") or "teig::" in k[:40])
    if note:
        print("#", note)
    print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare SHARES)")
    print(f"# {'kernel':48s} {'launches':>9s} {'total_ms':>10s} {'mean_us':>9s} {'share_of_teig':>13s}")
    for k in sorted(tot, key=lambda k: -tot[k]):
        share = tot[k] / teig if ("teig::" in k[:40]) and teig else float("nan")
        print(f"  {k[:48]:48s} {cnt[k]:9d} {tot[k]:10.3f} {1e3 * tot[k] / cnt[k]:9.1f} {share:13.3f}")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
