"""Stall-reason breakdown per CUDA source line from an ncu report
(source page, cuda,sass).  Usage: python tools/ncu_stalls.py REPORT [top]"""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
hdr = None
file = line = None
agg = collections.defaultdict(collections.Counter)
src = {}
for x in csv.reader(io.StringIO(out)):
    if not x:
        continue
    if x[0] == "File Path":
        file = x[1].split("/")[-1]
        continue
    if x[0] == "Function Name":
        continue
    if x[0] == "Line No":
        hdr = x
        continue
    if x[0] != "":
        line = (file, int(x[0]))
        src[line] = x[1]
        continue
    if x[2] in ("...", "-") or hdr is None:
        continue
    for k, v in zip(hdr, x):
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                agg[line][k[6:]] += int(v or 0)
            except ValueError:
                pass
tot = collections.Counter()
for c in agg.values():
    tot.update(c)
print("all:", ", ".join(f"{k} {v}" for k, v in tot.most_common(8)))
for l, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
    print(f"{sum(c.values()):6d} {l[0]}:{l[1]}  " + ", ".join(f"{k} {v}" for k, v in c.most_common(3)),
          "|", src.get(l, "").strip()[:60])
