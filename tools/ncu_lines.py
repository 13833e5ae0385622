"""Aggregate an ncu report's source page (cuda,sass) by CUDA source line:
warp-stall samples and executed warp instructions.
Usage: python tools/ncu_lines.py REPORT.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
samp, inst, src = collections.Counter(), collections.Counter(), {}
file = line = None
for x in csv.reader(io.StringIO(out)):
    if not x:
        continue
    if x[0] == "File Path":
        file = x[1].split("/")[-1]
        continue
    if x[0] in ("Function Name", "Line No"):
        continue
    if x[0] != "":
        line = (file, int(x[0]))
        src[line] = x[1]
        continue
    if x[2] in ("...", "-"):
        continue
    try:
        samp[line] += int(x[4])
        inst[line] += int(x[7])
    except (ValueError, IndexError):
        pass
tot = sum(samp.values())
print(f"samples {tot}  warp instructions {sum(inst.values())}")
for k, v in samp.most_common(top):
    print(f"{v:7d} {100.0 * v / max(tot, 1):5.1f}% {inst[k]:9d}  {k[0]}:{k[1]}  {src.get(k, '').strip()[:80]}")
