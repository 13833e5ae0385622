set -x
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -3 gpurun_out/bench_full.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_full.json'))
print("headline", d["value"], d["unit"], "e2e", d["e2e"]["value"], "roof", d["roofline"]["frac"], d["roofline"]["aggregate"]["frac"], "cpu", d["cpu_baseline"]["value"])
for k in ("c2_n10000","greorder_c5","schur_c3"):
    x=d[k]; print(k, x["value"], x.get("e2e",{}).get("value"), x.get("cpu_baseline",{}).get("value"), x["parity"].get("pass"))
PY
