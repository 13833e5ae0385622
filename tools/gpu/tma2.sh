set -x
timeout 1200 python -m pytest tests/test_reorder_gpu.py tests/test_dist_gpu.py -x -q 2>&1 | tail -3
B="python bench.py --n 20000 --steps 1 --warmup 0 --no-cpu --no-e2e --no-schur --c2-n 0 --c5-n 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_bulk2.csv $B > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launch_bulk2.csv bulk 2>/dev/null | grep teig
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-schur --c5-n 0 > gpurun_out/tma_on.json 2> gpurun_out/tma_on.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/tma_on.json").read().strip().splitlines()[-1])
print(d["value"], d["roofline"]["frac"], d["roofline"]["aggregate"]["frac"], d["parity"]["pass"], d.get("c2_n10000", {}).get("value"))
PY
