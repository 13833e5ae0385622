# TMA update kernels: GPU tests, then C4 (and C2) with the TMA and the cp.async kernels
set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-schur --c5-n 0 > gpurun_out/tma_on.json 2> gpurun_out/tma_on.err
TEIG_NO_TMA=1 timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-schur --c5-n 0 > gpurun_out/tma_off.json 2> gpurun_out/tma_off.err
python - <<'PY'
import json
for f in ("gpurun_out/tma_on.json", "gpurun_out/tma_off.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d["roofline"]["frac"], d["roofline"]["aggregate"]["frac"], d["parity"]["pass"], d.get("c2_n10000", {}).get("value"))
    except Exception as e:
        print(f, "ERR", e)
PY
tail -3 gpurun_out/tma_on.err
