set -x
timeout 300 python tools/tma_debug.py 600
timeout 900 python -m pytest tests/test_reorder_gpu.py tests/test_dist_gpu.py tests/test_greorder_gpu.py -x -q 2>&1 | tail -2
B="python bench.py --n 20000 --steps 1 --warmup 0 --no-cpu --no-e2e --no-schur --c2-n 0 --c5-n 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/nb.csv $B > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/nb.csv 2>/dev/null | grep "teig::update"
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-schur --c5-n 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['step_ms'], d['roofline']['aggregate']['frac'], d['parity']['pass'], d['c2_n10000']['value'])"
