set -x
timeout 900 python -m pytest tests/test_reorder_gpu.py tests/test_dist_gpu.py -x -q 2>&1 | tail -2
run() { timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-schur --c5-n 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['value'], d['roofline']['aggregate']['frac'], d['parity']['pass'], d['c2_n10000']['value'], d['step_ms'])"; }
run prio_short
TEIG_FACTOR_PERSIST=1 run prio_persist
TEIG_NO_PRIO=1 TEIG_FACTOR_PERSIST=1 run old
TEIG_NO_PRIO=1 run noprio_short
