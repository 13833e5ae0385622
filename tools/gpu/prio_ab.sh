set -x
run() { timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-schur --c5-n 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['value'], d['step_ms'], d['c2_n10000']['value'])"; }
run base
TEIG_PRIO=1 run prio
TEIG_PRIO=1 TEIG_SHORT_Q=1 run prio_short
TEIG_SHORT_Q=1 run short
