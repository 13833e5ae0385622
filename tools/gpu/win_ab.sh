set -x
timeout 900 python -m pytest tests/test_reorder_gpu.py tests/test_dist_gpu.py -x -q 2>&1 | tail -2
for v in "" build/wold/libtaskeig_b200.so; do
  TEIG_LIB_PATH=$v TEIG_WINDOW_PROF=1 timeout 600 python bench.py --n 10000 --steps 1 --warmup 1 --no-cpu --no-e2e --no-schur --c2-n 0 --c5-n 0 2>&1 | grep "kernel cycles per step"
  TEIG_LIB_PATH=$v timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-schur --c5-n 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['value'], d['step_ms'], d['roofline']['window_ms_per_step'], d['c2_n10000']['value'], d['c2_n10000']['step_ms'])"
done
