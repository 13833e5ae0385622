set -x
timeout 900 python -m pytest tests/test_reorder_gpu.py tests/test_dist_gpu.py -x -q 2>&1 | tail -2
B="python bench.py --n 20000 --steps 1 --warmup 0 --no-cpu --no-e2e --no-schur --c2-n 0 --c5-n 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l64.csv $B > /dev/null 2>&1
TEIG_LIB_PATH=build/lsub32/libtaskeig_b200.so timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l32.csv $B > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/l64.csv 2>/dev/null | grep "teig::update"
python tools/launch_summary.py gpurun_out/l32.csv 2>/dev/null | grep "teig::update"
for v in "" build/lsub32/libtaskeig_b200.so; do TEIG_LIB_PATH=$v timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-schur --c5-n 0 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['value'], d['roofline']['aggregate']['frac'], d['parity']['pass'], d['c2_n10000']['value'])"; done
