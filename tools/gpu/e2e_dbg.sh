set -x
TEIG_HOST_PROF=1 timeout 1500 python bench.py --no-cpu --no-schur --c5-n 0 > gpurun_out/b_e2e.json 2> gpurun_out/b_e2e.err
grep "teig host" gpurun_out/b_e2e.err
python -c "
import json; d=json.load(open('gpurun_out/b_e2e.json')); print(d['value'], d['step_ms'], d['e2e']['calls_s'], d['c2_n10000']['step_ms'], d['c2_n10000']['e2e']['calls_s'])"
free -g | head -2; numactl -H 2>/dev/null | head -3; nproc
