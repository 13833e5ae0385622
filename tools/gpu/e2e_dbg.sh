set -x
for P in 0 1; do
TEIG_POOL_RELEASE=$P timeout 1500 python bench.py --no-cpu --no-schur --c5-n 0 > gpurun_out/b_e2e.json 2> gpurun_out/b_e2e.err
python -c "
import json; d=json.load(open('gpurun_out/b_e2e.json')); print('release=$P', d['value'], d['step_ms'], d['e2e']['calls_s'], d['c2_n10000']['value'], d['c2_n10000']['e2e']['calls_s'])"
done
