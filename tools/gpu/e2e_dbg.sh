set -x
for P in 0 0; do
TEIG_NO_DRAIN=$P timeout 1500 python bench.py --no-cpu --no-schur --c5-n 0 > gpurun_out/b_e2e.json 2> gpurun_out/b_e2e.err
python -c "
import json; d=json.load(open('gpurun_out/b_e2e.json')); print('nodrain=$P', d['value'], d['e2e']['calls_s'], d['c2_n10000']['e2e']['calls_s'])"
done
