set -x
timeout 1500 python bench.py --no-cpu --no-schur --c5-n 0 --no-e2e > gpurun_out/b_fs.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/b_fs.json')); print('fs', d['value'], d['step_ms'], d['c2_n10000']['step_ms'])"
