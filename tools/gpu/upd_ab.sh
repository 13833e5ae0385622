run() { timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu --no-schur --no-e2e --c2-n 10000 --c5-n 0 2>&1 | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['value'], d['roofline']['achieved'], d['roofline']['aggregate']['frac'], d['c2_n10000']['value'], d['parity']['pass'])"; }
run A
for v in B C D E; do TEIG_LIB_PATH=build/upd$v/libtaskeig_b200.so run $v; done
