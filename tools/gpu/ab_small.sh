set -x
TEIG_AED_PROF=1 timeout 300 python tools/schur_time.py 10000 1 2>&1 | grep -v "^{"
TEIG_SMALL_MODE=1 TEIG_AED_PROF=1 timeout 300 python tools/schur_time.py 10000 1 2>&1 | grep -v "^{"
timeout 900 python -m pytest tests/test_schur_gpu.py -x -q 2>&1 | tail -3
