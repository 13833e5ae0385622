TEIG_AED_PROF=1 timeout 300 python tools/schur_time.py 10000 1 2>&1 | grep -v "^{"
