set -x
for nt in 32 64 128; do TEIG_AED_PROF=1 TEIG_LIB_PATH=build/nt$nt/libtaskeig_b200.so timeout 300 python tools/schur_time.py 10000 1 2>&1 | tail -3; done
TEIG_AED_PROF=1 timeout 300 python tools/schur_time.py 10000 1 2>&1 | tail -3
timeout 300 python tools/chase_err.py
