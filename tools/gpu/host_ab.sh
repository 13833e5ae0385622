set -x
TEIG_HOST_PROF=1 python tools/host_e2e.py 40000
