set -x
TEIG_HOST_PROF=1 python tools/host_e2e.py 40000 2>&1 | grep -E "teig host|call"
TEIG_Q_SERIAL=1 TEIG_HOST_PROF=1 python tools/host_e2e.py 40000 2>&1 | grep -E "teig host|^call"
TEIG_NO_DRAIN=1 TEIG_HOST_PROF=1 python tools/host_e2e.py 40000 2>&1 | grep -E "teig host|^call"
