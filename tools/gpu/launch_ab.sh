set -x
B="python bench.py --n 20000 --steps 1 --warmup 0 --no-cpu --no-e2e --no-schur --c2-n 0 --c5-n 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_bulk.csv $B > /dev/null 2>&1
TEIG_NO_TMA=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_legacy.csv $B > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launch_bulk.csv bulk | head -8
python tools/launch_summary.py gpurun_out/launch_legacy.csv legacy | head -8
