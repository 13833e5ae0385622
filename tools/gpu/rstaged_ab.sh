set -x
TEIG_LIB_PATH=build/rstaged/libtaskeig_b200.so timeout 900 python -m pytest tests/test_reorder_gpu.py tests/test_dist_gpu.py -x -q 2>&1 | tail -2
B="python bench.py --n 20000 --steps 1 --warmup 0 --no-cpu --no-e2e --no-schur --c2-n 0 --c5-n 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r_def.csv $B > /dev/null 2>&1
TEIG_LIB_PATH=build/rstaged/libtaskeig_b200.so timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r_stg.csv $B > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r_def.csv 2>/dev/null | grep "teig::update"
python tools/launch_summary.py gpurun_out/r_stg.csv 2>/dev/null | grep "teig::update"
