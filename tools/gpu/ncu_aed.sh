set -x
timeout 900 ncu --kernel-name regex:aed_window_kernel --launch-skip 20 --launch-count 1 --set full --import-source on --clock-control none -o gpurun_out/aed_prof -f python tools/schur_time.py 2000 > gpurun_out/ncu_aed.log 2>&1
tail -5 gpurun_out/ncu_aed.log
timeout 900 ncu --kernel-name regex:chase_window_kernel --launch-skip 20 --launch-count 1 --set full --import-source on --clock-control none -o gpurun_out/chase_prof -f python tools/schur_time.py 2000 > gpurun_out/ncu_chase.log 2>&1
tail -3 gpurun_out/ncu_chase.log
ls -la gpurun_out
