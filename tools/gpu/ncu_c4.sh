set -x
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-schur --c2-n 0 --c5-n 0 > gpurun_out/ncu_c4_run.log 2>&1
tail -2 gpurun_out/ncu_c4_run.log
timeout 900 ncu --kernel-name regex:update_left_kernel --launch-skip 200 --launch-count 1 --set full --import-source on --clock-control none -o gpurun_out/upd_left -f python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-schur --c2-n 0 --c5-n 0 > /dev/null 2>&1
timeout 900 ncu --kernel-name regex:"update_right_kernel<128, 2>" --launch-skip 200 --launch-count 1 --set full --import-source on --clock-control none -o gpurun_out/upd_factor -f python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-schur --c2-n 0 --c5-n 0 > /dev/null 2>&1
ls -la gpurun_out | tail -5
