set -x
B="python bench.py --n 20000 --steps 1 --warmup 0 --no-cpu --no-e2e --no-schur --c2-n 0 --c5-n 0"
timeout 900 ncu --kernel-name regex:update_left_bulk --launch-skip 100 --launch-count 1 --set full --import-source on --clock-control none -o gpurun_out/bulk_left -f $B > /dev/null 2>&1
timeout 900 ncu --kernel-name regex:update_right_bulk --launch-skip 201 --launch-count 1 --set full --import-source on --clock-control none -o gpurun_out/bulk_right -f $B > /dev/null 2>&1
ls -la gpurun_out | tail -4
