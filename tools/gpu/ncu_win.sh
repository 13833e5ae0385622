set -x
B="python bench.py --n 10000 --steps 1 --warmup 0 --no-cpu --no-e2e --no-schur --c2-n 0 --c5-n 0"
timeout 900 ncu --kernel-name regex:window_reorder_kernel --launch-skip 60 --launch-count 1 --set full --import-source on --clock-control none -o gpurun_out/win_r02 -f $B > /dev/null 2>&1
ls -la gpurun_out/win_r02.ncu-rep
