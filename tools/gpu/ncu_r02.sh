# round-2 profiles of the headline (C4 n=40000): launch list + one full capture
# of the dominant kernels, with per-level tile counts for the algorithmic bytes
set -x
B="python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-schur --c2-n 0 --c5-n 0"
TEIG_LAUNCH_LOG=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv $B > gpurun_out/ncu_r02_run.log 2> gpurun_out/levels_r02.txt
python tools/launch_summary.py gpurun_out/launches_r02.csv "round 2: $B (C4 reorder n=40000, ws=128, Q)" > gpurun_out/r02_launches_summary.txt 2>&1
head -12 gpurun_out/r02_launches_summary.txt
timeout 900 ncu --kernel-name regex:update_right_bulk_kernel --launch-skip 401 --launch-count 1 --set full --import-source on --clock-control none -o gpurun_out/r02_factor -f $B > /dev/null 2>&1
timeout 900 ncu --kernel-name regex:update_left_bulk --launch-skip 200 --launch-count 1 --set full --import-source on --clock-control none -o gpurun_out/r02_left -f $B > /dev/null 2>&1
ls -la gpurun_out | tail -6
