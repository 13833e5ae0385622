set -x
timeout 900 ncu --kernel-name regex:aed_window_kernel --launch-skip 20 --launch-count 1 --set full --import-source on --clock-control none -o gpurun_out/aed_prof2 -f python tools/schur_time.py 2000 > gpurun_out/ncu_aed2.log 2>&1
tail -2 gpurun_out/ncu_aed2.log
/usr/bin/time -v timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/ref_arm.json 2> gpurun_out/ref_arm.err; tail -20 gpurun_out/ref_arm.err | grep -i "maximum resident\|elapsed"; cat gpurun_out/ref_arm.json
