#!/bin/bash
# Round-3 profiling evidence, run on the GPU box from the repo root:
#   TMA tensor-map probe (compute-sanitizer log), C4 launch list, ncu --set
#   full captures of the dominant kernels, compute-sanitizer racecheck /
#   synccheck / memcheck over every kernel family.
set -x
O=gpurun_out
mkdir -p $O
# 1. TMA tensor-map probe
nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/microbench/tma_min.cu -o /tmp/tma_min -lcuda > $O/tma_build.log 2>&1
for m in 0 2 3 4 6; do timeout 60 /tmp/tma_min $m > $O/tma_mode$m.log 2>&1; echo "rc=$?" >> $O/tma_mode$m.log; done
timeout 120 compute-sanitizer /tmp/tma_min 0 > $O/tma_sanitizer.log 2>&1; echo "rc=$?" >> $O/tma_sanitizer.log
cuobjdump -sass /tmp/tma_min | grep -E "UTMALDG|UBLKCP|SYNCS" | head -5 > $O/tma_sass.txt
# 2. C4 launch list (serialised, cold) with per-level tile counts
B="python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-schur --c2-n 0 --c5-n 0"
TEIG_LAUNCH_LOG=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_r03.csv $B > $O/ncu_r03_run.log 2> $O/levels_r03.txt
python tools/launch_summary.py $O/launches_r03.csv "round 3: $B (C4 reorder n=40000, ws=128, Q)" > $O/r03_launches_summary.txt 2>&1
# 3. full captures
timeout 900 ncu --kernel-name regex:update_left_bulk --launch-skip 200 --launch-count 1 --set full --import-source on --clock-control none -o $O/r03_left -f $B > /dev/null 2>&1
timeout 900 ncu --kernel-name regex:col_matvec --launch-skip 3000 --launch-count 1 --set full --import-source on --clock-control none -o $O/r03_hess_matvec -f python tools/hess_time.py 4000 > /dev/null 2>&1
timeout 900 ncu --kernel-name regex:gemm_kernel --launch-skip 100 --launch-count 2 --set full --import-source on --clock-control none -o $O/r03_hess_gemm -f python tools/hess_time.py 4000 > /dev/null 2>&1
timeout 900 ncu --kernel-name regex:aed_window_kernel --launch-skip 60 --launch-count 1 --set full --import-source on --clock-control none -o $O/r03_aed -f python bench.py --workload schur --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
# 4. sanitizers
for t in racecheck synccheck memcheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_small.py > $O/sanitizer_$t.log 2>&1; echo "rc=$?" >> $O/sanitizer_$t.log
done
ls -la $O
