set -x
free -g; nproc; df -h /dev/shm | tail -1
timeout 900 python bench.py --n 4000 --steps 2 --warmup 1 --force-dist --no-cpu 2>&1 | tail -3
timeout 1500 python bench.py --steps 3 --warmup 2 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -5 gpurun_out/bench_c4.err
cat gpurun_out/bench_c4.json
