TEIG_WINDOW_PROF=1 timeout 600 python bench.py --n 10000 --steps 1 --warmup 1 --no-cpu --no-e2e --no-schur --c2-n 0 --c5-n 0 2>&1 | grep -A12 "window prof" | tail -13
