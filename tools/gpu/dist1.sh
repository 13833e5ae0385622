set -x
timeout 900 python -m pytest tests/test_dist_gpu.py -x -q 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 600 python bench.py --n 40000 --steps 1 --warmup 1 --no-cpu --no-e2e --no-schur 2>&1 | tail -2
