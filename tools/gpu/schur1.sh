set -x
timeout 900 python -m pytest tests/test_schur_gpu.py -x -q 2>&1 | tail -25
timeout 300 python tools/schur_time.py 2000 1
timeout 600 python tools/schur_time.py 10000 1
