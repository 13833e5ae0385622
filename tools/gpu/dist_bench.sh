set -x
timeout 900 python bench.py --n 8000 --steps 2 --warmup 1 --force-dist --no-cpu 2>&1 | tail -2
