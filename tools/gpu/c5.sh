set -x
timeout 1200 python bench.py --steps 1 --warmup 1 --n 2000 --c2-n 0 --no-schur --no-e2e > gpurun_out/c5.json 2> gpurun_out/c5.err; tail -3 gpurun_out/c5.err
python -c "import json;d=json.load(open('gpurun_out/c5.json'));print(json.dumps(d['greorder_c5'],indent=1))"
