set -x
CUDA_LAUNCH_BLOCKING=1 timeout 300 compute-sanitizer --show-backtrace device python tools/tma_debug.py 600 2>&1 | head -60
