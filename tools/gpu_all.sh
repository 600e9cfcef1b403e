bash tools/gpu_tests.sh
timeout 1500 python bench.py 2>&1 | tail -c 3500
