timeout 600 python tools/small_bench.py 2>&1 | grep -v Warn | tail -3
timeout 1500 python -m pytest tests -q -m gpu -rf 2>&1 | grep -E "FAILED|passed|failed|^E " | head -20
