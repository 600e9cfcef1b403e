timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -3
timeout 1500 python bench.py --no-cpu-baseline 2>&1 | tail -c 2500
