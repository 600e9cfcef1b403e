timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 1500 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -c 1500
FVB_BI_VARIANT=1 timeout 1500 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -c 400
