timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
timeout 1500 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -c 700
FVB_BI_VARIANT=5 timeout 1500 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -c 400
