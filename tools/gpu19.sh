timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -k decomposed 2>&1 | tail -4
