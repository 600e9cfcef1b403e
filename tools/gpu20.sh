timeout 900 python -m pytest tests/test_gpu_coupling.py -q -k reseeded 2>&1 | tail -5
