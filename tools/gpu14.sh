timeout 1500 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_coupling.py tests/test_gpu_configs.py tests/test_gpu_team.py -q -x 2>&1 | tail -2
timeout 1500 python bench.py --no-cpu-baseline --no-e2e --no-aux 2>&1 | tail -c 420
FVB_BI_TILE=0 timeout 1500 python bench.py --no-cpu-baseline --no-e2e --no-aux 2>&1 | tail -c 420
