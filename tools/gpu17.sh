timeout 900 python tools/team_bench.py 128 1 2 4 8 2>&1 | grep -v Warn
FVB_TEAM_SCOPE=sys timeout 900 python tools/team_bench.py 128 2 4 2>&1 | grep -v Warn
timeout 900 python -m pytest tests/test_gpu_team.py tests/test_gpu_configs.py -q 2>&1 | tail -2
