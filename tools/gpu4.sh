mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_team.py -q 2>&1 | tail -60 > gpurun_out/pytest_team.log
tail -12 gpurun_out/pytest_team.log
