# team (domain decomposition) tests + full GPU suite + smoke + short bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_team.py -x -q 2>&1 | tail -30 > gpurun_out/pytest_team.log
tail -5 gpurun_out/pytest_team.log
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -c 2500 gpurun_out/bench.log
