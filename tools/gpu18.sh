mkdir -p gpurun_out
for sc in sys gpu; do for P in 2 4; do FVB_TEAM_SCOPE=$sc timeout 600 python tools/team_bench.py 128 $P 2>&1 | grep -v Warn | grep "ranks_on\|Error" | sed "s/^/$sc /"; done; done > gpurun_out/team_bench.log 2>&1
cat gpurun_out/team_bench.log | cut -c1-200
FVB_TEAM_SCOPE=sys timeout 900 python -m pytest tests/test_gpu_team.py tests/test_gpu_configs.py -q 2>&1 | tail -2
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -2
