mkdir -p gpurun_out
for sc in sys gpu; do for P in 2 4; do FVB_TEAM_SCOPE=$sc timeout 600 python tools/team_bench.py 128 $P 2>&1 | grep -v Warn | grep "ranks_on\|Error" | sed "s/^/$sc /"; done; done > gpurun_out/team_bench.log 2>&1
timeout 600 python tools/team_bench.py 128 1 2>&1 | grep -v Warn | grep "ranks_on\|Error" >> gpurun_out/team_bench.log
cat gpurun_out/team_bench.log | cut -c1-200
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -2
