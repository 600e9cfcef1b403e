mkdir -p gpurun_out
timeout 600 python tools/team_bench.py 128 1 2>&1 | grep -v Warn | grep "ranks_on\|Error" | sed "s/^/gpu /" > gpurun_out/team_bench.log
for sc in sys gpu; do for P in 2 4; do FVB_TEAM_SCOPE=$sc timeout 600 python tools/team_bench.py 128 $P 2>&1 | grep -v Warn | grep "ranks_on\|Error" | sed "s/^/$sc /"; done; done >> gpurun_out/team_bench.log 2>&1
cat gpurun_out/team_bench.log | cut -c1-200
