# kernel / team micro-benchmarks (CG per-iteration, team overhead, small configs)
for n in 128 256; do timeout 300 python tools/cg_micro.py $n 1000; done 2>&1 | grep -v Warn
timeout 600 python tools/team_bench.py 128 1 2 4 2>&1 | grep -v Warn | grep "ranks_on\|Error"
timeout 600 python tools/small_bench.py 2>&1 | grep -v Warn | tail -2
