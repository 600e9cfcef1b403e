mkdir -p gpurun_out
for c in "cav6 2" "pcav5 2" "cav6 3" "chan 2"; do timeout 120 python tools/team_debug.py $c 2>&1 | tail -25; done > gpurun_out/team_debug.log 2>&1
cat gpurun_out/team_debug.log | cut -c1-400
