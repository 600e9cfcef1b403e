# round-2 pass bp: determinism stress on the final binary (one-warp-per-value reductions)
mkdir -p gpurun_out
timeout 1500 python tools/team_stress.py 64 2 3 20 > gpurun_out/r02bp_team2.log 2>&1; tail -1 gpurun_out/r02bp_team2.log | cut -c1-160
timeout 1500 python tools/team_stress.py 64 4 3 12 > gpurun_out/r02bp_team4.log 2>&1; tail -1 gpurun_out/r02bp_team4.log | cut -c1-160
timeout 2400 python tools/stress_determinism.py --step2 200 --out gpurun_out/r02bp_step2.jsonl > gpurun_out/r02bp_step2.log 2>&1; tail -1 gpurun_out/r02bp_step2.log
