# round-2 pass ap: determinism stress after the round-2 changes: the flat team
# reduction (2 and 4 co-resident ranks, fresh runs) and the single-domain
# step with graph replay (PISO step 2 at 128^3 repeated)
mkdir -p gpurun_out
timeout 1500 python tools/team_stress.py 64 2 3 40 > gpurun_out/r02ap_team2.log 2>&1; tail -1 gpurun_out/r02ap_team2.log | cut -c1-200
timeout 1500 python tools/team_stress.py 64 4 3 25 > gpurun_out/r02ap_team4.log 2>&1; tail -1 gpurun_out/r02ap_team4.log | cut -c1-200
timeout 2400 python tools/stress_determinism.py --step2 400 --out gpurun_out/r02ap_step2.jsonl > gpurun_out/r02ap_step2.log 2>&1; tail -3 gpurun_out/r02ap_step2.log | cut -c1-400
