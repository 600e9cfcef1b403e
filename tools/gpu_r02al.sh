# round-2 pass al: flat all-to-all team reduction (no last arriver / mailbox
# / broadcast) — full suite, then team overhead per CG iteration at 128^3
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rf -x 2>&1 | tail -6
timeout 900 python tools/team_bench.py 128 1 2 4 > gpurun_out/r02al_team_gpu.log 2>&1; cat gpurun_out/r02al_team_gpu.log
FVB_TEAM_SCOPE=sys timeout 900 python tools/team_bench.py 128 2 4 > gpurun_out/r02al_team_sys.log 2>&1; cat gpurun_out/r02al_team_sys.log
