# round-2 pass an: flat team reduction, acquire load instead of the acquire fence,
# reduction — team tests, team overhead at 128^3 (gpu and sys scope)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rf -x -k "team or decomposed or decompose" 2>&1 | tail -4
timeout 900 python tools/team_bench.py 128 1 2 4 > gpurun_out/r02an_team_gpu.log 2>&1; cat gpurun_out/r02an_team_gpu.log
FVB_TEAM_SCOPE=sys timeout 900 python tools/team_bench.py 128 2 4 > gpurun_out/r02an_team_sys.log 2>&1; cat gpurun_out/r02an_team_sys.log
