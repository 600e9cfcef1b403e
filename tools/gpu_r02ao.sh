# round-2 pass ao: full suite with the flat team reduction; team overhead
# with 8 co-resident ranks (gpu and system scope)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rf 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python tools/team_bench.py 128 8 > gpurun_out/r02ao_team_gpu.log 2>&1; cat gpurun_out/r02ao_team_gpu.log
FVB_TEAM_SCOPE=sys timeout 900 python tools/team_bench.py 128 8 > gpurun_out/r02ao_team_sys.log 2>&1; cat gpurun_out/r02ao_team_sys.log
