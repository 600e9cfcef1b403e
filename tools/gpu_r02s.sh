mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02s_c1_launches.csv python tools/c1_steps.py 5 > gpurun_out/r02s_c1.log 2>&1; tail -2 gpurun_out/r02s_c1.log
timeout 120 python tools/c1_steps.py 5
timeout 900 python -m pytest tests/test_gpu_solvers.py -q -rf -k "small_system" > gpurun_out/r02s_tests.log 2>&1; tail -3 gpurun_out/r02s_tests.log
timeout 900 python tools/team_bench.py 128 1 2 4 > gpurun_out/r02s_team_gpu.log 2>&1; cat gpurun_out/r02s_team_gpu.log
FVB_TEAM_SCOPE=sys timeout 900 python tools/team_bench.py 128 2 4 > gpurun_out/r02s_team_sys.log 2>&1; cat gpurun_out/r02s_team_sys.log
timeout 600 python tools/report_run.py 128 3 gpurun_out/r02_report > gpurun_out/r02s_report.log 2>&1; cat gpurun_out/r02s_report.log
