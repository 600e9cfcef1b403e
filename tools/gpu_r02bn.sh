# round-2 last evidence on the final binary: suite + smoke, both bench arms (driver flags), launch list
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rf --durations=10 > gpurun_out/r02bn_tests.log 2>&1; tail -2 gpurun_out/r02bn_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02bn_smoke.log 2>&1; tail -1 gpurun_out/r02bn_smoke.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02bn_ref.json 2> gpurun_out/r02bn_ref.err; tail -c 200 gpurun_out/r02bn_ref.json
timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r02bn_bench.json 2> gpurun_out/r02bn_bench.err; tail -c 200 gpurun_out/r02bn_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02bn_launches_c5.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-aux > gpurun_out/r02bn_ncu_launch.log 2>&1; tail -c 100 gpurun_out/r02bn_ncu_launch.log
