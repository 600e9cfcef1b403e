# round-2 final binary (CG reductions one warp per value): suite, smoke, both bench arms under the driver's flags
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rf --durations=5 > gpurun_out/r02bt_tests.log 2>&1; tail -2 gpurun_out/r02bt_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02bt_smoke.log 2>&1; tail -1 gpurun_out/r02bt_smoke.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02bt_ref.json 2> gpurun_out/r02bt_ref.err; tail -c 150 gpurun_out/r02bt_ref.json
timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r02bt_bench.json 2> gpurun_out/r02bt_bench.err; tail -c 150 gpurun_out/r02bt_bench.json
