mkdir -p gpurun_out
for n in 10 12 15 20; do echo "cg n=$n $(timeout 120 python tools/cg_micro.py $n 300 | cut -c1-170)"; done > gpurun_out/r02o_micro.log 2>&1
for n in 12 15; do echo "bi n=$n $(timeout 120 python tools/bi_micro.py $n 60 | cut -c1-170)"; done >> gpurun_out/r02o_micro.log 2>&1
cat gpurun_out/r02o_micro.log
timeout 2400 python -m pytest tests -q -m gpu -rf --durations=10 > gpurun_out/r02o_tests.log 2>&1; tail -15 gpurun_out/r02o_tests.log
timeout 300 python tools/small_bench.py > gpurun_out/r02o_small.log 2>&1; cat gpurun_out/r02o_small.log
timeout 900 python tools/stress_determinism.py --step2 300 --out gpurun_out/r02o_step2.jsonl > gpurun_out/r02o_step2.log 2>&1; tail -2 gpurun_out/r02o_step2.log
