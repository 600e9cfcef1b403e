# round-2 pass b: barrier acquire fix -> determinism stress, suite, CG micro
mkdir -p gpurun_out
timeout 900 python tools/stress_determinism.py --reseed 600 --fresh 10 --big 0 --out gpurun_out/r02b_stress.jsonl > gpurun_out/r02b_stress.log 2>&1
tail -3 gpurun_out/r02b_stress.log
timeout 1500 python -m pytest tests -q -m gpu -rf -x --deselect tests/test_gpu_golden_full.py > gpurun_out/r02b_tests.log 2>&1
tail -3 gpurun_out/r02b_tests.log
timeout 600 python -m pytest tests/test_gpu_golden_full.py -q -k c3 -rf > gpurun_out/r02b_c3.log 2>&1
tail -25 gpurun_out/r02b_c3.log
for n in 128 256; do timeout 300 python tools/cg_micro.py $n 400; done > gpurun_out/r02b_cg_micro.log 2>&1
cat gpurun_out/r02b_cg_micro.log
