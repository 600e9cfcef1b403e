# round-2 pass d: reduction-buffer fix -> stress, full suite, small-grid sweep
mkdir -p gpurun_out
timeout 900 python tools/stress_determinism.py --step2 1500 --out gpurun_out/r02d_step2.jsonl > gpurun_out/r02d_step2.log 2>&1
tail -2 gpurun_out/r02d_step2.log
timeout 900 python tools/stress_determinism.py --reseed 300 --fresh 10 --big 256 --out gpurun_out/r02d_stress.jsonl > gpurun_out/r02d_stress.log 2>&1
tail -4 gpurun_out/r02d_stress.log
timeout 2400 python -m pytest tests -q -m gpu -rf --durations=15 > gpurun_out/r02d_tests.log 2>&1
tail -30 gpurun_out/r02d_tests.log
for n in 26 40; do for g in 1 2 4 8 16 32 74 148; do timeout 120 python tools/cg_micro.py $n 300 box grid=$g | cut -c1-170; done; done > gpurun_out/r02d_grid.log 2>&1
cat gpurun_out/r02d_grid.log
timeout 300 python tools/small_bench.py > gpurun_out/r02d_small.log 2>&1; cat gpurun_out/r02d_small.log
for v in r01 cur; do for n in 128 256; do
  if [ $v = r01 ]; then FVB_PKG_ROOT=variants/r01 timeout 300 python tools/cg_micro.py $n 400 | cut -c1-200; else timeout 300 python tools/cg_micro.py $n 400 | cut -c1-200; fi
done; done > gpurun_out/r02d_ab.log 2>&1; cat gpurun_out/r02d_ab.log
