# round-2 pass e: plane-marching BiCGStab A/B, solver tests, bench
mkdir -p gpurun_out
for n in 256 128; do
  echo "== n=$n march (512x2)"; timeout 300 python tools/bi_micro.py $n 60 | cut -c1-260
  echo "== n=$n row sweep"; timeout 300 python tools/bi_micro.py $n 60 box nomarch | cut -c1-260
  echo "== n=$n march (512x1)"; FVB_PKG_ROOT=variants/minb1 timeout 300 python tools/bi_micro.py $n 60 | cut -c1-260
  echo "== n=$n r01 build"; FVB_PKG_ROOT=variants/r01 timeout 300 python tools/bi_micro.py $n 60 | cut -c1-260
done > gpurun_out/r02e_bi.log 2>&1
cat gpurun_out/r02e_bi.log
timeout 1200 python -m pytest tests/test_gpu_solvers.py -q -rf > gpurun_out/r02e_solvers.log 2>&1; tail -5 gpurun_out/r02e_solvers.log
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/r02e_bench.json 2> gpurun_out/r02e_bench.err
tail -c 3000 gpurun_out/r02e_bench.json
