# round-2 pass c: A/B of diagnostic builds on the step-2 determinism stress
mkdir -p gpurun_out
for v in base fence gathercg; do
  FVB_PKG_ROOT=variants/$v timeout 600 python tools/stress_determinism.py --step2 1000 --out gpurun_out/r02c_$v.jsonl > gpurun_out/r02c_$v.log 2>&1
  echo "== $v"; tail -2 gpurun_out/r02c_$v.log
  for n in 128 256; do FVB_PKG_ROOT=variants/$v timeout 300 python tools/cg_micro.py $n 400 | cut -c1-200; done
done
