# round-2 pass m: 16-CTA clusters with parallel DSMEM reads
mkdir -p gpurun_out
for n in 16 20 26 32 34; do for o in cluster nocluster; do
  echo "cg n=$n $o $(timeout 120 python tools/cg_micro.py $n 300 box $o | cut -c1-160)"
done; done > gpurun_out/r02m_cluster.log 2>&1
for n in 20 26 34; do for o in cluster nocluster; do
  echo "bi n=$n $o $(timeout 120 python tools/bi_micro.py $n 60 box $o | cut -c1-180)"
done; done >> gpurun_out/r02m_cluster.log 2>&1
cat gpurun_out/r02m_cluster.log
timeout 1200 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_configs.py tests/test_gpu_coupling.py tests/test_gpu_ops.py "tests/test_gpu_golden_full.py::test_c3_backward_step_nh16_simple_to_convergence" -q -rf > gpurun_out/r02m_tests.log 2>&1; tail -5 gpurun_out/r02m_tests.log
timeout 300 python tools/small_bench.py > gpurun_out/r02m_small.log 2>&1; cat gpurun_out/r02m_small.log
