# round-2 pass p: shared-memory single-block solvers
mkdir -p gpurun_out
for n in 5 7 10 12; do for o in smem nocluster; do echo "cg n=$n $o $(timeout 120 python tools/cg_micro.py $n 300 box $o | cut -c1-170)"; done; done > gpurun_out/r02p_micro.log 2>&1
for n in 7 10; do for o in smem nocluster; do echo "bi n=$n $o $(timeout 120 python tools/bi_micro.py $n 60 box $o | cut -c1-170)"; done; done >> gpurun_out/r02p_micro.log 2>&1
cat gpurun_out/r02p_micro.log
timeout 300 python tools/small_bench.py > gpurun_out/r02p_small.log 2>&1; cat gpurun_out/r02p_small.log
timeout 1500 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_configs.py tests/test_gpu_coupling.py tests/test_gpu_ops.py tests/test_gpu_next.py tests/test_gpu_team.py "tests/test_gpu_golden_full.py::test_c3_backward_step_nh16_simple_to_convergence" -q -rf > gpurun_out/r02p_tests.log 2>&1; tail -5 gpurun_out/r02p_tests.log
