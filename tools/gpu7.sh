for n in 128 256; do for v in 0 1 6 7 8 9 10; do FVB_CG_VARIANT=$v timeout 300 python tools/cg_micro.py $n 400; done; done 2>&1 | grep -v Warn
for v in 6 7; do FVB_CG_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_coupling.py tests/test_gpu_team.py -q 2>&1 | tail -2; done
