for n in 128 256; do for v in 12 17; do FVB_CG_VARIANT=$v timeout 300 python tools/cg_micro.py $n 400; done; done 2>&1 | grep -v Warn
timeout 900 python -m pytest tests/test_gpu_team.py tests/test_gpu_solvers.py tests/test_gpu_coupling.py -q -x 2>&1 | tail -2
