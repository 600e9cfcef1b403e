for n in 128 256; do for v in -1 21 22; do FVB_CG_VARIANT=$v timeout 300 python tools/cg_micro.py $n 1000; done; done 2>&1 | grep -v Warn
FVB_CG_VARIANT=21 timeout 900 python -m pytest tests/test_gpu_solvers.py tests/test_gpu_coupling.py -q -x 2>&1 | tail -2
