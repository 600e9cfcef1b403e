for n in 256 128; do for v in 12 14 15 16; do FVB_CG_VARIANT=$v timeout 300 python tools/cg_micro.py $n 400; done; done 2>&1 | grep -v Warn
