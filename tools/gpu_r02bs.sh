# round-2 pass bs: CG reductions with one warp per value (M = 2, 3) vs the value-inner warp-0 form
mkdir -p gpurun_out
for r in 1 2; do
  for n in 48 64 128 256; do
    it=400; [ $n = 256 ] && it=100
    echo "new  $(timeout 600 python tools/cg_micro.py $n $it | cut -c1-150)"
    echo "head $(FVB_PKG_ROOT=variants/head timeout 600 python tools/cg_micro.py $n $it | cut -c1-150)"
  done
done
