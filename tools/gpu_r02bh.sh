# round-2 pass bh: lane_sums in the value-inner form only (no all-loads-first
# path) vs HEAD: CG at 64^3 and 256^3
mkdir -p gpurun_out
for r in 1 2; do
  for n in 64 256; do
    it=400; [ $n = 256 ] && it=100
    echo "new  $(timeout 600 python tools/cg_micro.py $n $it | cut -c1-200)"
    echo "head $(FVB_PKG_ROOT=variants/head timeout 600 python tools/cg_micro.py $n $it | cut -c1-200)"
  done
done
