mkdir -p gpurun_out
for rep in 1 2; do for v in r01 cur biunb biteam biteamb; do for n in 256; do
  if [ $v = cur ]; then R=""; else R="FVB_PKG_ROOT=variants/$v"; fi
  echo "bi $v n=$n $(env $R timeout 300 python tools/bi_micro.py $n 60 | cut -c1-200)"
done; done; done > gpurun_out/r02h_ab.log 2>&1
cat gpurun_out/r02h_ab.log
