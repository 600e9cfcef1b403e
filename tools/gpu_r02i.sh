mkdir -p gpurun_out
for rep in 1 2; do for v in r01 c963 c507 cdca biunb; do
  R="FVB_PKG_ROOT=variants/$v"
  echo "bi $v $(env $R timeout 300 python tools/bi_micro.py 256 60 | cut -c1-200)"
done; done > gpurun_out/r02i_ab.log 2>&1
cat gpurun_out/r02i_ab.log
