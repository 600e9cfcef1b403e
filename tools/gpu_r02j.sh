mkdir -p gpurun_out
for rep in 1 2; do for v in cdca cur; do
  if [ $v = cur ]; then R=""; else R="FVB_PKG_ROOT=variants/$v"; fi
  echo "bi $v $(env $R timeout 300 python tools/bi_micro.py 256 60 | cut -c1-200)"
  echo "cg $v $(env $R timeout 300 python tools/cg_micro.py 256 400 | cut -c1-200)"
done; done > gpurun_out/r02j_ab.log 2>&1
cat gpurun_out/r02j_ab.log
