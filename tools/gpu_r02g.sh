# round-2 pass g: CG gathers batched; BiCGStab gather batching / occupancy A/B
mkdir -p gpurun_out
for v in r01 cur; do for n in 256 128; do
  if [ $v = cur ]; then R=""; else R="FVB_PKG_ROOT=variants/$v"; fi
  echo "cg $v n=$n $(env $R timeout 300 python tools/cg_micro.py $n 400 | cut -c1-170)"
done; done > gpurun_out/r02g_ab.log 2>&1
for v in r01 cur biunb bi1; do for n in 256 128; do
  if [ $v = cur ]; then R=""; else R="FVB_PKG_ROOT=variants/$v"; fi
  echo "bi $v n=$n $(env $R timeout 300 python tools/bi_micro.py $n 60 | cut -c1-230)"
done; done >> gpurun_out/r02g_ab.log 2>&1
cat gpurun_out/r02g_ab.log
timeout 900 python tools/bicgstab_diag.py 64 128 > gpurun_out/r02g_bidiag.log 2>&1; cat gpurun_out/r02g_bidiag.log
