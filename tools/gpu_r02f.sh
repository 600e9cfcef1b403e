# round-2 pass f: bisect the CG per-iteration regression across commits
mkdir -p gpurun_out
for rep in 1 2; do
for v in r01 c507 cdca caf7 cur; do
  for n in 256 128; do
    if [ $v = cur ]; then R=""; else R="FVB_PKG_ROOT=variants/$v"; fi
    echo "$v n=$n $(env $R timeout 300 python tools/cg_micro.py $n 400 | cut -c1-150)"
  done
done
done > gpurun_out/r02f_bisect.log 2>&1
cat gpurun_out/r02f_bisect.log
for v in r01 cur; do if [ $v = cur ]; then R=""; else R="FVB_PKG_ROOT=variants/$v"; fi; echo "$v $(env $R timeout 300 python tools/bi_micro.py 256 60 | cut -c1-200)"; done
