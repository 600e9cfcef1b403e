# round-2 pass bf: block partials summed with their loads issued together
# (lane_sums) vs HEAD (variants/head): CG per iteration, BiCGStab, C3/C2
mkdir -p gpurun_out
for n in 48 64 128 256; do
  it=400; [ $n = 256 ] && it=60
  echo "new  $(timeout 600 python tools/cg_micro.py $n $it | cut -c1-140)"
  echo "head $(FVB_PKG_ROOT=variants/head timeout 600 python tools/cg_micro.py $n $it | cut -c1-140)"
done
for n in 128 256; do
  echo "new  $(timeout 600 python tools/bi_micro.py $n 40 | cut -c1-140)"
  echo "head $(FVB_PKG_ROOT=variants/head timeout 600 python tools/bi_micro.py $n 40 | cut -c1-140)"
done
for v in new head; do
  root=; [ $v = head ] && root=variants/head
  echo "c3 nh64 $v $(timeout 600 python -c "
import sys, json; import bench
if '$root': sys.path.insert(0, '$root')
o = bench.measure_c3(64, 3, 2)
print(json.dumps({k: o[k] for k in ('ms_per_sweep', 'cg_iters_per_sweep', 'k_cg_frac')}))" 2>&1 | tail -1)"
done
