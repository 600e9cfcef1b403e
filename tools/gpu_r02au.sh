# round-2 pass au: threads per block of the single-domain persistent CG grid
# (one block per SM): 1024 (product) vs 512 (variants/gt512), mid-size to C5
mkdir -p gpurun_out
for n in 48 64 80 100 128 256; do
  it=400; [ $n = 256 ] && it=60
  echo "1024 $(timeout 600 python tools/cg_micro.py $n $it | cut -c1-150)"
  echo "512  $(FVB_PKG_ROOT=variants/gt512 timeout 600 python tools/cg_micro.py $n $it | cut -c1-150)"
done
for nh in 64; do
  for v in p v; do
    root=; [ $v = v ] && root=variants/gt512
    echo "c3 nh$nh $v $(timeout 600 python -c "
import sys, json; import bench
if '$root': sys.path.insert(0, '$root')
o = bench.measure_c3($nh, 3, 2)
print(json.dumps({k: o[k] for k in ('ms_per_sweep', 'cg_iters_per_sweep', 'k_cg_frac')}))" 2>&1 | tail -1)"
  done
done
