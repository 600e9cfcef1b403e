# round-2 pass ad: one-barrier single-block reduction — tests, then A/B
# against the two-barrier diagnostic build (variants/two_sync) on C1, C3
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rf -x 2>&1 | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for r in 1 2; do
  echo "new  $(timeout 300 python tools/small_bench.py | tr '\n' ' ' | cut -c1-900)"
  echo "old  $(FVB_PKG_ROOT=variants/two_sync timeout 300 python tools/small_bench.py | tr '\n' ' ' | cut -c1-900)"
done
for nh in 64 128; do
  for v in new old; do
    root=; [ $v = old ] && root=variants/two_sync
    echo "c3 nh$nh $v $(timeout 600 python -c "
import sys, json; import bench
if '$root': sys.path.insert(0, '$root')
o = bench.measure_c3($nh, 3, 2)
import paper_1207_1571_b200 as P; print(P.__file__, json.dumps({k: o[k] for k in ('ms_per_sweep', 'cg_iters_per_sweep')}), o.get('roofline', {}).get('frac'))" 2>&1 | tail -1)"
  done
done
