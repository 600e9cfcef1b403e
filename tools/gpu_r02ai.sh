# round-2 pass ai: the C1 momentum batch as three single-block solves (k_bicgstab_split)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rf -x 2>&1 | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for r in 1 2 3; do
  echo "split $(timeout 300 python tools/small_bench.py | head -1 | cut -c1-600)"
done
