# round-2 pass aj: cluster reduction by remote stores (no remote loads, no
# block barriers after the cluster barrier) — tests, C1/C3 timings
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rf -x 2>&1 | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for r in 1 2; do
  timeout 300 python tools/small_bench.py | cut -c1-300
done
timeout 900 python tools/cg_micro.py 24 400 2>&1 | tail -2 | cut -c1-300
