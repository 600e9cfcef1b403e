# round-2 pass at: product with 512-thread cluster CTAs — full suite, smoke, small configs
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rf 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for r in 1 2; do timeout 300 python tools/small_bench.py | cut -c1-240; done
