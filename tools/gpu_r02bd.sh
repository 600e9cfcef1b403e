# round-2 pass bd: HEAD check — full suite, smoke, and bench.py with no flags
# (the default run must finish within minutes)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rf 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
t0=$(date +%s); timeout 1500 python bench.py > gpurun_out/r02bd_bench.json 2> gpurun_out/r02bd_bench.err; echo "bench rc=$? $(( $(date +%s) - t0 )) s"; tail -c 300 gpurun_out/r02bd_bench.json
