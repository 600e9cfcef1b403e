# round-2 pass bl: one warp per value in the many-value and team reductions — suite, team bench
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rf 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python tools/team_bench.py 128 1 2 4 2>&1 | tail -3
timeout 900 python tools/team_bench.py 128 2 4 sys 2>&1 | tail -2
