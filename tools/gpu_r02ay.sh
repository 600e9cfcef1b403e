# round-2 pass ay: team scope as a DecomposedRun argument (no env variant in
# the package) — team tests and the system-scope team bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -rf -k "team or decomposed" 2>&1 | tail -3
timeout 900 python tools/team_bench.py 128 2 4 sys 2>&1 | tail -2
