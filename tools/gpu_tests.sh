# GPU test suite + smoke on a B200 (run under gpurun from the repo root)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -rf --durations=5 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
