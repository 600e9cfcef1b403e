mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rf --durations=5 2>&1 | tail -12
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for n in 256 128; do echo "cg n=$n $(timeout 300 python tools/cg_micro.py $n 400 | cut -c1-150)"; done
echo "bi $(timeout 300 python tools/bi_micro.py 256 60 | cut -c1-170)"
