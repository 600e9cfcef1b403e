mkdir -p gpurun_out
for n in 5 7 10; do echo "cg n=$n $(timeout 120 python tools/cg_micro.py $n 300 | cut -c1-170)"; done
for n in 7 10; do echo "bi n=$n $(timeout 120 python tools/bi_micro.py $n 60 | cut -c1-170)"; done
timeout 300 python tools/small_bench.py
timeout 1500 python -m pytest tests -q -m gpu -rf -x 2>&1 | tail -4
