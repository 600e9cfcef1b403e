mkdir -p gpurun_out
for n in 256 128; do for o in tile notile; do echo "bi n=$n $o $(timeout 300 python tools/bi_micro.py $n 60 box $o | cut -c1-330)"; done; done
timeout 900 python -m pytest tests/test_gpu_solvers.py -q -rf -k "tiled or stencil or batched" 2>&1 | tail -3
