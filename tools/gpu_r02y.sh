# round-2 pass y: driver-shaped bench runs (both arms) and the 2-rank path on one GPU
mkdir -p gpurun_out
t0=$(date +%s); timeout 1800 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02y_ref.json 2> gpurun_out/r02y_ref.err; echo "ref arm $(( $(date +%s) - t0 )) s"; tail -c 300 gpurun_out/r02y_ref.json
t0=$(date +%s); timeout 2400 python bench.py --steps 20 --warmup 5 > gpurun_out/r02y_bench.json 2> gpurun_out/r02y_bench.err; echo "bench $(( $(date +%s) - t0 )) s"; tail -c 300 gpurun_out/r02y_bench.json
FVB_DEVICE=0 FVB_SM_SHARE=2 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --edge 48 --steps 2 --warmup 3 --no-aux > gpurun_out/r02y_n2.log 2>&1; tail -c 1500 gpurun_out/r02y_n2.log
