timeout 1200 python -m pytest tests/test_gpu_configs.py tests/test_gpu_solvers.py -q 2>&1 | tail -15
FVB_DEVICE=0 FVB_SM_SHARE=2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --edge 64 --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | grep -v Warn | tail -3 | cut -c1-1500
