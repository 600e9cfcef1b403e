# round-2 pass ax: bench.py --gpus 2 under torchrun with both ranks on one GPU
# (IPC pools, flat team reduction) — correctness of the N>1 bench path
mkdir -p gpurun_out
FVB_DEVICE=0 FVB_SM_SHARE=2 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --edge 48 --steps 2 --warmup 3 --no-aux > gpurun_out/r02ax_n2.log 2>&1; echo "rc=$?"; tail -c 1800 gpurun_out/r02ax_n2.log
