mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_team.py -q -k ipc 2>&1 | tail -2
FVB_DEVICE=0 FVB_SM_SHARE=2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --n 64 --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | grep -v Warn | tail -3 | cut -c1-1500
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_c5.log 2>&1; tail -c 600 gpurun_out/ncu_launch_c5.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_cg -s 2 -c 1 -o gpurun_out/prof_k_cg_c5 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_c5.log 2>&1; tail -3 gpurun_out/ncu_full_c5.log
