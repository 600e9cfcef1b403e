export FVB_DEVICE=0 FVB_SM_SHARE=2
timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/ipc_team_check.py 8 2>&1 | grep -v Warn | tail -15
unset FVB_SM_SHARE
timeout 600 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 1200 python bench.py --no-cpu-baseline 2>&1 | tail -c 1800
