# round-2 pass v: fence-based acquire, team kernels without spills
mkdir -p gpurun_out
for n in 256 128; do echo "cg n=$n $(timeout 300 python tools/cg_micro.py $n 400 | cut -c1-170)"; done
echo "bi $(timeout 300 python tools/bi_micro.py 256 60 | cut -c1-170)"
timeout 900 python tools/team_bench.py 128 1 2 4 > gpurun_out/r02v_team_gpu.log 2>&1; cat gpurun_out/r02v_team_gpu.log
FVB_TEAM_SCOPE=sys timeout 900 python tools/team_bench.py 128 2 4 > gpurun_out/r02v_team_sys.log 2>&1; cat gpurun_out/r02v_team_sys.log
timeout 900 python tools/stress_determinism.py --step2 600 --out gpurun_out/r02v_step2.jsonl > gpurun_out/r02v_step2.log 2>&1; tail -2 gpurun_out/r02v_step2.log
timeout 2400 python -m pytest tests -q -m gpu -rf 2>&1 | tail -4
