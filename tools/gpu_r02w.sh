# round-2 pass w: lean block reductions for the single-block and cluster paths
mkdir -p gpurun_out
for n in 7 20 26; do echo "cg n=$n $(timeout 120 python tools/cg_micro.py $n 300 | cut -c1-170)"; done
for n in 7 20; do echo "bi n=$n $(timeout 120 python tools/bi_micro.py $n 60 | cut -c1-170)"; done
for n in 256 128; do echo "cg n=$n $(timeout 300 python tools/cg_micro.py $n 400 | cut -c1-170)"; done
timeout 300 python tools/small_bench.py
timeout 900 python tools/team_bench.py 128 2 > gpurun_out/r02w_team.log 2>&1; cat gpurun_out/r02w_team.log
timeout 600 python bench.py --edge 96 --steps 3 --warmup 3 --no-aux --no-cpu-baseline > gpurun_out/r02w_bench96.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r02w_bench96.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['cg_iters_per_step'], d['iterations_per_step'])"
timeout 900 python tools/stress_determinism.py --edge 24 --reseed 300 --fresh 5 --big 0 --out gpurun_out/r02w_stress24.jsonl > gpurun_out/r02w_stress24.log 2>&1; tail -1 gpurun_out/r02w_stress24.log
timeout 900 python tools/stress_determinism.py --edge 10 --reseed 300 --fresh 5 --big 0 --out gpurun_out/r02w_stress10.jsonl > gpurun_out/r02w_stress10.log 2>&1; tail -1 gpurun_out/r02w_stress10.log
timeout 2400 python -m pytest tests -q -m gpu -rf 2>&1 | tail -4
