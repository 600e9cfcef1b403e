# round-2 pass bi: lane_sums (value-inner) — full suite, smoke, C5 bench vs HEAD, small configs
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rf 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python bench.py --steps 10 --warmup 3 --no-aux --no-cpu-baseline > gpurun_out/r02bi_bench_new.json 2>/dev/null; python -c "
import json; b=json.loads(open('gpurun_out/r02bi_bench_new.json').read().strip().splitlines()[-1]); print('new ', b['ms_per_step'], b['roofline']['frac'], b['bicgstab_roofline']['k_bicgstab_ms'], b['clocks']['sm_mhz'])"
timeout 1500 python variants/head/bench.py --steps 10 --warmup 3 --no-aux --no-cpu-baseline > gpurun_out/r02bi_bench_head.json 2>/dev/null; python -c "
import json; b=json.loads(open('gpurun_out/r02bi_bench_head.json').read().strip().splitlines()[-1]); print('head', b['ms_per_step'], b['roofline']['frac'], b['bicgstab_roofline']['k_bicgstab_ms'], b['clocks']['sm_mhz'])"
timeout 300 python tools/small_bench.py | cut -c1-200
