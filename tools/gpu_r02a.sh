# round-2 first GPU pass: suite, determinism stress, both bench arms
mkdir -p gpurun_out
(nproc; lscpu | head -20; free -g) > gpurun_out/r02a_host.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -rf --durations=10 > gpurun_out/r02a_tests.log 2>&1
tail -5 gpurun_out/r02a_tests.log
timeout 1500 python tools/stress_determinism.py --out gpurun_out/r02_stress.jsonl > gpurun_out/r02a_stress.log 2>&1
tail -4 gpurun_out/r02a_stress.log
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r02a_ref.json 2> gpurun_out/r02a_ref.err
tail -c 600 gpurun_out/r02a_ref.json
timeout 900 python bench.py --steps 5 --warmup 3 --no-aux > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
tail -c 1500 gpurun_out/r02a_bench.json
