# Evidence run: default bench line, ncu launch list, ncu --set full of k_cg and k_bicgstab3
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench_final.log 2>&1; tail -c 4000 gpurun_out/bench_final.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-aux > gpurun_out/ncu_launch_c5.log 2>&1; tail -c 300 gpurun_out/ncu_launch_c5.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_cg -s 2 -c 1 -o gpurun_out/prof_k_cg_c5 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-aux > gpurun_out/ncu_full_c5.log 2>&1; tail -2 gpurun_out/ncu_full_c5.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_bicgstab3 -s 1 -c 1 -o gpurun_out/prof_k_bi_c5 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-aux > gpurun_out/ncu_full_bi.log 2>&1; tail -2 gpurun_out/ncu_full_bi.log
