# C2 (gen_cavity(128), BASELINE configs[1]) evidence: bench line, launch list,
# ncu --set full of one k_cg launch exported to CSV on the box
mkdir -p gpurun_out
timeout 900 python bench.py --config c2 --no-aux > gpurun_out/bench_c2.log 2>&1; tail -c 1500 gpurun_out/bench_c2.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c2.csv python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-aux \
  > gpurun_out/ncu_launch_c2.log 2>&1; tail -c 200 gpurun_out/ncu_launch_c2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cg -s 2 -c 1 -o /tmp/prof_cg128 \
  python bench.py --config c2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-aux > gpurun_out/ncu_full_cg128.log 2>&1
tail -2 gpurun_out/ncu_full_cg128.log
ncu -i /tmp/prof_cg128.ncu-rep --page raw --csv > gpurun_out/ncu_raw_cg128.csv 2>&1
