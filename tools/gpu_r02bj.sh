# round-2 final evidence (driver flags): suite + smoke, bench (both arms), ncu launch list and
# full captures of k_cg and k_bicgstab3 (CSV exported on the box)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rf --durations=20 > gpurun_out/r02bj_tests.log 2>&1; tail -25 gpurun_out/r02bj_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02bj_smoke.log 2>&1; tail -2 gpurun_out/r02bj_smoke.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02bj_ref.json 2> gpurun_out/r02bj_ref.err; tail -c 400 gpurun_out/r02bj_ref.json
timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r02bj_bench.json 2> gpurun_out/r02bj_bench.err; tail -c 600 gpurun_out/r02bj_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02bj_launches_c5.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-aux > gpurun_out/r02bj_ncu_launch.log 2>&1; tail -c 300 gpurun_out/r02bj_ncu_launch.log
for spec in "k_cg:2:cg" "k_bicgstab3:1:bi"; do
  IFS=: read -r kname skip tag <<< "$spec"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$kname -s $skip -c 1 \
    -o /tmp/prof_$tag python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-aux \
    > gpurun_out/r02bj_ncu_full_$tag.log 2>&1; tail -2 gpurun_out/r02bj_ncu_full_$tag.log
  ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > gpurun_out/r02bj_ncu_raw_$tag.csv 2>&1
  ncu -i /tmp/prof_$tag.ncu-rep --page details --csv > gpurun_out/r02bj_ncu_details_$tag.csv 2>&1
done
