# Evidence run: default bench line, ncu launch list, ncu --set full of k_cg
# and k_bicgstab3 (reports exported to CSV on the box: the .ncu-rep files
# are too large to travel back)
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/bench_final.log 2>&1; tail -c 4000 gpurun_out/bench_final.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-aux > gpurun_out/ncu_launch_c5.log 2>&1; tail -c 300 gpurun_out/ncu_launch_c5.log
for spec in "k_cg:2:cg" "k_bicgstab3:1:bi"; do
  IFS=: read -r kname skip tag <<< "$spec"
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$kname -s $skip -c 1 \
    -o /tmp/prof_$tag python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-aux \
    > gpurun_out/ncu_full_$tag.log 2>&1; tail -2 gpurun_out/ncu_full_$tag.log
  ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$tag.csv 2>&1
  ncu -i /tmp/prof_$tag.ncu-rep --page details --csv > gpurun_out/ncu_details_$tag.csv 2>&1
  ncu -i /tmp/prof_$tag.ncu-rep --page source --csv --print-source sass > /tmp/src_$tag.csv 2>&1
  gzip -c /tmp/src_$tag.csv > gpurun_out/ncu_source_$tag.csv.gz
  ls -la gpurun_out/ncu_*_$tag.*
done
