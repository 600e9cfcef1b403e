mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bicgstab3 -c 1 -o /tmp/prof_bi7 python tools/bi_micro.py 7 60 > gpurun_out/r02ab_ncu_bi7.log 2>&1; tail -2 gpurun_out/r02ab_ncu_bi7.log
ncu -i /tmp/prof_bi7.ncu-rep --page details --csv > gpurun_out/r02ab_bi7_details.csv 2>&1
ncu -i /tmp/prof_bi7.ncu-rep --page source --csv --print-source sass > gpurun_out/r02ab_bi7_source.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cg -c 1 -o /tmp/prof_cg7 python tools/cg_micro.py 7 300 > gpurun_out/r02ab_ncu_cg7.log 2>&1; tail -2 gpurun_out/r02ab_ncu_cg7.log
ncu -i /tmp/prof_cg7.ncu-rep --page details --csv > gpurun_out/r02ab_cg7_details.csv 2>&1
ncu -i /tmp/prof_cg7.ncu-rep --page source --csv --print-source sass > gpurun_out/r02ab_cg7_source.csv 2>&1
ls -la gpurun_out/r02ab_*
