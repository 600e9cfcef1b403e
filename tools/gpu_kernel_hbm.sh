# Per-kernel achieved DRAM bandwidth for one C5 PISO step (every libfvb
# kernel): ncu launch list with duration + DRAM read/write bytes
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/kernels_hbm_c5.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-aux > gpurun_out/kernels_hbm_c5.log 2>&1
tail -c 400 gpurun_out/kernels_hbm_c5.log; ls -la gpurun_out/kernels_hbm_c5.csv
