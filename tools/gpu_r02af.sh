# round-2 pass af: where the C1 momentum solve spends its time (single-block
# shared-memory BiCGStab, 400 rows x 3 components): full ncu capture with source
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bicgstab3 -s 3 -c 1 \
  -o gpurun_out/r02af_bi_c1 -f python tools/c1_steps.py 3 > gpurun_out/r02af_ncu.log 2>&1; tail -3 gpurun_out/r02af_ncu.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cg -s 6 -c 1 \
  -o gpurun_out/r02af_cg_c1 -f python tools/c1_steps.py 3 > gpurun_out/r02af_ncu2.log 2>&1; tail -3 gpurun_out/r02af_ncu2.log
for r in bi cg; do
  ncu -i gpurun_out/r02af_${r}_c1.ncu-rep --page source --csv --print-source cuda > gpurun_out/r02af_${r}_source.csv 2>/dev/null
  ncu -i gpurun_out/r02af_${r}_c1.ncu-rep --page details --csv > gpurun_out/r02af_${r}_details.csv 2>/dev/null
done
ls -la gpurun_out/ | grep r02af
