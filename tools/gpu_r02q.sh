mkdir -p gpurun_out
nproc
timeout 1200 python tools/bicgstab_diag.py c4 > gpurun_out/r02q_bidiag_c4.log 2>&1; cat gpurun_out/r02q_bidiag_c4.log
