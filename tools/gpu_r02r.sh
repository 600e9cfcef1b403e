mkdir -p gpurun_out
BIDIAG_CURVE=50:80 timeout 1800 python tools/bicgstab_diag.py c4 > gpurun_out/r02r_bicurve_c4.log 2>&1; cat gpurun_out/r02r_bicurve_c4.log
