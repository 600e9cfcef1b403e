# round-2 pass bu: compute-sanitizer memcheck over the round-2 additions
mkdir -p gpurun_out
timeout 1800 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_r02.py > gpurun_out/r02bu_memcheck.log 2>&1; echo "rc=$?"; tail -8 gpurun_out/r02bu_memcheck.log
