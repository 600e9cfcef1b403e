# round-2 HEAD check after the last Python changes (report PNGs): suite + smoke
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rf 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python tools/report_run.py 64 3 gpurun_out/r02br_report > gpurun_out/r02br_report.log 2>&1; tail -3 gpurun_out/r02br_report.log; ls gpurun_out/r02br_report
