# round-2 pass ae: CUDA-graph replay of the step's assembly segments,
# rhie_chow_flux on the device, and the reference's own unit tests run
# against the package (tools/ref_conformance.py; staged copy in baseline/_ref_tests)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rf -x 2>&1 | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for r in 1 2; do
  echo "graphs    $(timeout 300 python tools/small_bench.py | tr '\n' ' ' | cut -c1-1000)"
  echo "no-graphs $(timeout 300 python tools/small_bench.py --no-graphs | tr '\n' ' ' | cut -c1-1000)"
done
timeout 1200 python tools/ref_conformance.py run > gpurun_out/r02ae_conformance.json 2> gpurun_out/r02ae_conformance.log
echo "conformance rc=$?"; head -c 3000 gpurun_out/r02ae_conformance.json
