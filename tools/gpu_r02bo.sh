# round-2 pass bo: the reference's own tests incl. test_report / test_acceptance against the package
mkdir -p gpurun_out
timeout 2400 python tools/ref_conformance.py run > gpurun_out/r02bo_conformance.json 2> gpurun_out/r02bo_conformance.log
echo "rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/r02bo_conformance.json')); print(d['files']); [print(f) for f in d['failed']]"
