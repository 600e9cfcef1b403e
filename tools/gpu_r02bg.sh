# round-2 pass bg: lane_sums vs HEAD at 256^3 (CG repeated, BiCGStab) and 128^3 BiCGStab
mkdir -p gpurun_out
for r in 1 2; do
  echo "new  $(timeout 600 python tools/cg_micro.py 256 100 | cut -c1-200)"
  echo "head $(FVB_PKG_ROOT=variants/head timeout 600 python tools/cg_micro.py 256 100 | cut -c1-200)"
done
for n in 128 256; do
  echo "new  $(timeout 600 python tools/bi_micro.py $n 40 | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:v for k,v in d.items() if "us" in k or "ms" in k})')"
  echo "head $(FVB_PKG_ROOT=variants/head timeout 600 python tools/bi_micro.py $n 40 | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:v for k,v in d.items() if "us" in k or "ms" in k})')"
done
