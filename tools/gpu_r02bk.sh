# round-2 pass bk: BiCGStab reductions with one warp per value (M > 3) vs HEAD
mkdir -p gpurun_out
for r in 1 2; do
for n in 64 128 256; do
  it=60; [ $n = 256 ] && it=30
  echo "new  $n $(timeout 600 python tools/bi_micro.py $n $it | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:round(v,1) for k,v in d.items() if "us" in k})')"
  echo "head $n $(FVB_PKG_ROOT=variants/head timeout 600 python tools/bi_micro.py $n $it | python -c 'import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:round(v,1) for k,v in d.items() if "us" in k})')"
done
done
