# round-2 pass bq: explicit-index CG pass A with every gather issued first (as the coded path) vs HEAD
mkdir -p gpurun_out
for r in 1 2; do
  for a in "128 400 explicit" "126 200 perm" "64 400 explicit"; do
    echo "new  $a $(timeout 900 python tools/cg_micro.py $a | cut -c1-160)"
    echo "head $a $(FVB_PKG_ROOT=variants/head timeout 900 python tools/cg_micro.py $a | cut -c1-160)"
  done
done
