# round-2 pass as: one-cluster CG, 1024 (product) vs 512 threads per CTA vs
# the full grid, at 32^3 and 34^3 (cluster range up to 40,000 rows)
mkdir -p gpurun_out
for n in 28 32 34; do
  echo "1024 $(timeout 300 python tools/cg_micro.py $n 400 | cut -c1-120)"
  echo "512  $(FVB_PKG_ROOT=variants/clt512 timeout 300 python tools/cg_micro.py $n 400 | cut -c1-120)"
  echo "grid $(timeout 300 python tools/cg_micro.py $n 400 nocluster | cut -c1-120)"
done
