# round-2 pass aq: threads per CTA of the one-cluster CG (C3 nh=16) —
# diagnostic build variants/clt512 (512 threads, 2 rows per thread) vs 1024
mkdir -p gpurun_out
for r in 1 2; do
  echo "1024 $(timeout 300 python tools/small_bench.py | tail -1 | cut -c1-200)"
  echo "512  $(FVB_PKG_ROOT=variants/clt512 timeout 300 python tools/small_bench.py | tail -1 | cut -c1-200)"
done
echo "1024 $(timeout 300 python tools/cg_micro.py 24 400 | cut -c1-220)"
echo "512  $(FVB_PKG_ROOT=variants/clt512 timeout 300 python tools/cg_micro.py 24 400 | cut -c1-220)"
