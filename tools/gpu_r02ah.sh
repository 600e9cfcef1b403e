# round-2 pass ah: cluster size of the one-cluster solvers (C3 nh=16: 16,640
# rows) — diagnostic builds variants/cl{8,4} against the product (16)
mkdir -p gpurun_out
for r in 1 2; do
  echo "cl16 $(timeout 300 python tools/small_bench.py | tail -1 | cut -c1-300)"
  for v in 8 4; do
    echo "cl$v $(FVB_PKG_ROOT=variants/cl$v timeout 300 python tools/small_bench.py | tail -1 | cut -c1-300)"
  done
done
