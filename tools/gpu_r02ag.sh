# round-2 pass ag: rows per thread of the single-block shared-memory solvers
# (C1: 400 rows) — diagnostic builds variants/smem_r{2,4,8} against the product (1)
mkdir -p gpurun_out
for r in 1 2; do
  echo "r1 $(timeout 300 python tools/small_bench.py | head -1 | cut -c1-420)"
  for v in 2 4 8; do
    echo "r$v $(FVB_PKG_ROOT=variants/smem_r$v timeout 300 python tools/small_bench.py | head -1 | cut -c1-420)"
  done
done
