# round-2 pass ar: one-cluster CG with 512 vs 256 threads per CTA (C3 nh=16)
mkdir -p gpurun_out
for r in 1 2; do
  echo "512 $(FVB_PKG_ROOT=variants/clt512 timeout 300 python tools/small_bench.py | tail -1 | cut -c1-200)"
  echo "256 $(FVB_PKG_ROOT=variants/clt256 timeout 300 python tools/small_bench.py | tail -1 | cut -c1-200)"
done
for n in 24 32; do
  echo "512 $(FVB_PKG_ROOT=variants/clt512 timeout 300 python tools/cg_micro.py $n 400 | cut -c1-220)"
  echo "256 $(FVB_PKG_ROOT=variants/clt256 timeout 300 python tools/cg_micro.py $n 400 | cut -c1-220)"
done
