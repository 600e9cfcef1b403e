# round-2 pass av: persistent CG grid size on mid-size systems (grid barrier
# cost vs rows per thread): 148 (auto) vs 112 / 74 / 37 blocks
mkdir -p gpurun_out
for n in 48 64 80 100; do
  for g in 0 112 74 37; do
    echo "g$g $(timeout 600 python tools/cg_micro.py $n 400 grid=$g | cut -c1-150)"
  done
done
