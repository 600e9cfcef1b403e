mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cluster_probe tools/probe/cluster_probe.cu && /tmp/cluster_probe
for n in 5 7 10 12 15; do echo "cg n=$n $(timeout 120 python tools/cg_micro.py $n 300 | cut -c1-170)"; done
for n in 7 12; do echo "bi n=$n $(timeout 120 python tools/bi_micro.py $n 60 | cut -c1-200)"; done
