# round-2 pass be: grid-reduction latency probe (tools/probe/barrier_probe.cu)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/barrier_probe tools/probe/barrier_probe.cu && timeout 300 /tmp/barrier_probe
