#!/bin/bash
# bench.py --gpus N under torchrun with all ranks on the one GPU of a gpurun box
# (DEM_BENCH_SHARE_GPU=1, gloo): a functional check of the multi-process slab
# path (CUDA IPC exchange); the times are GPU time-slicing, not scaling.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for N in ${NS:-2 4}; do
  DEM_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port $((29500 + N)) bench.py --gpus $N --steps ${STEPS:-10} \
    --warmup 3 --reps 1 --no-cpu-baseline --no-e2e > gpurun_out/shared_N$N.json 2> gpurun_out/shared_N$N.err
  echo "N=$N rc=$?"; tail -c 400 gpurun_out/shared_N$N.json; echo
done
