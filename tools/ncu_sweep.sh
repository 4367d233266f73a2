#!/bin/bash
# ncu evidence for the bench workload: launch list (cold, serialised) + a full capture of k_sweep.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-C4}
TAG=${TAG:-r1}
ncu --metrics gpu__time_duration.sum --clock-control none -s 8 -c 40 --csv \
    --log-file gpurun_out/launches_${CFG}_${TAG}.csv \
    python bench.py --config $CFG --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench_stdout.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 3 -c 1 \
    -o gpurun_out/sweep_${CFG}_${TAG} -f \
    python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_stdout.txt 2>&1
ncu --set full --clock-control none -k regex:"k_scan|k_scatter|k_rank" -s 6 -c 3 \
    -o gpurun_out/sort_${CFG}_${TAG} -f \
    python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_sort_stdout.txt 2>&1
ls -la gpurun_out
