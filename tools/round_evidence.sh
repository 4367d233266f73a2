#!/bin/bash
# Round evidence: full bench line (cpu_baseline + e2e), reference arm, ncu launch list and
# full captures of the top kernels. Everything lands in gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r1}
python bench.py --steps ${STEPS:-50} --warmup 10 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"
python bench.py --config C3 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_C3_${TAG}.json 2>&1
python bench.py --config C2 --model simple --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_C2simple_${TAG}.json 2>&1
python bench.py --config C2 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_C2practical_${TAG}.json 2>&1
python bench.py --sweep tpp --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_tpp_${TAG}.json 2>&1
python bench.py --sweep half --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_half_${TAG}.json 2>&1
python bench.py --sweep lanes --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_lanes_${TAG}.json 2>&1
python bench.py --config C5 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_${TAG}.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 40 --csv \
    --log-file gpurun_out/launches_C4_${TAG}.csv \
    python bench.py --steps 10 --warmup 5 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_force|k_detect" -s 8 -c 2 \
    -o gpurun_out/full_C4_${TAG} -f \
    python bench.py --steps 2 --warmup 5 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo "ncu full rc=$?"
ncu --set full --clock-control none -k regex:"k_scan|k_tile|k_scatter|k_rank|k_mv" -s 12 -c 4 \
    -o gpurun_out/sort_C4_${TAG} -f \
    python bench.py --steps 2 --warmup 5 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo "ncu sort rc=$?"
