#!/bin/bash
# Round evidence in one gpurun call: smoke, pytest -m gpu, the default bench
# line (cpu_baseline + e2e), C3/C5/C2 lines, the ablation lines, the ncu launch
# list, one --set full capture of the sweep (-> profiles/traffic json) and of
# k_merge. Everything lands in gpurun_out/ with the TAG.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r2}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"
if [ -z "$NOTEST" ]; then
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?"
  tail -3 gpurun_out/pytest_${TAG}.log
fi
python bench.py --steps ${STEPS:-20} --warmup 5 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"
python bench.py --config C3 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_C3_${TAG}.json 2>&1
python bench.py --config C5 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5_${TAG}.json 2>&1
python bench.py --config C2 --model simple --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_C2simple_${TAG}.json 2>&1
python bench.py --config C2 --steps 100 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_C2practical_${TAG}.json 2>&1
if [ -z "$NOABL" ]; then
  for s in tpp half lanes; do
    python bench.py --sweep $s --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${s}_${TAG}.json 2>&1
  done
fi
ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 40 --csv \
    --log-file gpurun_out/launches_C4_${TAG}.csv \
    python bench.py --steps 10 --warmup 5 --reps 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_force|k_detect" -s 8 -c 2 \
    -o gpurun_out/full_C4_${TAG} -f \
    python bench.py --steps 2 --warmup 5 --reps 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu full rc=$?"
ncu --set full --clock-control none -k regex:"k_merge" -s 4 -c 1 \
    -o gpurun_out/merge_C4_${TAG} -f \
    python bench.py --steps 2 --warmup 5 --reps 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo "ncu merge rc=$?"
