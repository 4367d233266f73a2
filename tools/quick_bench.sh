#!/bin/bash
# Quick A/B: gpu tests (optional) + C4/C3/C2 bench lines (no cpu baseline, no e2e).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-q}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1
if [ -z "$NOTEST" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
  tail -2 gpurun_out/pytest_${TAG}.log
fi
for c in ${CONFIGS:-C4 C3 C2}; do
  ${ENVV} python bench.py --config $c --steps ${STEPS:-50} --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bq_${c}_${TAG}.json 2> gpurun_out/bq_${c}_${TAG}.err
  python - <<PY
import json
d=json.load(open("gpurun_out/bq_${c}_${TAG}.json"))
print("${c}", round(d["ms_per_step"],4), "prof", round(d["ms_per_step_profiled"],4), {k:round(v,4) for k,v in d["kernel_ms_avg"].items() if v}, "frac", round(d["roofline"]["frac"],3), d["clocks"]["sm_mhz"])
PY
done
