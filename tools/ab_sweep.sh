#!/bin/bash
# A/B of the default sweep against --sweep variants on one box: optional
# pytest -m gpu, then per config the default line and each variant's line
# (no cpu baseline, no e2e). TAG, CONFIGS, VARIANTS (name or name:extra_flags), STEPS, NOTEST.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-ab}
if [ -z "$NOTEST" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
  tail -2 gpurun_out/pytest_${TAG}.log
fi
for c in ${CONFIGS:-C4 C3}; do
  for vv in full ${VARIANTS:-split}; do
    v=${vv%%:*}; xf=0; [ "$vv" != "$v" ] && xf=${vv#*:}; v=$vv
    python bench.py --config $c --sweep ${vv%%:*} --extra-flags $xf --steps ${STEPS:-50} --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/ab_${c}_${v}_${TAG}.json 2> gpurun_out/ab_${c}_${v}_${TAG}.err
    python - <<PY
import json
try:
    d=json.load(open("gpurun_out/ab_${c}_${v}_${TAG}.json"))
    print("${c} ${v}", round(d["ms_per_step"],4), "prof", round(d["ms_per_step_profiled"],4), {k:round(v,4) for k,v in d["kernel_ms_avg"].items() if v}, "frac", round(d["roofline"]["frac"],3), "step_frac", round(d["roofline"]["step_frac"],3), d["clocks"]["sm_mhz"])
except Exception as e:
    print("${c} ${v} failed", e)
PY
  done
done
