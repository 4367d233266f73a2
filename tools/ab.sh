#!/bin/bash
# A/B on one box: optional gpu tests, then C4 (and $CONFIGS) bench lines for the
# in-tree libdem.so and every paper_1301_1714_b200/variants/libdem_*.so.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-ab}
python -c "from paper_1301_1714_b200 import build as B; B.build()" > gpurun_out/build_${TAG}.log 2>&1
if [ -n "$TESTS" ]; then
  timeout ${TEST_TIMEOUT:-1200} python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_${TAG}.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
  tail -4 gpurun_out/pytest_${TAG}.log
fi
run() {  # $1 label, $2 lib or "", $3 config
  DEM_LIB=$2 timeout 300 python bench.py --config $3 --steps ${STEPS:-50} --warmup 10 --no-cpu-baseline --no-e2e \
    > gpurun_out/ab_${TAG}_$1_$3.json 2> gpurun_out/ab_${TAG}_$1_$3.err
  python - "$1" "$3" "gpurun_out/ab_${TAG}_$1_$3.json" <<'PY'
import json, sys
try:
    d = json.load(open(sys.argv[3]))
    print(sys.argv[1], sys.argv[2], round(d["ms_per_step"], 4), "prof", round(d["ms_per_step_profiled"], 4),
          {k: round(v, 4) for k, v in d["kernel_ms_avg"].items() if v}, "frac", round(d["roofline"]["frac"], 3),
          "cbar", round(d["config"].get("c_bar", 0), 3), d["clocks"]["sm_mhz"], flush=True)
except Exception as e:
    print(sys.argv[1], sys.argv[2], "FAILED", e)
PY
}
for rep in $(seq ${REPS:-1}); do
for c in ${CONFIGS:-C4}; do
  run main "" $c
  for f in paper_1301_1714_b200/variants/libdem_*.so; do
    [ -e "$f" ] || continue
    v=$(basename $f .so); v=${v#libdem_}
    run $v $f $c
  done
done
done
