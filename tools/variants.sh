#!/bin/bash
# bench every built variant of libdem (paper_1301_1714_b200/variants/*.so) on $CFG
cd "$(dirname "$0")/.."
CFG=${CFG:-C4}
for f in paper_1301_1714_b200/variants/libdem_*.so; do
  v=$(basename $f .so)
  DEM_LIB=$f python bench.py --config $CFG --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/var_${CFG}_${v}.json 2>gpurun_out/var_${CFG}_${v}.err
  python -c "import json; d=json.load(open('gpurun_out/var_${CFG}_${v}.json')); print('$v', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['kernel_ms_avg'].items() if v})"
done
