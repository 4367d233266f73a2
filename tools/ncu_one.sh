#!/bin/bash
# Full ncu capture of one kernel (regex $KREGEX) of the bench workload. TAG names the report.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-C4}; TAG=${TAG:-x}; KREGEX=${KREGEX:-k_sweep}; EXTRA=${EXTRA:-}
ncu --set full --clock-control none --import-source on -k regex:"$KREGEX" -s ${SKIP:-3} -c ${COUNT:-1} \
    -o gpurun_out/${TAG} -f \
    python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline $EXTRA > gpurun_out/ncu_${TAG}.txt 2>&1
echo "ncu rc=$?"
