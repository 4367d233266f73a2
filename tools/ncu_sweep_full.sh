#!/bin/bash
# ncu --set full of one k_detect + one k_force launch of the C4 bench (in-tree libdem).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-x}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_force|k_detect" -s ${SKIP:-8} -c 2 \
    -o gpurun_out/full_${CFG:-C4}_${TAG} -f \
    python bench.py --config ${CFG:-C4} --steps 2 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu full rc=$?"
