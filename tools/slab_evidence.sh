#!/bin/bash
# Slab per-rank cost: ncu launch lists of P = 2 in-process slab
# ranks on C4/2 and of one GPU holding one rank's share (the bed narrowed in
# z), both from tools/slab_launches.py; summaries via tools/launch_summary.py.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-slab}
python tools/slab_launches.py --scale 2 --P 2 > gpurun_out/slab_P2_${TAG}.log 2>&1; echo "slab P2 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_slab_P2_${TAG}.csv \
    python tools/slab_launches.py --scale 2 --P 2 > /dev/null 2>&1; echo "ncu P2 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_single_z2_${TAG}.csv \
    python tools/slab_launches.py --scale 2 --P 1 --z 2 > /dev/null 2>&1; echo "ncu z2 rc=$?"
