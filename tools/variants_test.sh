#!/bin/bash
# parity tests of the detect path + bench of every built variant (paper_1301_1714_b200/variants/*.so)
cd "$(dirname "$0")/.."
for f in paper_1301_1714_b200/variants/libdem_*.so; do
  v=$(basename $f .so)
  DEM_LIB=$f timeout 600 python -m pytest tests -m gpu -x -q -k "${PYTEST_K:-T2 or contact or analysis or band or mono or bitwise}" > gpurun_out/vt_${v}.log 2>&1
  echo "$v tests: $(tail -1 gpurun_out/vt_${v}.log)"
done
for c in ${CONFIGS:-C4 C3}; do CFG=$c STEPS=${STEPS:-50} bash tools/variants.sh; done
