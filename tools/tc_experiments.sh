#!/bin/bash
# Which part bounds the tensor-core fold?  Trace builds with pieces compiled
# out -- results are wrong in those builds (diagnostics):
#   1 no MMAs, 2 no conversion, 3 no proxy fence, 4 no plane stores, 5 no raw loads
for v in ${@:-0 1 2 3 4 5}; do
  echo "== TC_EXPERIMENT=$v"
  lib=$(CYC_NVCC_EXTRA="-DTC_TRACE -DTC_EXPERIMENT=$v" python -c "from paper_2405_16911_b200 import build as b; print(b.build(force=True))") || exit 1
  CYC_LIB=$lib python tools/tc_trace.py 2>&1 | grep -E "kernel:|mma_go interval"
done
