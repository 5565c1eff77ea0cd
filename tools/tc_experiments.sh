#!/bin/bash
# Which part bounds the tensor-core fold?  Trace builds with the MMAs (1) or the
# conversions (2) compiled out -- results are wrong in those builds (diagnostics).
for v in 0 1 2; do
  echo "== TC_EXPERIMENT=$v"
  CYC_NVCC_EXTRA="-DTC_TRACE -DTC_EXPERIMENT=$v" python -c "from paper_2405_16911_b200 import build as b; b.build(force=True)" || exit 1
  python tools/tc_trace.py 2>&1 | grep -E "kernel:|mma_go interval"
done
