#!/bin/bash
# tensor-core fold ring depth / converter-warp variants (rebuild per variant)
for v in "" "-DTC_NR_SELF=6 -DTC_NP_SELF=3" "-DTC_NR_SELF=4 -DTC_NP_SELF=4" "-DTC_TNC=8" "-DTC_TNC=16"; do
  echo "== $v"
  lib=$(CYC_NVCC_EXTRA="$v" python -c "from paper_2405_16911_b200 import build as b; print(b.build(force=True))") || continue
  export CYC_LIB=$lib  # the variant loads from its own _diag/ directory; the product library is untouched
  python tools/host_bound.py | tail -1
  HB_PROF=1 python tools/host_bound.py | tail -1
done
