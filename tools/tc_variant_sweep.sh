#!/bin/bash
# Build tensor-core fold variants into _diag/ (CYC_NVCC_EXTRA) and time the fold
# on C2 and C5 (tools/fold_time.py); the product library is untouched.
for v in "$@"; do
  lib=$(CYC_NVCC_EXTRA="$v" python -c "from paper_2405_16911_b200 import build as b; print(b.build())") || continue
  CYC_LIB=$lib CYC_NVCC_EXTRA="$v" timeout 300 python tools/fold_time.py c2 c5
done
