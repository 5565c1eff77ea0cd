#!/bin/bash
# converter stage-group variants of the tensor-core fold (rebuild per variant):
# parity on the fused/fuzz suites, then the C2 device step and fold time
for v in "$@"; do
  echo "== $v"
  lib=$(CYC_NVCC_EXTRA="$v" python -c "from paper_2405_16911_b200 import build as b; print(b.build(force=True))") || continue
  export CYC_LIB=$lib  # the variant loads from its own _diag/ directory; the product library is untouched
  timeout 300 python -m pytest tests/test_gpu_fused.py tests/test_gpu_fuzz.py -m gpu -x -q 2>&1 | tail -1
  timeout 120 python tools/host_bound.py | tail -1
  HB_PROF=1 timeout 120 python tools/host_bound.py | tail -1
done
