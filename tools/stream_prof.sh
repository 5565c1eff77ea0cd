#!/bin/bash
# per-phase host profile (CYC_PROFILE=1) of the C1/C3 streaming drivers (diagnostics)
python - <<'PY'
import numpy as np, sys
sys.path.insert(0, '.')
from paper_2405_16911_b200 import siggen
from paper_2405_16911_b200.build import build_tools
build_tools()
siggen.c1_record().astype(np.complex64).tofile('/dev/shm/c1.cf32')
siggen.c3_record(n=2**28).astype(np.complex64).tofile('/dev/shm/c3.cf32')
PY
for c in c1 c3; do
  echo "== $c"
  CYC_PROFILE=1 ./tools/stream_bench $c /dev/shm/$c.cf32 1 1 2>&1 | tail -8
done
