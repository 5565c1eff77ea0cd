#!/bin/bash
# ncu launch list of the C1 streaming driver (2^18-sample prefix; diagnostics).
# `c1_launches.sh warm` keeps caches between kernels (--cache-control none).
python - <<'PY'
import numpy as np, sys
sys.path.insert(0, '.')
from paper_2405_16911_b200 import siggen
from paper_2405_16911_b200.build import build_tools
build_tools()
siggen.c1_record()[: 1 << 18].astype(np.complex64).tofile('/dev/shm/c1s.cf32')
PY
CC=""
[ "$1" = "warm" ] && CC="--cache-control none"
mkdir -p gpurun_out
./tools/stream_bench c1 /dev/shm/c1s.cf32 1 1
ncu --metrics gpu__time_duration.sum --clock-control none $CC -c 60 --csv --log-file gpurun_out/c1_launches.csv ./tools/stream_bench c1 /dev/shm/c1s.cf32 1 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/c1_launches.csv 2>&1 | head -30
