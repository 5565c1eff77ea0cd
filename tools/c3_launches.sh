#!/bin/bash
# ncu launch list of the C3 recursive streaming driver on a 2^22-sample prefix (diagnostics).
# `c3_launches.sh warm` keeps caches between kernels (--cache-control none): in-stream durations.
python - <<'PY'
import numpy as np, sys
sys.path.insert(0, '.')
from paper_2405_16911_b200 import siggen
from paper_2405_16911_b200.build import build_tools
build_tools()
siggen.c3_record(n=2**22).astype(np.complex64).tofile('/dev/shm/c3s.cf32')
PY
CC=""
[ "$1" = "warm" ] && CC="--cache-control none"
mkdir -p gpurun_out
./tools/stream_bench c3 /dev/shm/c3s.cf32 1 1
ncu --metrics gpu__time_duration.sum --clock-control none $CC -c 60 --csv --log-file gpurun_out/c3_launches.csv ./tools/stream_bench c3 /dev/shm/c3s.cf32 1 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/c3_launches.csv 2>&1 | head -30
