#!/bin/bash
# C3 streaming driver with and without the small-fold path (diagnostics)
bash tools/stream_prof.sh
echo "== c3 CYC_NO_SMALL_FOLD"
CYC_NO_SMALL_FOLD=1 CYC_PROFILE=1 ./tools/stream_bench c3 /dev/shm/c3.cf32 1 1 2>&1 | tail -3
