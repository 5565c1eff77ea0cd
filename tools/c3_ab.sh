#!/bin/bash
# C3 streaming driver: default, without the non-temporal staging copy, without the small fold (diagnostics)
bash tools/stream_prof.sh
echo "== c3 CYC_NO_ZERO_COPY"
CYC_NO_ZERO_COPY=1 CYC_PROFILE=1 ./tools/stream_bench c3 /dev/shm/c3.cf32 1 1 2>&1 | tail -3
echo "== c3 CYC_NO_NT_COPY"
CYC_NO_NT_COPY=1 CYC_PROFILE=1 ./tools/stream_bench c3 /dev/shm/c3.cf32 1 1 2>&1 | tail -3
echo "== c3 CYC_NO_SMALL_FOLD"
CYC_NO_SMALL_FOLD=1 CYC_PROFILE=1 ./tools/stream_bench c3 /dev/shm/c3.cf32 1 1 2>&1 | tail -3
