# C1 direct-kernel split count (diagnostics): kernel time (warm) and the driver's ms/step
python - <<'PY'
import numpy as np, sys
sys.path.insert(0, '.')
from paper_2405_16911_b200 import siggen
from paper_2405_16911_b200.build import build_tools
build_tools()
siggen.c1_record().astype(np.complex64).tofile('/dev/shm/c1.cf32')
siggen.c1_record()[: 1 << 18].astype(np.complex64).tofile('/dev/shm/c1s.cf32')
PY
for s in ${SPLITS:-0 2 4 8 16 32}; do
  k=$(CYC_DIRECT_SPLITS=$s ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none -k regex:direct -s 20 -c 10 --csv ./tools/stream_bench c1 /dev/shm/c1s.cf32 1 1 2>/dev/null | grep direct | awk -F'","' '{gsub(/"/,"",$NF); s+=$NF; n++} END {print s/n}')
  r=$(CYC_DIRECT_SPLITS=$s ./tools/stream_bench c1 /dev/shm/c1.cf32 5 2)
  echo "splits $s kernel_ns $k $r"
done
