"""Host trace of e2e C2 steps (CYC_TRACE=1; diagnostics)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_16911_b200 as cyc
from paper_2405_16911_b200 import siggen
L = 1 << 24
x = siggen.c2_record(n=L)
cfg = cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=1024, lag_spec=cyc.LagSpec.Explicit(range(64)),
                          flags=cyc.Flags.BOTH, emit_frames=False)
est = cyc.CyclicCorrelator(cfg)
px = cyc.host_alloc(x.shape); px[:] = x
out = cyc.host_alloc((1, 2, 65536), dtype=np.complex128)
for i in range(4):
    print("---- step", i, flush=True)
    est.reset(); est.push(px); est.average_all(out=out)
