"""Host trace of C5 e2e steps (CYC_TRACE=1; diagnostics)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_16911_b200 as cyc
from paper_2405_16911_b200 import siggen
x = siggen.c5_record(n=1 << 26)
est = cyc.CyclicCorrelator(cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=8192, lag_spec=cyc.LagSpec.Explicit(range(256)),
                           flags=cyc.Flags.BOTH, emit_frames=False))
px = cyc.host_alloc(x.shape); px[:] = x
out = cyc.host_alloc((1, 2, 256 * 8192), dtype=np.complex128)
for i in range(3):
    t0 = time.perf_counter(); est.reset(); est.push(px); t1 = time.perf_counter(); est.average_all(out=out); t2 = time.perf_counter()
    print(f"step {i}: push {1e3*(t1-t0):.2f} ms avg {1e3*(t2-t1):.2f} ms", flush=True)
