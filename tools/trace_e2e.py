"""Host-side timeline of one e2e C2 step (diagnostics)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
import paper_2405_16911_b200 as cyc
from paper_2405_16911_b200 import siggen
L = 1 << 24
x = siggen.c2_record(n=L)
cfg = cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=1024, lag_spec=cyc.LagSpec.Explicit(range(64)),
                          flags=cyc.Flags.BOTH, emit_frames=False)
est = cyc.CyclicCorrelator(cfg)
px = cyc.host_alloc(x.shape); px[:] = x
o1 = np.zeros(65536, np.complex128); o2 = np.zeros(65536, np.complex128)
Lb = cyc.lib()
for rep in range(5):
    t0 = time.perf_counter(); est.reset(); t1 = time.perf_counter()
    rc = Lb.cyc_push(est._h, px.ctypes.data, None, L, cyc._SINK(0), None); t2 = time.perf_counter()
    est.average(flag=1, out=o1); t3 = time.perf_counter(); est.average(flag=2, out=o2); t4 = time.perf_counter()
    print(f"reset {1e3*(t1-t0):.3f} push {1e3*(t2-t1):.3f} avg1 {1e3*(t3-t2):.3f} avg2 {1e3*(t4-t3):.3f} total {1e3*(t4-t0):.3f}")
# python-side push overhead
for rep in range(3):
    est.reset()
    t1 = time.perf_counter(); est.push(px); t2 = time.perf_counter()
    print(f"python push {1e3*(t2-t1):.3f}")
os.environ["CYC_TRACE"] = "1"
