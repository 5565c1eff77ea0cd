"""Per-phase wall-clock breakdown of one C2 step (diagnostics, not a bench)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_16911_b200 as cyc
from paper_2405_16911_b200 import siggen

L = 1 << 24
x = siggen.c2_record(n=L)
cfg = cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=1024, lag_spec=cyc.LagSpec.Explicit(range(64)),
                          flags=cyc.Flags.BOTH, emit_frames=False)
est = cyc.CyclicCorrelator(cfg)
dx = torch.from_numpy(x.view(np.float32)).cuda()
px = cyc.host_alloc(x.shape); px[:] = x
def t(fn, *a, **k):
    t0 = time.perf_counter(); r = fn(*a, **k); torch.cuda.synchronize(); return r, (time.perf_counter() - t0) * 1e3
for rep in range(4):
    _, tr = t(est.reset)
    _, tp = t(est.push_device, dx.data_ptr(), L)
    _, ta = t(est.average, flag=1)
    _, tb = t(est.average, flag=2)
    print(f"device: reset {tr:.3f} push_device {tp:.3f} avg1 {ta:.3f} avg2 {tb:.3f} ms")
for rep in range(3):
    _, tr = t(est.reset)
    _, tp = t(est.push, px)
    _, ta = t(est.average, flag=1)
    print(f"e2e pinned: reset {tr:.3f} push {tp:.3f} avg {ta:.3f} ms")
for rep in range(2):
    _, tr = t(est.reset)
    _, tp = t(est.push, x)
    print(f"e2e pageable: push {tp:.3f} ms")
