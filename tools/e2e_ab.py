"""e2e C2 step timing only (A/B of env knobs; diagnostics)."""
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
px = cyc.host_alloc(x.shape); px[:] = x
out = cyc.host_alloc((1, 2, 65536), dtype=np.complex128)
st = torch.cuda.ExternalStream(est.stream())
def step():
    est.reset(); est.push(px); est.average_all(out=out)
for _ in range(3): step()
ts = []
for _ in range(5):
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(10): step()
    e1.record(st); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) / 10)
print(os.environ.get("TAG", ""), "e2e ms/step", " ".join(f"{t:.3f}" for t in ts), "min", f"{min(ts):.3f}")
