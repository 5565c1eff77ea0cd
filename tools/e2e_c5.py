"""e2e C5 step timing only (pinned host record through cyc_push, every table to
pinned host; repeated rounds to show variance; diagnostics)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_16911_b200 as cyc
L = 1 << 26
rng = np.random.default_rng(0)
x = (rng.standard_normal(L, dtype=np.float32) + 1j * rng.standard_normal(L, dtype=np.float32)).astype(np.complex64)
cfg = cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=8192, lag_spec=cyc.LagSpec.Explicit(range(256)),
                          flags=cyc.Flags.BOTH, emit_frames=False)
est = cyc.CyclicCorrelator(cfg)
px = cyc.host_alloc(x.shape); px[:] = x
out = cyc.host_alloc((1, 2, 256 * 8192), dtype=np.complex128)
st = torch.cuda.ExternalStream(est.stream())
def step():
    est.reset(); est.push(px); est.average_all(out=out)
for _ in range(3): step()
ts = []
for _ in range(4):
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(5): step()
    e1.record(st); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) / 5)
print(os.environ.get("TAG", ""), "e2e ms/step", " ".join(f"{t:.3f}" for t in ts), "min", f"{min(ts):.3f}")
