"""Is the device-resident C2 step host-bound?  Host enqueue time per step vs
the device time per step (events), 50 steps (diagnostics)."""
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
out = torch.empty((1, 2, 65536), dtype=torch.complex128, device="cuda")
def step():
    est.reset(); est.push_device(dx.data_ptr(), L); est.average_all(out=out)
for _ in range(10): step()
torch.cuda.synchronize()
K = 50
PROF = int(os.environ.get("HB_PROF", "0"))
if PROF:
    est.profile(True)
for trial in range(3):
    hs = [0.0, 0.0, 0.0]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(); t0 = time.perf_counter()
    for _ in range(K):
        a = time.perf_counter(); est.reset(); b = time.perf_counter()
        est.push_device(dx.data_ptr(), L); c = time.perf_counter()
        est.average_all(out=out); d = time.perf_counter()
        hs[0] += b - a; hs[1] += c - b; hs[2] += d - c
    t1 = time.perf_counter(); e1.record(); torch.cuda.synchronize()
    print(f"host enqueue {1e6*(t1-t0)/K:.1f} us/step (reset {1e6*hs[0]/K:.1f}, push {1e6*hs[1]/K:.1f}, "
          f"avg {1e6*hs[2]/K:.1f}); device {1e3*e0.elapsed_time(e1)/K:.1f} us/step", flush=True)
if PROF:
    print(est.profile_read_ex())
