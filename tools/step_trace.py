"""Host timeline of device-resident C2 steps (CYC_TRACE=1; diagnostics)."""
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
for i in range(6):
    t0 = time.perf_counter()
    est.reset(); t1 = time.perf_counter()
    est.push_device(dx.data_ptr(), L); t2 = time.perf_counter()
    est.average_all(out=out); t3 = time.perf_counter()
    print(f"---- step {i}: reset {1e6*(t1-t0):.0f} us, push {1e6*(t2-t1):.0f} us, avg {1e6*(t3-t2):.0f} us", flush=True)
