"""Where does cyc_average's time go (diagnostics): D2H of one table vs the rest."""
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
o1 = np.zeros(65536, np.complex128); o2 = np.zeros(65536, np.complex128)
for rep in range(6):
    est.reset(); est.push_device(dx.data_ptr(), L); torch.cuda.synchronize()
    t0 = time.perf_counter(); est.average(flag=1, out=o1); t1 = time.perf_counter()
    est.average(flag=2, out=o2); t2 = time.perf_counter()
    print(f"avg1 {1e3*(t1-t0):.3f} avg2 {1e3*(t2-t1):.3f} ms", flush=True)
# raw D2H of 1 MiB into pinned / pageable
dev = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
pin = torch.empty(1 << 20, dtype=torch.uint8).pin_memory()
pg = torch.empty(1 << 20, dtype=torch.uint8)
for name, dst in (("pinned", pin), ("pageable", pg)):
    for rep in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter(); dst.copy_(dev); torch.cuda.synchronize()
        print(f"D2H 1 MiB {name}: {1e6*(time.perf_counter()-t0):.1f} us", flush=True)
a = np.empty(1 << 17); b = np.ones(1 << 17)
for rep in range(3):
    t0 = time.perf_counter(); a[:] = b; print(f"host memcpy 1 MiB {1e6*(time.perf_counter()-t0):.1f} us")
