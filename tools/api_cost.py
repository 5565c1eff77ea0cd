"""Host cost of the public calls of a C2 device step (diagnostics)."""
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
for _ in range(6):
    est.reset(); est.push_device(dx.data_ptr(), L); est.average_all(out=out)
torch.cuda.synchronize()
def t(fn, k=200):
    torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(k): fn()
    b = time.perf_counter()
    torch.cuda.synchronize()
    return 1e6 * (b - a) / k
L_ = cyc.lib()
h = est._h
print("consumed()", t(est.consumed))
print("raw cyc_consumed", t(lambda: L_.cyc_consumed(h)))
print("average_all(out)", t(lambda: est.average_all(out=out)))
print("raw cyc_average_all", t(lambda: L_.cyc_average_all(h, 0, out.data_ptr())))
print("reset()", t(est.reset))
