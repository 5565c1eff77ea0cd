import os, sys
import numpy as np
sys.path.insert(0, "/root/repo")
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
px = cyc.host_alloc(x.shape); px[:] = x
oh = cyc.host_alloc((1, 2, 65536), dtype=np.complex128)
def step():
    est.reset(); est.push_device(dx.data_ptr(), L); est.average_all(out=out)
def e2e():
    est.reset(); est.push(px); est.average_all(out=oh)
for _ in range(5): step(); step(); e2e()
for trial in range(3):
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
    ev[0].record()
    for i in range(10):
        step(); ev[i + 1].record()
    torch.cuda.synchronize()
    print([round(1e3 * ev[i].elapsed_time(ev[i + 1]), 1) for i in range(10)], flush=True)
    e2e()
