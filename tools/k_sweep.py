import os, sys, time, threading
import numpy as np
sys.path.insert(0, "/root/repo")
import torch
import paper_2405_16911_b200 as cyc
from paper_2405_16911_b200 import siggen
import bench
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
def timed(k, clocks):
    torch.cuda.synchronize()
    c = bench.Clocks(0) if clocks else None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): step()
    e1.record(); torch.cuda.synchronize()
    if c: c.stop()
    return 1e3 * e0.elapsed_time(e1) / k
for k in (3, 10, 20, 50):
    print(k, "no-clk", [round(timed(k, False), 1) for _ in range(3)], "clk", [round(timed(k, True), 1) for _ in range(3)], flush=True)
