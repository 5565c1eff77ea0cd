"""Device timeline of device-resident C2 steps (CYC_TIMELINE=1): mean offset of
each named point from the step's reset, over 40 steps (diagnostics)."""
import os, sys
os.environ["CYC_TIMELINE"] = "1"
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
for _ in range(40):
    est.reset(); est.push_device(dx.data_ptr(), L); est.average_all(out=out)
est.reset()
torch.cuda.synchronize()
del est
