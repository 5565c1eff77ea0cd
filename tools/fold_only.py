"""Run the C2 device-resident step a few times (for ncu captures of fold_kernel)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_16911_b200 as cyc
L = 1 << 24
rng = np.random.default_rng(0)
x = (rng.standard_normal(L) + 1j * rng.standard_normal(L)).astype(np.complex64)
lags = int(os.environ.get("LAGS", "64")); N = int(os.environ.get("NWIN", "1024"))
cfg = cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=N, lag_spec=cyc.LagSpec.Explicit(range(lags)),
                          flags=cyc.Flags.BOTH, emit_frames=False)
est = cyc.CyclicCorrelator(cfg)
dx = torch.from_numpy(x.view(np.float32)).cuda()
for _ in range(int(os.environ.get("REPS", "3"))):
    est.reset(); est.push_device(dx.data_ptr(), L); est.average(flag=1)
torch.cuda.synchronize()
print("ok", est.algorithm())
