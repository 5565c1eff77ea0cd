"""A/B the fold kernel of two libcycb200 builds through the same driver (CYC_LIB)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_16911_b200 as cyc
L = 1 << 24
rng = np.random.default_rng(0)
x = (rng.standard_normal(L) + 1j * rng.standard_normal(L)).astype(np.complex64)
cfg = cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=1024, lag_spec=cyc.LagSpec.Explicit(range(64)),
                          flags=cyc.Flags.BOTH, emit_frames=False)
est = cyc.CyclicCorrelator(cfg)
dx = torch.from_numpy(x.view(np.float32)).cuda()
for _ in range(3):
    est.reset(); est.push_device(dx.data_ptr(), L); est.average(flag=1)
est.profile(True)
n0, ms0, _ = est.profile_read()
for _ in range(20):
    est.reset(); est.push_device(dx.data_ptr(), L); est.average(flag=1)
n1, ms1, _ = est.profile_read()
print(os.environ.get("CYC_LIB", "new"), "fold ms/launch %.4f launches %d" % ((ms1 - ms0) / (n1 - n0), n1 - n0))
