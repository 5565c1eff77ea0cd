"""FP32 rest (head/tail periods) vs numpy when the TC part is planned but not launched (diagnostics)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
os.environ["CYC_TC_DRYRUN"] = "1"
import torch
import paper_2405_16911_b200 as cyc
from paper_2405_16911_b200.shard import DeviceArray
from conftest import rand_c
L0, L1 = int(os.environ.get("L0", -16)), int(os.environ.get("L1", 16))
lags = list(range(L0, L1))
Pf = 1024
x = rand_c(Pf * 60, 31)
d = torch.from_numpy(x).cuda()
est = cyc.CyclicCorrelator(cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=Pf, lag_spec=cyc.LagSpec.Explicit(lags),
                           emit_frames=False))
est.push_device(d.data_ptr(), len(x))
p, n, _ = est.fold_state()
S = torch.as_tensor(DeviceArray(p, n), device="cuda").cpu().numpy()
tp = S.size // (Pf * 4)
S = S.reshape(tp, Pf, 4)
f_lo = L0 - (L0 % 4)
xr, xi = x.real.astype(np.float64), x.imag.astype(np.float64)
m_minus = max(0, -L0)
F = est.frames_emitted()
n_start, n_end = m_minus, m_minus + F * Pf
nlb = (tp + 63) // 64
pa = max(-(-n_start // Pf), -(-(0 - f_lo) // Pf))
pb = min(n_end // Pf, (len(x) - Pf - f_lo - 64 * nlb) // Pf + 1)
ranges = [(n_start, min(n_end, pa * Pf)), (max(n_start, pb * Pf), n_end)]
print("rest ranges", ranges)
E = np.zeros_like(S)
for t in range(tp):
    lag = f_lo + t
    for a, b in ranges:
        if b <= a: continue
        nn = np.arange(a, b)
        xs = nn + lag
        ok = (xs >= 0) & (xs < len(x))
        r = nn % Pf
        xr_ = np.where(ok, xr[np.clip(xs, 0, len(x) - 1)], 0); xi_ = np.where(ok, xi[np.clip(xs, 0, len(x) - 1)], 0)
        np.add.at(E[t, :, 0], r, xr_ * xr[nn]); np.add.at(E[t, :, 1], r, xi_ * xr[nn])
        np.add.at(E[t, :, 2], r, xr_ * xi[nn]); np.add.at(E[t, :, 3], r, xi_ * xi[nn])
err = np.abs(S - E).max() / max(np.abs(E).max(), 1e-30)
print("FP32-rest vs numpy: max rel", err, "max|E|", np.abs(E).max(), "max|S|", np.abs(S).max())
if err > 1e-4:
    bad = np.argwhere(np.abs(S - E).max(axis=2) > 1e-4 * np.abs(E).max())
    print("bad cells", len(bad), "lags", np.unique(bad[:, 0])[:10], "res", np.unique(bad[:, 1])[:20])
