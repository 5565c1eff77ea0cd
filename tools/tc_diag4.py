"""TC-only S (interior periods) vs numpy (diagnostics)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
import paper_2405_16911_b200 as cyc
from paper_2405_16911_b200.shard import DeviceArray
from conftest import rand_c
os.environ["CYC_TC_SKIP_REST"] = "1"
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
f_lo = L0 - (L0 % 4)  # engine rounding (multiple of 4 when free)
print("t_pad", tp, "f_lo guess", f_lo)
xr, xi = x.real.astype(np.float64), x.imag.astype(np.float64)
# interior periods: find which periods TC covered by trying ranges
m_minus = max(0, -L0)
F = est.frames_emitted()
n_start, n_end = m_minus, m_minus + F * Pf
pa = max(-(-n_start // Pf), -(-(0 - f_lo) // Pf))
nlb = (tp + 63) // 64
pb = min(n_end // Pf, (len(x) - Pf - f_lo - 64 * nlb) // Pf + 1)
print("pa pb", pa, pb)
E = np.zeros_like(S)
for t in range(tp):
    lag = f_lo + t
    for p_ in range(pa, pb):
        n0 = p_ * Pf
        nn = np.arange(n0, n0 + Pf)
        xs = nn + lag
        ok = (xs >= 0) & (xs < len(x))
        yr_, yi_ = xr[nn], xi[nn]
        xr_ = np.where(ok, xr[np.clip(xs, 0, len(x) - 1)], 0); xi_ = np.where(ok, xi[np.clip(xs, 0, len(x) - 1)], 0)
        E[t, :, 0] += xr_ * yr_; E[t, :, 1] += xi_ * yr_; E[t, :, 2] += xr_ * yi_; E[t, :, 3] += xi_ * yi_
err = np.abs(S - E).max() / np.abs(E).max()
print("TC-only vs numpy interior: max rel", err)
if err > 1e-4:
    for t in (0, 1, tp // 2, tp - 1):
        e = np.abs(S[t] - E[t]).max(axis=1)
        print("lag idx", t, "worst residues", np.argsort(-e)[:8], e.max())
