"""S-level diff TC vs FP32 fold for lags -16..15 (diagnostics)."""
import os, sys, subprocess
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
import paper_2405_16911_b200 as cyc
from paper_2405_16911_b200.shard import DeviceArray
from conftest import rand_c
lags = list(range(int(os.environ.get("L0", -16)), int(os.environ.get("L1", 16))))
x = rand_c(1024 * 60, 31)
d = torch.from_numpy(x).cuda()
if os.environ.get("CHILD"):
    est = cyc.CyclicCorrelator(cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=1024, lag_spec=cyc.LagSpec.Explicit(lags),
                               emit_frames=False))
    est.push_device(d.data_ptr(), len(x))
    p, n, _ = est.fold_state()
    S = torch.as_tensor(DeviceArray(p, n), device="cuda").cpu().numpy()
    np.save(f"/tmp/tcd3_{os.environ['CHILD']}.npy", S)
    sys.exit(0)
for tag, env in (("tc", {}), ("fp32", {"CYC_NO_TC": "1"})):
    subprocess.run([sys.executable, __file__], env={**os.environ, **env, "CHILD": tag}, check=True)
a, b = np.load("/tmp/tcd3_tc.npy"), np.load("/tmp/tcd3_fp32.npy")
tp = a.size // (1024 * 4)
a = a.reshape(tp, 1024, 4); b = b.reshape(tp, 1024, 4)
e = np.abs(a - b).max(axis=2)
scale = np.abs(b).max()
print("t_pad", tp, "max |dS| / max|S|", e.max() / scale)
bad = np.argwhere(e > 1e-3 * scale)
print("bad cells", len(bad), "of", e.size)
if len(bad):
    lg = np.unique(bad[:, 0]); rs = np.unique(bad[:, 1])
    print("lags idx", lg[:40], "...", len(lg))
    print("residues", rs[:64], "...", len(rs), "min", rs.min(), "max", rs.max())
    t, r = bad[0]
    print("example", t, r, a[t, r], b[t, r])
best = []
for dt in range(-20, 21):
    for dr in range(-40, 41):
        t0, t1 = max(0, -dt), min(tp, tp - dt)
        if t1 - t0 < 8: continue
        aa = a[t0:t1]
        bb = np.roll(b, -dr, axis=1)[t0 + dt:t1 + dt]
        err = np.abs(aa - bb).max() / scale
        best.append((err, dt, dr))
best.sort()
print("best shifts (err, dlag, dres):", best[:4])
