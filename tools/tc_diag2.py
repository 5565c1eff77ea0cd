"""TC vs FP32 fold, Full-mode block averages over lag sets / window sizes (diagnostics)."""
import os, sys, subprocess, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
import paper_2405_16911_b200 as cyc
from conftest import rand_c
cases = [(1024, list(range(64))), (1024, list(range(32))), (1024, list(range(-16, 16))), (1024, list(range(-32, 32))),
         (1280, list(range(64))), (1024, list(range(8, 72)))]
x = rand_c(1024 * 200, 31)
d = torch.from_numpy(x).cuda()
if os.environ.get("CHILD"):
    res = {}
    for i, (N, lags) in enumerate(cases):
        est = cyc.CyclicCorrelator(cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=N, lag_spec=cyc.LagSpec.Explicit(lags),
                                   emit_frames=False))
        est.push_device(d.data_ptr(), len(x))
        np.save(f"/tmp/tcd2_{os.environ['CHILD']}_{i}.npy", est.average())
    sys.exit(0)
for tag, env in (("tc", {}), ("fp32", {"CYC_NO_TC": "1"})):
    subprocess.run([sys.executable, __file__], env={**os.environ, **env, "CHILD": tag}, check=True)
for i, (N, lags) in enumerate(cases):
    a, b = np.load(f"/tmp/tcd2_tc_{i}.npy"), np.load(f"/tmp/tcd2_fp32_{i}.npy")
    print(N, lags[0], lags[-1], "rel diff %.3e" % (np.linalg.norm(a - b) / np.linalg.norm(b)))
for i in (2, 3):
    N, lags = cases[i]
    a = np.load(f"/tmp/tcd2_tc_{i}.npy").reshape(len(lags), N)
    b = np.load(f"/tmp/tcd2_fp32_{i}.npy").reshape(len(lags), N)
    e = np.linalg.norm(a - b, axis=1) / np.linalg.norm(b, axis=1)
    print("case", i, "per-lag rel err:", " ".join(f"{l}:{v:.0e}" for l, v in zip(lags, e)))
