"""Fold kernel timing (diagnostics): device-resident block steps of C2 and C5
(or the configs named in argv), CUDA events around every fold launch.
Prints one JSON line per config: fold ms per launch and per step, step ms."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_16911_b200 as cyc

GEO = {"c2": (1 << 24, 1024, 64, 1), "c5": (1 << 26, 8192, 256, 1), "c4": (1 << 22, 256, 32, 64)}
for name in (sys.argv[1:] or ["c2", "c5"]):
    L, N, T, C_ = GEO[name]
    rng = np.random.default_rng(0)
    x = (rng.standard_normal((C_, L), dtype=np.float32) + 1j * rng.standard_normal((C_, L), dtype=np.float32))
    x = x.astype(np.complex64)
    est = cyc.CyclicCorrelator(cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=N, lag_spec=cyc.LagSpec.Explicit(range(T)),
                                                   flags=cyc.Flags.BOTH, emit_frames=False, channels=C_))
    d = torch.from_numpy(x.view(np.float32)).cuda()
    out = torch.empty((C_, 2, T * N), dtype=torch.complex128, device="cuda")

    def step():
        est.reset(); est.push_device(d.data_ptr(), L); est.average_all(out=out)
    for _ in range(4):
        step()
    torch.cuda.synchronize()
    K = 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        step()
    e1.record(); torch.cuda.synchronize()
    ms_step = e0.elapsed_time(e1) / K
    est.profile(True)
    for _ in range(4):
        step()
    p0 = est.profile_read_ex()
    for _ in range(K):
        step()
    torch.cuda.synchronize()
    p1 = est.profile_read_ex()
    est.profile(False)
    n = p1["launches"] - p0["launches"]
    ms = (p1["ms"] - p0["ms"])
    print(json.dumps({"cfg": name, "extra": os.environ.get("CYC_NVCC_EXTRA", ""), "ms_step": ms_step,
                      "fold_ms_per_step": ms / K, "fold_launches_per_step": n / K,
                      "fold_ms_per_launch": ms / max(n, 1), "tensor_launches": p1["tensor_launches"] - p0["tensor_launches"]}),
          flush=True)
