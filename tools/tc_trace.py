"""Pipeline trace of the tensor-core fold (CTA 0): run on a -DTC_TRACE build
(CYC_NVCC_EXTRA=-DTC_TRACE build under _diag/, loaded with CYC_LIB) -- diagnostics only."""
import ctypes as C
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_16911_b200 as cyc
# TRACE_CFG=c5: Pf = 8192, lags 0..255 (the trace keeps the last launch's CTA 0: a non-self lag block)
c5 = os.environ.get("TRACE_CFG") == "c5"
L = 1 << (26 if c5 else 24)
rng = np.random.default_rng(0)
x = (rng.standard_normal(L) + 1j * rng.standard_normal(L)).astype(np.complex64)
cfg = cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=8192 if c5 else 1024,
                          lag_spec=cyc.LagSpec.Explicit(range(256 if c5 else 64)),
                          flags=cyc.Flags.BOTH, emit_frames=False)
est = cyc.CyclicCorrelator(cfg)
dx = torch.from_numpy(x.view(np.float32)).cuda()
for _ in range(3):
    est.reset(); est.push_device(dx.data_ptr(), L); est.average(flag=1)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (8 * 128))()
assert cyc.lib().cyc_debug_tc_trace(buf) == 0
t = np.array(buf, dtype=np.int64).reshape(8, 128)
t0 = t[7, 0]
names = ["issue", "mma_go", "mma_done", "cv_full", "cv_pfree", "cv_done"]
n = int(np.count_nonzero(t[1]))
print(f"kernel: {(t[7,1]-t0)} cycles; epilogue starts {t[6,0]-t0}; stages {n}")
print("stage " + " ".join(f"{k:>9s}" for k in names))
for i in range(n):
    print(f"{i:5d} " + " ".join(f"{(t[k, i] - t0 if t[k, i] else -1):9d}" for k in range(6)))
d = np.diff(t[1, :n])
print("mma_go interval mean", d[5:].mean(), "converter full->done mean", (t[5, :n] - t[4, :n])[5:].mean(),
      "pfree wait mean", (t[4, :n] - t[3, :n])[5:].mean(), "tma issue->full mean", (t[3, :n] - t[0, :n])[5:].mean(),
      "issue interval mean", np.diff(t[0, :n])[5:].mean())

w = (C.c_ulonglong * (16 * 64 * 2))()
assert cyc.lib().cyc_debug_tc_warps(w) == 0
w = np.array(w, dtype=np.int64).reshape(16, 64, 2)
print("per converter warp (stage 20..23): full-seen / conv-arrive, cycles from kernel start")
for it in range(20, 24):
    print(it, "full", [int(w[k, it, 0] - t0) for k in range(2, 14)])
    print(it, "done", [int(w[k, it, 1] - t0) for k in range(2, 14)], "mma_go", int(t[1, it] - t0))
