"""Pipeline trace of the planes fold (fold_tcp_kernel, CTA 0 of the last
launch; -DTC_TRACE build under _diag/, loaded with CYC_LIB) -- diagnostics.
C5 geometry on random data: per stage the producer's issue time, the MMA
warp's full-barrier completion, drain wait and MMA issue end."""
import ctypes as C
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_16911_b200 as cyc
L = 1 << 26
rng = np.random.default_rng(0)
x = (rng.standard_normal(L, dtype=np.float32) + 1j * rng.standard_normal(L, dtype=np.float32)).astype(np.complex64)
est = cyc.CyclicCorrelator(cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=8192,
                                               lag_spec=cyc.LagSpec.Explicit(range(256)),
                                               flags=cyc.Flags.BOTH, emit_frames=False))
dx = torch.from_numpy(x.view(np.float32)).cuda()
for _ in range(3):
    est.reset(); est.push_device(dx.data_ptr(), L); est.average(flag=1)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (8 * 128))()
assert cyc.lib().cyc_debug_tc_trace(buf) == 0
t = np.array(buf, dtype=np.int64).reshape(8, 128)
t0 = t[7, 0]
n = int(np.count_nonzero(t[2]))
print(f"stages traced {n}")
print("stage   issue  fullseen  mma_go  mma_end")
for i in range(min(n, 128)):
    print(f"{i:5d} " + " ".join(f"{(t[k, i] - t0):8d}" for k in (0, 3, 1, 2)))
iv = np.diff(t[1, :n])
print("mma_go interval mean", iv[5:].mean(), "median", np.median(iv[5:]))
print("issue->fullseen mean", (t[3, :n] - t[0, :n])[5:].mean())
print("fullseen->mma_go (drain waits) mean", (t[1, :n] - t[3, :n])[5:].mean())
print("mma issue time mean", (t[2, :n] - t[1, :n])[5:].mean())
print("issue interval mean", np.diff(t[0, :n])[5:].mean())
for name, b in (("CTA 0", 100), ("last CTA", 110)):
    c0, g0, c1, g1 = (int(t[6, b + k]) for k in range(4))
    if g1 > g0:
        print(f"{name}: {c1 - c0} cycles in {(g1 - g0) / 1e3:.1f} us -> SM clock {(c1 - c0) / (g1 - g0):.3f} GHz")
print("kernel span (CTA 0 start -> last CTA end) us", (int(t[6, 113]) - int(t[6, 101])) / 1e3)
