"""C1 call pattern (Set N=4096, Symmetric(15), 10 alphas, 4096-sample pushes) for
a short ncu launch list (diagnostics)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_16911_b200 as cyc
C1_CONV = [k / 8 for k in range(-2, 3)]
C1_CONJ = [0.1 + k / 16 for k in range(-2, 3)]
est = cyc.CyclicCorrelator(cyc.EstimatorConfig(mode=cyc.Mode.Set, win_len=4096, alphas=C1_CONV + C1_CONJ,
                                               lag_spec=cyc.LagSpec.Symmetric(15), flags=cyc.Flags.BOTH))
rng = np.random.default_rng(1)
x = (rng.standard_normal(64 * 4096) + 1j * rng.standard_normal(64 * 4096)).astype(np.complex64)
px = cyc.host_alloc(x.shape)
px[:] = x
for off in range(0, len(x), 4096):
    est.push(px[off:off + 4096])
print("ok", est.algorithm(), est.frames_emitted())
