import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2405_16911_b200 as cyc
N, FRAMES = 4096, 16
x = (np.random.default_rng(1).standard_normal(N*FRAMES) + 0j).astype(np.complex64)
cfg = cyc.EstimatorConfig(mode=cyc.Mode.Full, conj=True, win_len=N, lag_spec=cyc.LagSpec.Explicit([0]))
for rep in range(3):
    a = time.perf_counter(); est = cyc.CyclicCorrelator(cfg); b = time.perf_counter()
    est.push(x); c = time.perf_counter()
    m = est.average(mode=cyc.AverageMode.Magnitude); d = time.perf_counter()
    est.close(); e = time.perf_counter()
    print(f"create {1e3*(b-a):.1f} push {1e3*(c-b):.1f} avg {1e3*(d-c):.1f} destroy {1e3*(e-d):.1f} ms", est and "", flush=True)
