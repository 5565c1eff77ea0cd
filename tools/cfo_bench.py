"""estimate_cfo_ccf: device vs the reference (oracle/_ref) wall time (diagnostics)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2405_16911_b200 as cyc
from oracle.oracle import RefLib
os.environ.setdefault("OMP_WAIT_POLICY", "passive")
N, FRAMES, BETA = 4096, 16, 0.25
rng = np.random.default_rng(3)
n = N * FRAMES + 64
t = np.arange(n)
sym = rng.choice([-1, 1], size=n // 8 + 1).repeat(8)[:n]
x = (sym * np.exp(1j * np.pi * 0.5 * t / 8) * np.exp(2j * np.pi * 0.003 * t)).astype(np.complex64)
ref = RefLib()
cyc.estimate_cfo_ccf(x, BETA, N, FRAMES)
for _ in range(2):
    a = time.perf_counter(); e = cyc.estimate_cfo_ccf(x, BETA, N, FRAMES); b = time.perf_counter()
    r = ref.estimate_cfo_ccf(x.astype(np.complex128), BETA, N, FRAMES); c = time.perf_counter()
    print(f"gpu {1e3*(b-a):.2f} ms  ref {1e3*(c-b):.2f} ms  eps {e:.9f} ref {r:.9f}")
