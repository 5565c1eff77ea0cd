import numpy as np, sys, os, subprocess
sys.path.insert(0, "/root/repo")
from paper_2405_16911_b200 import siggen
x = siggen.gmsk(1 << 24, 0.3, 8, 0.02, 3).astype(np.complex64)
x.tofile("/tmp/c3.cf32")
x[:1 << 20].tofile("/tmp/c1.cf32")
