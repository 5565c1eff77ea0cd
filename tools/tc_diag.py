"""TC vs FP32 fold on a Set-mode block average (diagnostics)."""
import os, sys, subprocess
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
import paper_2405_16911_b200 as cyc
from conftest import rand_c
x = rand_c(40_000, 31)
M, N = int(os.environ.get("M", 15)), 4096
alphas = [0.1 + k / 16 for k in range(-2, 3)]
def run(kind):
    est = cyc.CyclicCorrelator(cyc.EstimatorConfig(mode=cyc.Mode.Set, win_len=N, alphas=alphas,
                               lag_spec=cyc.LagSpec.Symmetric(M), emit_frames=False))
    if kind == "host":
        est.push(x)
    else:
        d = torch.from_numpy(x).cuda()
        est.push_device(d.data_ptr(), len(x))
    return est.average(), est.algorithm()
if os.environ.get("CHILD"):
    for k in ("host", "device"):
        a, alg = run(k)
        np.save(f"/tmp/tcd_{os.environ['CHILD']}_{k}.npy", a)
        print(os.environ["CHILD"], k, alg)
    sys.exit(0)
for tag, env in (("tc", {}), ("fp32", {"CYC_NO_TC": "1"})):
    subprocess.run([sys.executable, __file__], env={**os.environ, **env, "CHILD": tag}, check=True)
ref = np.load("/tmp/tcd_fp32_host.npy")
for tag in ("tc_host", "tc_device", "fp32_device"):
    a = np.load(f"/tmp/tcd_{tag}.npy")
    print(tag, "rel diff vs fp32 host %.3e" % (np.linalg.norm(a - ref) / np.linalg.norm(ref)))
