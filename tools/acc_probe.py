"""Accuracy probe (diagnostics): worst-cell error / mean power and relative L2 of
the device block fold against the fp64 oracle at a BASELINE geometry.
    python tools/acc_probe.py c5|c2|c4   (env knobs such as CYC_TC_MAXP apply)"""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_16911_b200 as cyc
from paper_2405_16911_b200 import siggen
from oracle.oracle import Oracle

name = sys.argv[1]
o = Oracle()
if name == "c5":
    x, N, T = siggen.c5_record(n=1 << 26)[None], 8192, 256
elif name == "c2":
    x, N, T = siggen.c2_record(n=1 << 24)[None], 1024, 64
else:
    x, N, T = np.stack([siggen.c4_channel(c, n=1 << 22) for c in range(0, 64)]), 256, 32
C_ = x.shape[0]
est = cyc.CyclicCorrelator(cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=N, lag_spec=cyc.LagSpec.Explicit(range(T)),
                                               flags=cyc.Flags.BOTH, emit_frames=False, channels=C_))
d = torch.from_numpy(np.ascontiguousarray(x).view(np.float32)).cuda()
est.push_device(d.data_ptr(), x.shape[-1])
got = est.average_all()
F = est.frames_emitted()
rng = np.random.default_rng(1)
bins = np.unique(np.concatenate([[0, 1, N - 1], rng.choice(N, min(N, 61), replace=False)]))
res = []
for c in range(C_):
    cv, cj = o.block_fold(x[c], x[c], bins, N, list(range(T)), 0, F * N)
    mp = float(np.mean(np.abs(x[c].astype(np.complex128)) ** 2))
    for fi, w in ((0, cv), (1, cj)):
        g = got[c, fi].reshape(T, N)[:, bins]
        e = np.abs(g - w.T)
        i = np.unravel_index(np.argmax(e), e.shape)
        res.append({"ch": c, "flag": fi, "max_over_mp": float(e.max() / mp),
                    "rel_l2": float(np.linalg.norm(g - w.T) / np.linalg.norm(w)),
                    "worst_lag": int(i[0]), "worst_bin": int(bins[i[1]]), "worst_rel": float(e.max() / abs(w.T[i]))})
worst = max(res, key=lambda r: r["max_over_mp"])
print(json.dumps({"cfg": name, "maxp": os.environ.get("CYC_TC_MAXP"), "algo": est.algorithm(), "worst": worst,
                  "max_rel_l2": max(r["rel_l2"] for r in res)}), flush=True)
