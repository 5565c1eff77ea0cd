"""Narrow (160-sample window) vs wide fused tensor-core fold on C4 channels
(diagnostics): run with CYC_TC_WIDE unset / set, save the tables, compare.
    python tools/narrow_check.py run <out.npy>
    python tools/narrow_check.py cmp <a.npy> <b.npy>"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if sys.argv[1] == "run":
    import torch
    import paper_2405_16911_b200 as cyc
    from paper_2405_16911_b200 import siggen
    C = 8
    xs = np.stack([siggen.c4_channel(c, n=1 << 22) for c in range(C)]).astype(np.complex64)
    est = cyc.CyclicCorrelator(cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=256,
                                                   lag_spec=cyc.LagSpec.Explicit(range(32)), flags=cyc.Flags.BOTH,
                                                   emit_frames=False, channels=C))
    d = torch.from_numpy(np.ascontiguousarray(xs).view(np.float32)).cuda()
    est.push_device(d.data_ptr(), xs.shape[-1])
    est.synchronize()
    t = est.average_all()  # [C, 2, 32 * 256]
    np.save(sys.argv[2], t)
    print("tensor launches", est.profile_read_ex().get("tensor_launches") if hasattr(est, "profile_read_ex") else "?")
else:
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    for c in range(a.shape[0]):
        for f in range(2):
            x, y = a[c, f].reshape(32, 256), b[c, f].reshape(32, 256)
            err = np.abs(x - y)
            rl2 = np.linalg.norm(x - y) / np.linalg.norm(y)
            lag, bn = np.unravel_index(np.argmax(err), err.shape)
            bylag = err.max(axis=1)
            print(f"ch {c} flag {f}: rel l2 {rl2:.2e} worst lag {lag} bin {bn}; lags with err > 1e-3 max: "
                  f"{np.nonzero(bylag > 1e-3 * err.max())[0][:12]}")
