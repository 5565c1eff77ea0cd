"""Monte-Carlo oracle: device vs the reference (oracle/_ref) on the acceptance
table's geometry (proj/tests/acceptance_main.cpp:330: 32 trials, N = 4096,
lags -16..16, alpha 1/8) and a larger one; prints JSON lines (diagnostics)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2405_16911_b200 as cyc
from oracle.oracle import RefLib, have_ref
lags = list(range(-16, 17))
cases = [("acceptance", [0.125], 32, 4096, 2 * 4096 + 32), ("wide", [k / 64 for k in range(-32, 32)], 64, 4096, 16 * 4096 + 32)]
for name, alphas, trials, n, rec in cases:
    cyc.gmsk_mc_oracle(None, alphas, lags, False, n, 1, rec, 1)  # warm
    t0 = time.perf_counter(); g = cyc.gmsk_mc_oracle(None, alphas, lags, False, n, trials, rec, 9001); tg = time.perf_counter() - t0
    line = {"case": name, "alphas": len(alphas), "lags": len(lags), "trials": trials, "win_len": n, "record_len": rec,
            "gpu_s": tg}
    if have_ref() and (name == "acceptance" or os.environ.get("REF_ALL")):
        os.environ.setdefault("OMP_WAIT_POLICY", "passive")
        t0 = time.perf_counter(); w = RefLib().gmsk_mc_oracle(alphas, lags, False, n, trials, rec, 9001); tr = time.perf_counter() - t0
        line.update({"ref_s": tr, "speedup": tr / tg, "max_abs_diff": float(np.max(np.abs(g.mean_magnitude - w.reshape(-1))))})
    print(json.dumps(line), flush=True)
