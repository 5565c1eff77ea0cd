"""Generate tests/golden/reference_golden.npz from the REFERENCE itself.

Run in the container that has /root/reference (oracle/_ref/libcycstat_ref.so,
built by oracle/Makefile from the reference's own sources):

    python tests/golden/make_golden.py

Every array is an output of the unmodified reference library (CyclicCorrelator
push, compute windows, cyclic_xcorr_direct, Fft, validate_config, average
frames) on small seeded inputs, so the CPU oracle and the GPU path can be
pinned against it on machines where the reference is absent (the GPU box).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import RefLib  # noqa: E402


def rand_c(n, seed):
    rng = np.random.default_rng(seed)
    return (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(np.complex64).astype(np.complex128)


def main():
    r = RefLib()
    g = {}
    # frozen literal-sum vector (proj/tests/test_reference.cpp:21-24)
    fz = np.array([1, 1j, -1 + 0.5j, 2 - 1j, 1 + 1j, -1j, 0.5, -1 - 1j])
    g["frozen_x"] = fz
    g["frozen_vals"] = np.array([r.direct(fz, fz, 0.25, 1, 0, 1, 4), r.direct(fz, fz, 0.25, 1, 1, 1, 4),
                                 r.direct(fz, fz, 0.11, -1, 0, 2, 4)])
    # Set-mode streams (test_estimator.cpp:211-229 geometry), x != y, both flags
    x, y = rand_c(400, 1234), rand_c(400, 4321)
    g["set_x"], g["set_y"] = x, y
    g["set_alphas"] = np.array([3 / 64, 0.0, -0.21])
    for conj in (0, 1):
        fr, st = r.stream(0, conj, 64, x, y, alphas=g["set_alphas"], max_lag=3, chunk=37)
        g[f"set_frames_conj{conj}"], g[f"set_start_conj{conj}"] = fr, st
    # Full-mode streams (test_estimator.cpp:242-272), lags {-3, 0, 5}
    x, y = rand_c(300, 777), rand_c(300, 888)
    g["full_x"], g["full_y"] = x, y
    for conj in (0, 1):
        fr, st = r.stream(1, conj, 64, x, y, lags=[-3, 0, 5], chunk=0)
        g[f"full_frames_conj{conj}"], g[f"full_start_conj{conj}"] = fr, st
    # coherent block average (average_frames over N-sized pushes), Full N=256 lags 0..7
    xb = rand_c(1 << 13, 5).astype(np.complex64)
    g["block_x"] = xb
    for conj in (0, 1):
        avg, F = r.block_average(1, conj, 256, xb, xb, lags=list(range(8)))
        g[f"block_avg_conj{conj}"], g["block_frames"] = avg, np.array(F)
    # FFT: radix-2 and the direct non-pow2 fallback (proj/src/fft.cpp)
    v = rand_c(100, 9)
    g["fft_in"], g["fft64"], g["fft100"] = v, r.fft(v[:64]), r.fft(v)
    # tone identities through the streaming estimator (test_estimator.cpp:81-105)
    t = r.tone(0.125, 0.0, 256)
    g["tone"] = t
    g["tone_frames"], _ = r.stream(0, 0, 64, t, t, alphas=[0.0], max_lag=2)
    # GMSK generator (cpm_modulate, BT 0.3, 8 sps) -- harness input reference
    g["gmsk_2048"] = r.gmsk(2048, 0.3, 8, 7)
    # validate_config messages (proj/src/types.cpp:30-63)
    cases = [
        dict(mode=0, win_len=8, alphas=[], lag_symmetric=True, max_lag=2),
        dict(mode=0, win_len=1, alphas=[0.1], lag_symmetric=False, lags=[0, 1]),
        dict(mode=1, win_len=8, lag_symmetric=True, max_lag=1),
        dict(mode=1, win_len=8, lag_symmetric=False, lags=[]),
        dict(mode=1, win_len=8, lag_symmetric=False, lags=[2, 1], alphas=[0.7]),
        dict(mode=0, win_len=16, alphas=[0.125], lag_symmetric=True, max_lag=8),
        dict(mode=0, win_len=4096, alphas=[0.125], lag_symmetric=True, max_lag=256),
    ]
    msgs = []
    for c in cases:
        msgs.append("\n".join(r.validate(c["mode"], c["win_len"], alphas=c.get("alphas", []),
                                         lag_symmetric=c["lag_symmetric"], max_lag=c.get("max_lag", 0),
                                         lags=c.get("lags", []))))
    g["validate_cases"] = np.array([repr(c) for c in cases])
    g["validate_msgs"] = np.array(msgs)
    out = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(out, **g)
    print(out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
