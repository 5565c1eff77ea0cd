"""Seeded random configurations against the fp64 oracle (oracle/cycoracle.c:
orc_stream restates CyclicCorrelator::push, proj/src/estimator.cpp:39-84).

Each case draws a mode (Set / Full), window, alpha set (on and off rational
grids), lag set, flag, input kind (pageable / pinned / device, auto or cross)
and chunking, then checks every emitted frame -- or, in block mode, the
coherent average -- at the north-star tolerance.  It sweeps the paths chosen
at plan and push time together (fold or direct, short-frame direct, tensor-core
fold with the fused finite check, CUDA-graph replays on the repeat pass).
"""
import numpy as np
import pytest

from conftest import assert_parity, mean_power, rand_c

pytestmark = pytest.mark.gpu


def draw_case(seed):
    r = np.random.default_rng(seed)
    full = bool(r.integers(0, 2))
    case = {"seed": seed, "full": full, "conj": bool(r.integers(0, 2)), "block": bool(r.integers(0, 2)),
            "cross": bool(r.integers(0, 2)), "kind": ["pageable", "pinned", "device"][int(r.integers(0, 3))]}
    if full:
        N = int(r.choice([64, 128, 256, 1024]))
        lo = int(r.integers(-8, 3))
        span = int(r.choice([1, 5, 16, 33, 64, 70]))
        lags = list(range(lo, lo + span))
        if r.integers(0, 3) == 0 and span > 4:  # an explicit, gappy lag set
            lags = sorted(set(int(v) for v in r.choice(lags, size=span // 2, replace=False)))
        case.update(N=N, lags=lags, alphas=[], max_lag=0)
    else:
        N = int(r.choice([200, 256, 1000, 2048, 4096]))
        A = int(r.integers(1, 7))
        P = int(r.choice([8, 16, 80, 1024]))
        alphas = [float(k) / P for k in r.integers(-P // 2, P // 2, size=A)]
        if r.integers(0, 3) == 0:
            alphas.append(float(r.uniform(-0.5, 0.5)))  # off any grid: the direct kernel
        case.update(N=N, alphas=alphas, max_lag=int(r.integers(0, min(20, N // 2 - 1))), lags=[])
    case["frames"] = int(r.integers(3, 24))
    case["chunks"] = int(r.integers(1, 5))
    return case


def draw_large(seed):
    """Full-mode block averages long enough for the tensor-core fold (>= 192 periods)."""
    r = np.random.default_rng(seed)
    N = int(r.choice([256, 512, 1024]))
    lo = int(r.choice([0, -32, -64, 4, -6]))
    span = int(r.choice([32, 64, 96, 128]))
    while N <= 2 * max(abs(lo), abs(lo + span - 1)):  # the span rule (types.cpp:30-63)
        N *= 2
    return {"seed": seed, "full": True, "conj": bool(r.integers(0, 2)), "block": True,
            "cross": bool(r.integers(0, 2)), "kind": ["pinned", "device"][int(r.integers(0, 2))], "N": N,
            "lags": list(range(lo, lo + span)), "alphas": [], "max_lag": 0, "frames": int(r.integers(200, 320)),
            "chunks": int(r.integers(1, 3))}


CASES = [draw_case(s) for s in range(24)] + [draw_large(100 + s) for s in range(8)]


@pytest.mark.parametrize("case", CASES, ids=[f"s{c['seed']}-{'full' if c['full'] else 'set'}-{c['kind']}"
                                             f"{'-block' if c['block'] else ''}" for c in CASES])
def test_random_config_against_oracle(cyc, oracle, case):
    import torch
    N, M = case["N"], case["max_lag"]
    lag_spec = cyc.LagSpec.Explicit(case["lags"]) if case["full"] else cyc.LagSpec.Symmetric(M)
    m_plus, m_minus = lag_spec.m_plus(), lag_spec.m_minus()
    n = case["frames"] * N + m_plus + m_minus + 17
    x = rand_c(n, 1000 + case["seed"])
    y = rand_c(n, 2000 + case["seed"]) if case["cross"] else x
    cfg = cyc.EstimatorConfig(mode=cyc.Mode.Full if case["full"] else cyc.Mode.Set, conj=case["conj"], win_len=N,
                              alphas=case["alphas"], lag_spec=lag_spec, emit_frames=not case["block"])
    want = oracle.stream(1 if case["full"] else 0, case["conj"], N, x.astype(complex), y.astype(complex),
                         alphas=case["alphas"], max_lag=M, lags=case["lags"])
    mp = np.sqrt(mean_power(x) * mean_power(y))
    est = cyc.CyclicCorrelator(cfg)
    cuts = np.linspace(0, n, case["chunks"] + 1).astype(int)
    if case["kind"] == "device":
        dx = torch.from_numpy(x).cuda()
        dy = torch.from_numpy(y).cuda() if case["cross"] else None
    for rep in range(2):  # the second pass replays captured push graphs where eligible
        est.reset()
        frames = []
        for a, b in zip(cuts[:-1], cuts[1:]):
            if case["kind"] == "device":
                frames += est.push_device(dx.data_ptr() + 8 * int(a), int(b - a),
                                          dy.data_ptr() + 8 * int(a) if dy is not None else None)
            elif case["kind"] == "pinned":
                px = cyc.host_alloc((int(b - a),))
                px[:] = x[a:b]
                if case["cross"]:
                    py = cyc.host_alloc((int(b - a),))
                    py[:] = y[a:b]
                    frames += est.push(px, py)
                else:
                    frames += est.push(px)
            else:
                frames += est.push(x[a:b], y[a:b] if case["cross"] else None)
        assert est.frames_emitted() == len(want)
        if case["block"]:
            assert_parity(est.average(), want.mean(axis=0), mp, what=f"{case} block average")
        else:
            got = np.array([f.values for f in frames])
            assert got.shape == want.shape
            assert_parity(got, want, mp, what=f"{case} frames")
