"""GPU parity at the BASELINE.json production geometries (configs C1-C5).

Every case runs the product path the bench times -- the tensor-core fold with
its 2048-period tile split and several lag blocks, the 64-channel batches, the
recursive emissions, the 4096-sample Set pushes -- on the FULL record (C3:
64 emissions), and compares it with the fp64 CPU oracle (oracle/cycoracle.c,
pinned to the reference in tests/test_oracle.py) at the north-star tolerance.
The reference's own at-scale agreement gate is
proj/tests/acceptance_main.cpp:123-180 (Full vs Set) and :185-242 (chunking).
The oracle folds lags / alphas on all host cores (OpenMP), so each case costs
seconds of CPU time.
"""
import numpy as np
import pytest

from conftest import assert_parity, mean_power

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def full_block(cyc, n, lags, channels=1):
    return cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=n, lag_spec=cyc.LagSpec.Explicit(lags),
                               flags=cyc.Flags.BOTH, emit_frames=False, channels=channels)


def push_kind(cyc, est, x, kind):
    """Push the whole record through one of the two bench paths."""
    import torch
    if kind == "device":  # bench `value`: input resident in HBM, zero-copy fold
        d = torch.from_numpy(np.ascontiguousarray(x).view(np.float32)).cuda()
        est.push_device(d.data_ptr(), x.shape[-1])
        est.synchronize()
        del d
    else:  # bench `e2e`: pinned host memory through cyc_push (DMA pieces)
        p = cyc.host_alloc(x.shape)
        p[:] = x
        est.push(p)


def check_tables(got, cv, cj, lags, n_bins_total, bins, mp, what):
    """got: [2, T * N] (conv, conj) in the Full lag-major layout; cv/cj: oracle [bins, lags]."""
    for fi, want in ((0, cv), (1, cj)):
        g = got[fi].reshape(len(lags), n_bins_total)[:, bins]
        assert_parity(g, want.T, mp, what=f"{what} flag {fi}")


# ---------------------------------------------------------------------------
# C5: 2^26 samples, 8192 alphas k/8192 x lags 0..255 (Pf = 8192: 4 lag blocks,
# 8191 periods -> 4 tiles of <= 2048 periods per residue block)
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def c5_record():
    from paper_2405_16911_b200 import siggen
    return siggen.c5_record(n=1 << 26)


@pytest.fixture(scope="module")
def c5_oracle(c5_record, oracle):
    x = c5_record
    N, lags = 8192, list(range(256))
    F = (len(x) - N - 255) // N + 1
    rng = np.random.default_rng(55)
    # the features (alpha = 0, +-2 f_c, symbol rates) plus random bins
    bins = np.unique(np.concatenate([[0, 1, 8191, 4096, 1147, 8192 - 1147, 1802, 8192 - 1802, 1638, 1024],
                                     rng.choice(8192, 54, replace=False)]))
    cv, cj = oracle.block_fold(x, x, bins, N, lags, 0, F * N)
    return F, bins, cv, cj


@pytest.mark.parametrize("kind", ["device", "pinned"])
def test_c5_full_record_tensor_core_vs_oracle(cyc, c5_record, c5_oracle, kind):
    x = c5_record
    F, bins, cv, cj = c5_oracle
    est = cyc.CyclicCorrelator(full_block(cyc, 8192, list(range(256))))
    est.profile(True)
    push_kind(cyc, est, x, kind)
    prof = est.profile_read_ex()
    est.profile(False)
    assert est.frames_emitted() == F == 8191
    # the production path: tcgen05 launches over 4 lag blocks with tile splits
    assert prof["tensor_launches"] > 0, prof
    assert prof["exec_flops"] > 5 * prof["flops"] * 0.5, prof
    got = est.average_all()[0]
    check_tables(got, cv, cj, range(256), 8192, bins, mean_power(x), f"C5 {kind}")


# ---------------------------------------------------------------------------
# C2: 2^24 QPSK-RRC, 1024 alphas k/1024 x lags 0..63, every bin checked
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def c2_case(oracle):
    from paper_2405_16911_b200 import siggen
    x = siggen.c2_record(seed=2, n=1 << 24)
    N, lags = 1024, list(range(64))
    F = (len(x) - N - 63) // N + 1
    cv, cj = oracle.block_fold(x, x, np.arange(N), N, lags, 0, F * N)
    return x, F, cv, cj


@pytest.mark.parametrize("kind", ["device", "pinned"])
def test_c2_full_record_vs_oracle(cyc, c2_case, kind):
    x, F, cv, cj = c2_case
    est = cyc.CyclicCorrelator(full_block(cyc, 1024, list(range(64))))
    est.profile(True)
    push_kind(cyc, est, x, kind)
    assert est.profile_read_ex()["tensor_launches"] > 0
    est.profile(False)
    assert est.frames_emitted() == F == 16383
    check_tables(est.average_all()[0], cv, cj, range(64), 1024, np.arange(1024), mean_power(x), f"C2 {kind}")


def test_c2_repeated_device_steps_are_identical(cyc, c2_case):
    """The bench's step (reset, device push, device-out average) replays a
    captured graph from the third step on: every step equals the oracle."""
    import torch
    x, F, cv, cj = c2_case
    est = cyc.CyclicCorrelator(full_block(cyc, 1024, list(range(64))))
    d = torch.from_numpy(x.view(np.float32)).cuda()
    out = torch.empty((1, 2, 64 * 1024), dtype=torch.complex128, device="cuda")
    first = None
    for step in range(5):
        est.reset()
        est.push_device(d.data_ptr(), len(x))
        est.average_all(out=out)
        est.synchronize()
        got = out.cpu().numpy()[0]
        if first is None:
            first = got
            check_tables(got, cv, cj, range(64), 1024, np.arange(1024), mean_power(x), "C2 step 0")
        else:
            assert np.array_equal(got, first), step


# ---------------------------------------------------------------------------
# C4: 64 channels x 2^22, 128 alphas in [-1/4, 1/4) x lags 0..31, per channel
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def c4_case(oracle):
    from paper_2405_16911_b200 import siggen
    xs = np.stack([siggen.c4_channel(c, n=1 << 22) for c in range(64)])
    N, lags = 256, list(range(32))
    F = (xs.shape[1] - N - 31) // N + 1
    bins = np.array([k % N for k in range(-64, 64)])  # alpha = k/256, the config's 128-alpha subset
    want = [oracle.block_fold(xs[c], xs[c], bins, N, lags, 0, F * N) for c in range(64)]
    return xs, F, bins, want


@pytest.mark.parametrize("kind", ["device", "pinned"])
def test_c4_64_channels_vs_oracle(cyc, c4_case, kind):
    xs, F, bins, want = c4_case
    est = cyc.CyclicCorrelator(full_block(cyc, 256, list(range(32)), channels=64))
    push_kind(cyc, est, xs, kind)
    assert est.frames_emitted() == F
    allt = est.average_all()
    assert allt.shape == (64, 2, 32 * 256)
    for c in range(64):
        cv, cj = want[c]
        check_tables(allt[c], cv, cj, range(32), 256, bins, mean_power(xs[c]), f"C4 {kind} channel {c}")


# ---------------------------------------------------------------------------
# C3: recursive lambda = 1 - 2^-12, 256 alphas m/1024 x lags 0..31, emit every
# 2^16, 8192-sample work() calls; 2^22 + 2^16 samples = 64 emissions
# ---------------------------------------------------------------------------
def test_c3_64_emissions_vs_oracle(cyc, oracle):
    from paper_2405_16911_b200 import siggen
    n = (1 << 22) + (1 << 16)
    x = siggen.c3_record(n=n)
    alphas = [m / 1024 for m in range(-128, 128)]
    lam, E = 1 - 2 ** -12, 1 << 16
    est = cyc.CyclicCorrelator(cyc.EstimatorConfig(mode=cyc.Mode.Recursive, win_len=E, alphas=alphas,
                                                   lag_spec=cyc.LagSpec.Explicit(range(32)), lam=lam))
    frames = []
    for off in range(0, n, 8192):
        frames += est.push(x[off:off + 8192])
    assert len(frames) == 64
    pick = list(range(0, 256, 8)) + [127, 128, 129, 255]
    want = oracle.recursive(x.astype(complex), x.astype(complex), [alphas[i] for i in pick], list(range(32)), 0,
                            lam, E)
    assert want.shape[0] == 64
    got = np.array([f.values.reshape(256, 32)[pick] for f in frames])
    mp = mean_power(x)
    for e in range(64):
        assert_parity(got[e], want[e], mp, what=f"C3 emission {e}")


# ---------------------------------------------------------------------------
# C1: 2^20 GMSK, Set N=4096 Symmetric(15), 4096-sample pushes; per-frame
# tables and the coherent average of both estimators (conv alpha=k/8, conj
# alpha=0.1+k/16, P = 80) -- also through the union-alpha estimator the bench
# drives (one pass, both functions)
# ---------------------------------------------------------------------------
def test_c1_full_record_vs_oracle(cyc, oracle):
    from paper_2405_16911_b200 import siggen
    x = siggen.c1_record(n=1 << 20)
    conv_a = [k / 8 for k in range(-2, 3)]
    conj_a = [0.1 + k / 16 for k in range(-2, 3)]
    mp = mean_power(x)
    wants = {}
    for conj, al in ((False, conv_a), (True, conj_a)):
        est = cyc.CyclicCorrelator(cyc.EstimatorConfig(mode=cyc.Mode.Set, conj=conj, win_len=4096, alphas=al,
                                                       lag_spec=cyc.LagSpec.Symmetric(15)))
        frames = []
        for off in range(0, len(x), 4096):
            frames += est.push(x[off:off + 4096])
        want = oracle.stream(0, conj, 4096, x.astype(complex), x.astype(complex), alphas=al, max_lag=15)
        wants[conj] = want
        assert len(frames) == len(want) == 255
        got = np.array([f.values for f in frames])
        assert_parity(got, want, mp, what=f"C1 frames conj={conj}")
        assert_parity(est.average(), want.mean(axis=0), mp, what=f"C1 average conj={conj}")
    # the bench's single pass: union alpha set, both flags
    est = cyc.CyclicCorrelator(cyc.EstimatorConfig(mode=cyc.Mode.Set, win_len=4096, alphas=conv_a + conj_a,
                                                   lag_spec=cyc.LagSpec.Symmetric(15), flags=cyc.Flags.BOTH))
    frames = []
    for off in range(0, len(x), 4096):
        frames += est.push(x[off:off + 4096])
    conv = np.array([f.values for f in frames if f.flag == 1]).reshape(255, 10, 31)[:, :5]
    conj = np.array([f.values for f in frames if f.flag == 2]).reshape(255, 10, 31)[:, 5:]
    assert_parity(conv.reshape(255, -1), wants[False], mp, what="C1 union conv")
    assert_parity(conj.reshape(255, -1), wants[True], mp, what="C1 union conj")
