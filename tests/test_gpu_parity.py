"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Every case replays a pin of the reference's own tests
(proj/tests/test_estimator.cpp, test_reference.cpp, acceptance_main.cpp) with
the north-star tolerance (relative L2 <= 1e-4 per table, |dR| <= 1e-5 * mean
power per value) in place of the reference's fp64 1e-12.
"""
import numpy as np
import pytest

from conftest import assert_parity, mean_power, rand_c

pytestmark = pytest.mark.gpu


def set_cfg(cyc, n, m, alphas, conj=False, **kw):
    return cyc.EstimatorConfig(mode=cyc.Mode.Set, conj=conj, win_len=n, alphas=list(alphas),
                               lag_spec=cyc.LagSpec.Symmetric(m), **kw)


def full_cfg(cyc, n, lags, conj=False, **kw):
    return cyc.EstimatorConfig(mode=cyc.Mode.Full, conj=conj, win_len=n,
                               lag_spec=cyc.LagSpec.Explicit(lags), **kw)


def frames_array(frames):
    return np.array([f.values for f in frames])


# test_estimator.cpp:211-229 -- Set windows vs the reference, x != y, both flags
@pytest.mark.parametrize("conj", [False, True])
def test_set_frames_match_oracle(cyc, oracle, conj):
    x = rand_c(400, 1234)
    y = rand_c(400, 4321)
    alphas = [3 / 64, 0.0, -0.21]
    est = cyc.CyclicCorrelator(set_cfg(cyc, 64, 3, alphas, conj))
    frames = est.push(x, y)
    want = oracle.stream(0, conj, 64, x.astype(complex), y.astype(complex), alphas=alphas, max_lag=3)
    assert len(frames) == len(want) >= 5
    for f, fr in enumerate(frames):
        assert fr.frame_index == f and fr.start_abs == 3 + 64 * f
    assert_parity(frames_array(frames), want, mean_power(x) ** 0.5 * mean_power(y) ** 0.5, what="set")


# test_estimator.cpp:242-272 -- Full mode bins, lags {-3, 0, 5}
@pytest.mark.parametrize("conj", [False, True])
def test_full_frames_match_oracle(cyc, oracle, conj):
    x = rand_c(300, 777)
    y = rand_c(300, 888)
    est = cyc.CyclicCorrelator(full_cfg(cyc, 64, [-3, 0, 5], conj))
    frames = est.push(x, y)
    want = oracle.stream(1, conj, 64, x.astype(complex), y.astype(complex), lags=[-3, 0, 5])
    assert len(frames) == len(want) >= 3
    assert_parity(frames_array(frames), want, 2.0, what="full")


def test_full_frames_match_reference(cyc, ref):
    x = rand_c(1 << 12, 5)
    for conj in (False, True):
        est = cyc.CyclicCorrelator(full_cfg(cyc, 256, [-2, 0, 3], conj))
        frames = est.push(x)
        want, st = ref.stream(1, conj, 256, x.astype(complex), x.astype(complex), lags=[-2, 0, 3], chunk=100)
        assert [f.start_abs for f in frames] == list(st)
        assert_parity(frames_array(frames), want, mean_power(x), what="full vs reference")


# test_estimator.cpp:81-105 -- tone identities
def test_tone_identities(cyc):
    f0 = 0.125
    n = np.arange(256)
    x = np.exp(2j * np.pi * f0 * n).astype(np.complex64)
    est = cyc.CyclicCorrelator(set_cfg(cyc, 64, 2, [0.0]))
    frames = est.push(x, x)
    assert frames
    lay = cyc.SetLayout(1, 2)
    for fr in frames:
        for m in range(-2, 3):
            want = np.exp(2j * np.pi * f0 * m)
            assert abs(fr.values[cyc.flat_index(lay, 0, m)] - want) <= 1e-5
    est = cyc.CyclicCorrelator(set_cfg(cyc, 64, 2, [0.25], conj=True))
    for fr in est.push(x, x):
        assert abs(fr.values[cyc.flat_index(lay, 0, 1)] - np.exp(2j * np.pi * f0)) <= 1e-5


# test_estimator.cpp:107-124 -- absolute anchoring at an off-grid alpha (direct path)
def test_absolute_anchoring_direct_path(cyc):
    alpha = 0.1234507
    f0 = alpha / 2
    n = np.arange(300 * 64 + 8)
    x = np.exp(1j * (2 * np.pi * np.fmod(f0 * n, 1.0) + 0.3)).astype(np.complex64)
    est = cyc.CyclicCorrelator(set_cfg(cyc, 64, 2, [alpha], conj=True))
    assert est.algorithm() == "direct"
    frames = est.push(x, x)
    assert len(frames) == 300
    first = frames[0].values
    for fr in frames:
        assert np.max(np.abs(fr.values - first)) <= 2e-5
    coh = est.average(cyc.AverageMode.Coherent)
    assert abs(abs(coh[2]) - 1.0) <= 2e-5


# test_estimator.cpp:126-140 -- mismatched chunks and NaN rejection, state unchanged
def test_push_rejects_bad_chunks(cyc):
    est = cyc.CyclicCorrelator(set_cfg(cyc, 8, 1, [0.0]))
    good = rand_c(4, 1)
    with pytest.raises(cyc.UsageError):
        est.push(good, rand_c(3, 2))
    poisoned = rand_c(4, 3)
    poisoned[2] = np.nan
    assert est.push(good, good) == []
    with pytest.raises(cyc.DataError, match="index 6") as ei:
        est.push(poisoned, poisoned)
    assert ei.value.index == 6
    assert est.consumed() == 4
    x = rand_c(32, 4)
    assert est.push(x, x)


def test_nan_in_y_names_y_stream(cyc):
    est = cyc.CyclicCorrelator(set_cfg(cyc, 8, 1, [0.0]))
    x = rand_c(16, 1)
    y = rand_c(16, 2)
    y[5] = np.inf
    with pytest.raises(cyc.DataError, match="index 5 in y stream"):
        est.push(x, y)
    assert est.consumed() == 0 and est.frames_emitted() == 0


# test_estimator.cpp:142-182 -- chunking invariance
def test_chunking_invariance(cyc):
    x = rand_c(1 << 13, 99)
    y = rand_c(1 << 13, 100)

    def run(cuts):
        est = cyc.CyclicCorrelator(set_cfg(cyc, 512, 5, [0.125, -0.3]))
        out, pos = [], 0
        for c in cuts:
            out += est.push(x[pos:pos + c], y[pos:pos + c])
            pos += c
        assert pos == len(x)
        return out

    whole = run([len(x)])
    assert len(whole) == 15
    rng = np.random.default_rng(7)
    parts = [[1] * 700 + [len(x) - 700], [1, 7, 64, 1000, len(x) - 1072]]
    for _ in range(2):
        cuts, left = [], len(x)
        while left:
            t = min(left, int(rng.integers(1, 701)))
            cuts.append(t)
            left -= t
        parts.append(cuts)
    for cuts in parts:
        got = run(cuts)
        assert len(got) == len(whole)
        for a, b in zip(whole, got):
            assert a.frame_index == b.frame_index and a.start_abs == b.start_abs
            assert np.max(np.abs(a.values - b.values)) <= 1e-12


# test_estimator.cpp:184-209 -- frame bookkeeping and the emission rule
def test_frame_bookkeeping(cyc):
    est = cyc.CyclicCorrelator(set_cfg(cyc, 16, 3, [0.1]))
    need = est.buffer_need()
    assert need == 22
    x = rand_c(200, 55)
    fed = emitted = 0
    rng = np.random.default_rng(3)
    while fed < len(x):
        take = min(len(x) - fed, int(rng.integers(0, 37)))
        frames = est.push(x[fed:fed + take], x[fed:fed + take])
        fed += take
        for fr in frames:
            assert fr.frame_index == emitted and fr.start_abs == 3 + emitted * 16
            emitted += 1
        assert est.frames_emitted() == ((fed - need) // 16 + 1 if fed >= need else 0)
        assert est.consumed() == fed
    assert est.frames_emitted() == 12


# test_estimator.cpp:60-68
def test_buffer_need(cyc):
    assert cyc.CyclicCorrelator(set_cfg(cyc, 8, 2, [0.125])).buffer_need() == 12
    assert cyc.CyclicCorrelator(full_cfg(cyc, 16, [-3, 5])).buffer_need() == 24
    assert cyc.CyclicCorrelator(full_cfg(cyc, 8, [0])).buffer_need() == 8
    assert cyc.CyclicCorrelator(full_cfg(cyc, 16, [-2, -1])).buffer_need() == 18


# test_estimator.cpp:231-240 -- Full-mode all-ones window
def test_full_window_all_ones(cyc):
    out = cyc.compute_full_window(np.ones(33), np.ones(32), [0, 1], False, 0)
    lay = cyc.FullLayout(2, 32)
    for l in range(2):
        assert abs(out[cyc.flat_index(lay, l, 0)] - 1) <= 1e-6
        for k in range(1, 32):
            assert abs(out[cyc.flat_index(lay, l, k)]) <= 1e-6


# test_reference.cpp:54-67 -- frozen golden values through the device window kernel
def test_frozen_values_via_set_window(cyc):
    x = np.array([1, 1j, -1 + 0.5j, 2 - 1j, 1 + 1j, -1j, 0.5, -1 - 1j])
    # a: cyclic_xcorr_direct(x, x, 0.25, m=1, conj=false, k0=1, N=4)
    v = cyc.compute_set_window(x[0:6], x[1:5], [0.25], 1, False, 1)
    assert abs(v[2] - (-0.12499999999999993 - 0.12500000000000011j)) <= 1e-6
    v = cyc.compute_set_window(x[0:6], x[1:5], [0.25], 1, True, 1)
    assert abs(v[2] - (0.12499999999999999 + 0.12500000000000006j)) <= 1e-6
    # c: alpha 0.11, m=-1, k0=2  -> window xw = x[1:7], yw = x[2:6]
    v = cyc.compute_set_window(x[1:7], x[2:6], [0.11], 1, False, 2)
    assert abs(v[0] - (-0.26908075755090433 + 0.66834328861739112j)) <= 1e-6


# test_reference.cpp:92-115 -- compute_set_window == direct sum
def test_set_window_vs_direct(cyc, oracle):
    x = rand_c(200, 2718).astype(complex)
    y = rand_c(200, 2719).astype(complex)
    alphas = [0.0, 0.125, -0.37, 0.11]
    M, k0 = 4, 37
    for conj in (False, True):
        vals = cyc.compute_set_window(x[k0 - M:k0 + 64 + M], y[k0:k0 + 64], alphas, M, conj, k0)
        lay = cyc.SetLayout(4, M)
        for a, al in enumerate(alphas):
            for m in range(-M, M + 1):
                want = oracle.direct(x, y, al, m, conj, k0, 64)
                assert abs(vals[cyc.flat_index(lay, a, m)] - want) <= 1e-5


# Block mode (emit_frames = 0): coherent average == reference average_frames
@pytest.mark.parametrize("conj", [False, True])
def test_block_average_full_mode(cyc, oracle, conj):
    x = rand_c(1 << 16, 11)
    N, lags = 256, list(range(8))
    est = cyc.CyclicCorrelator(full_cfg(cyc, N, lags, conj, emit_frames=False))
    assert est.push(x) == []
    F = est.frames_emitted()
    assert F == (len(x) - N - 7) // N + 1
    got = est.average()
    cv, cj = oracle.block_fold(x, x, np.arange(N), N, lags, 0, F * N)
    want = (cj if conj else cv).T.reshape(-1)
    assert_parity(got, want, mean_power(x), what="block full")


def test_block_average_both_flags_chunked(cyc, oracle):
    x = rand_c(100_000, 12)
    N, lags = 1024, list(range(64))
    cfg = full_cfg(cyc, N, lags, flags=cyc.Flags.BOTH, emit_frames=False)
    est = cyc.CyclicCorrelator(cfg)
    for c in np.array_split(np.arange(len(x)), 7):
        est.push(x[c[0]:c[-1] + 1])
    F = est.frames_emitted()
    cv, cj = oracle.block_fold(x, x, np.arange(N), N, lags, 0, F * N)
    assert_parity(est.average(flag=cyc.Flags.CONV), cv.T.reshape(-1), mean_power(x), what="conv")
    assert_parity(est.average(flag=cyc.Flags.CONJ), cj.T.reshape(-1), mean_power(x), what="conj")


def test_block_average_matches_reference_block(cyc, ref):
    x = rand_c(1 << 15, 21)
    N, lags = 512, list(range(16))
    for conj in (False, True):
        est = cyc.CyclicCorrelator(full_cfg(cyc, N, lags, conj, emit_frames=False))
        est.push(x)
        want, F = ref.block_average(1, conj, N, x, x, lags=lags)
        assert F == est.frames_emitted()
        assert_parity(est.average(), want, mean_power(x), what="vs reference")


def test_set_block_average_grid_alphas(cyc, oracle):
    """Set-mode block average at the C1 conjugate grid alpha = 0.1 + k/16 (P = 80)."""
    x = rand_c(40_000, 31)
    alphas = [0.1 + k / 16 for k in range(-2, 3)]
    M, N = 15, 4096
    for conj in (False, True):
        est = cyc.CyclicCorrelator(set_cfg(cyc, N, M, alphas, conj, emit_frames=False))
        assert est.algorithm().startswith("fold")
        est.push(x)
        F = est.frames_emitted()
        want = oracle.block_direct(x.astype(complex), x.astype(complex), alphas, list(range(-M, M + 1)), conj,
                                   M, F * N)
        assert_parity(est.average(), want.reshape(-1), mean_power(x), what="set block")


def test_direct_block_average(cyc, oracle):
    x = rand_c(20_000, 41)
    alphas = [0.1234507, -0.3333333]
    est = cyc.CyclicCorrelator(set_cfg(cyc, 1000, 4, alphas, False, emit_frames=False))
    assert est.algorithm() == "direct"
    est.push(x)
    F = est.frames_emitted()
    want = oracle.block_direct(x.astype(complex), x.astype(complex), alphas, list(range(-4, 5)), False, 4, F * 1000)
    assert_parity(est.average(), want.reshape(-1), mean_power(x), what="direct block")


def test_magnitude_average(cyc):
    x = rand_c(64, 31)
    est = cyc.CyclicCorrelator(set_cfg(cyc, 16, 1, [0.25]))
    frames = est.push(x, x)
    assert len(frames) >= 2
    mag = est.average(cyc.AverageMode.Magnitude)
    want = cyc.average_frames(frames, cyc.AverageMode.Magnitude)
    assert np.max(np.abs(mag - want)) <= 1e-12
    coh = est.average(cyc.AverageMode.Coherent)
    assert np.max(np.abs(coh - cyc.average_frames(frames))) <= 1e-12


def test_recursive_matches_oracle(cyc, oracle):
    x = rand_c(5000, 51)
    alphas = [m / 64 for m in range(-4, 4)]
    lags = [0, 1, 2, 3]
    lam, E = 1 - 2 ** -6, 512
    cfg = cyc.EstimatorConfig(mode=cyc.Mode.Recursive, win_len=E, alphas=alphas,
                              lag_spec=cyc.LagSpec.Explicit(lags), lam=lam)
    est = cyc.CyclicCorrelator(cfg)
    frames = []
    for c in np.array_split(np.arange(len(x)), 5):
        frames += est.push(x[c[0]:c[-1] + 1])
    want = oracle.recursive(x.astype(complex), x.astype(complex), alphas, lags, False, lam, E)
    assert len(frames) == len(want)
    got = np.array([f.values for f in frames]).reshape(want.shape)
    assert_parity(got, want, mean_power(x), what="recursive")


def test_multichannel_block(cyc, oracle):
    C_, L = 4, 30_000
    xs = np.stack([rand_c(L, 100 + c) for c in range(C_)])
    N, lags = 256, list(range(32))
    est = cyc.CyclicCorrelator(full_cfg(cyc, N, lags, flags=cyc.Flags.BOTH, emit_frames=False, channels=C_))
    est.push(xs)
    F = est.frames_emitted()
    for c in range(C_):
        cv, cj = oracle.block_fold(xs[c], xs[c], np.arange(N), N, lags, 0, F * N)
        assert_parity(est.average(flag=cyc.Flags.CONV, channel=c), cv.T.reshape(-1), mean_power(xs[c]))
        assert_parity(est.average(flag=cyc.Flags.CONJ, channel=c), cj.T.reshape(-1), mean_power(xs[c]))


def test_pinned_and_f64_inputs_agree(cyc):
    x = rand_c(50_000, 61)
    N, lags = 1024, list(range(16))
    outs = []
    for kind in ("pageable", "pinned", "f64"):
        est = cyc.CyclicCorrelator(full_cfg(cyc, N, lags, emit_frames=False))
        if kind == "pinned":
            px = cyc.host_alloc(x.shape)
            px[:] = x
            est.push(px)
        elif kind == "f64":
            est.push(x.astype(np.complex128))
        else:
            est.push(x)
        outs.append(est.average())
    assert np.max(np.abs(outs[0] - outs[1])) <= 1e-12
    assert np.max(np.abs(outs[0] - outs[2])) <= 1e-12


def test_device_push(cyc):
    import torch
    x = rand_c(70_000, 71)
    N, lags = 1024, list(range(64))
    a = cyc.CyclicCorrelator(full_cfg(cyc, N, lags, emit_frames=False))
    a.push(x)
    b = cyc.CyclicCorrelator(full_cfg(cyc, N, lags, emit_frames=False))
    dx = torch.from_numpy(x).cuda()
    b.push_device(dx.data_ptr(), len(x))
    # host and device ingest tile the fold differently (fp32 partial sums in a
    # different grouping): equal to well inside the north-star tolerance
    mp = mean_power(x)
    assert np.max(np.abs(a.average() - b.average())) <= 1e-6 * mp


def test_device_push_tensor_core_fold_vs_oracle(cyc, oracle):
    """The block fold of a device-resident chunk runs on the tensor cores
    (bf16x3 split, fold_tc.cu) for every interior fold period; parity with the
    fp64 oracle at the north-star tolerance, both flags, lags 0..63 and
    64..127 (second lag block: y is staged separately from the x window)."""
    import torch
    N = 1024
    x = rand_c(N * 300 + 77, 72)
    dx = torch.from_numpy(x).cuda()
    mp = mean_power(x)
    bins = np.array([0, 1, 3, 100, 511, 512, 700, 1023])
    # negative lags: the x window starts before the residue block, and the
    # partial head/tail periods fold on the FP32 kernel into the same slot
    for lags in (list(range(64)), list(range(128)), list(range(-32, 32)), list(range(-16, 16)), list(range(32))):
        est = cyc.CyclicCorrelator(full_cfg(cyc, N, lags, flags=cyc.Flags.BOTH, emit_frames=False))
        est.push_device(dx.data_ptr(), len(x))
        F = est.frames_emitted()
        m_minus = max(0, -lags[0])
        cv, cj = oracle.block_fold(x, x, bins, N, lags, m_minus, F * N)
        for fl, want in ((cyc.Flags.CONV, cv), (cyc.Flags.CONJ, cj)):
            got = est.average(flag=fl).reshape(len(lags), N)[:, bins]
            assert_parity(got, want.T, mp, what=f"tc fold {len(lags)} lags flag {fl}")


# Speculative block pushes (pinned host / device input): the GPU finite scan
# runs while the chunk is folded into a pending accumulator; a bad chunk must
# leave the estimator exactly as it was (estimator.cpp:43-52).
@pytest.mark.parametrize("kind", ["pinned", "device"])
def test_speculative_push_rollback(cyc, kind):
    import torch
    N, lags = 1024, list(range(64))
    x = rand_c(3 << 20, 81)
    bad = rand_c(5 << 20, 82)
    bad[(3 << 20) + 12345] = np.nan + 1j
    cfg = full_cfg(cyc, N, lags, flags=cyc.Flags.BOTH, emit_frames=False)
    ref_est, est = cyc.CyclicCorrelator(cfg), cyc.CyclicCorrelator(cfg)

    def push(e, a):
        if kind == "pinned":
            p = cyc.host_alloc(a.shape)
            p[:] = a
            return e.push(p)
        d = torch.from_numpy(a.view(np.float32)).cuda()
        return e.push_device(d.data_ptr(), len(a))

    push(ref_est, x[: 1 << 20])
    push(est, x[: 1 << 20])
    c0, f0 = est.consumed(), est.frames_emitted()
    with pytest.raises(cyc.DataError, match=f"index {c0 + (3 << 20) + 12345} in x stream"):
        push(est, bad)
    assert est.consumed() == c0 and est.frames_emitted() == f0
    push(ref_est, x[1 << 20:])
    push(est, x[1 << 20:])
    for fl in (cyc.Flags.CONV, cyc.Flags.CONJ):
        assert np.max(np.abs(est.average(flag=fl) - ref_est.average(flag=fl))) <= 1e-12


@pytest.mark.parametrize("n", [(1 << 16) + 1, 1 << 16, 1000, 3])
def test_device_scan_names_first_bad_sample(cyc, n):
    """The device finite scan (vectorised + scalar tail) reports exactly the
    reference's first offender: lowest index, x before y at the same index."""
    import torch
    rng = np.random.default_rng(n)
    cases = [[0], [n - 1], [n // 2, n // 2 + 1], [n - 2, n - 1]] + [sorted(rng.choice(n, 3, replace=False))
                                                                      for _ in range(3)]
    for pos in cases:
        pos = [int(p) for p in pos if 0 <= p < n]
        for stream in ("x", "y", "both"):
            x, y = rand_c(n, 5), rand_c(n, 6)
            for p in pos:
                if stream in ("x", "both"):
                    x[p] = np.inf
                if stream in ("y", "both"):
                    y[p] = np.nan
            est = cyc.CyclicCorrelator(full_cfg(cyc, 2, [0], flags=cyc.Flags.BOTH, emit_frames=False))
            dx = torch.from_numpy(x).cuda()
            dy = torch.from_numpy(y).cuda()
            with pytest.raises(cyc.DataError) as ei:
                est.push_device(dx.data_ptr(), n, dy.data_ptr())
            first = min(pos)
            assert ei.value.index == first, (n, pos, stream)
            assert f"in {'y' if stream == 'y' else 'x'} stream" in str(ei.value)
            assert est.consumed() == 0


def test_c2_scale_block_average_vs_oracle(cyc, oracle):
    """Config 2 geometry at 2^22 samples (the oracle's fold finishes in seconds)."""
    from paper_2405_16911_b200 import siggen
    x = siggen.c2_record(seed=2, n=1 << 22)
    N, lags = 1024, list(range(64))
    est = cyc.CyclicCorrelator(full_cfg(cyc, N, lags, flags=cyc.Flags.BOTH, emit_frames=False))
    p = cyc.host_alloc(x.shape)
    p[:] = x
    est.push(p)
    F = est.frames_emitted()
    cv, cj = oracle.block_fold(x, x, np.arange(N), N, lags, 0, F * N)
    mp = mean_power(x)
    assert_parity(est.average(flag=cyc.Flags.CONV), cv.T.reshape(-1), mp, what="C2 conv")
    assert_parity(est.average(flag=cyc.Flags.CONJ), cj.T.reshape(-1), mp, what="C2 conj")


def test_average_all_matches_per_channel(cyc):
    C_, L = 3, 20_000
    xs = np.stack([rand_c(L, 200 + c) for c in range(C_)])
    est = cyc.CyclicCorrelator(full_cfg(cyc, 256, list(range(8)), flags=cyc.Flags.BOTH, emit_frames=False, channels=C_))
    est.push(xs)
    allt = est.average_all()
    assert allt.shape == (C_, 2, 8 * 256)
    for c in range(C_):
        assert np.max(np.abs(allt[c, 0] - est.average(flag=cyc.Flags.CONV, channel=c))) <= 1e-15
        assert np.max(np.abs(allt[c, 1] - est.average(flag=cyc.Flags.CONJ, channel=c))) <= 1e-15
    # the same tables DMA'd into pinned host memory and into device memory
    pinned = cyc.host_alloc(allt.shape, dtype=np.complex128)
    assert est.average_all(out=pinned) is pinned
    assert np.array_equal(np.asarray(pinned), allt)
    import torch
    dev = torch.empty(allt.shape, dtype=torch.complex128, device="cuda")
    est.average_all(out=dev)  # stream-ordered on the estimator's stream
    est.synchronize()
    assert np.array_equal(dev.cpu().numpy(), allt)
    one = cyc.host_alloc(8 * 256, dtype=np.complex128)
    est.average(flag=cyc.Flags.CONJ, channel=2, out=one)
    assert np.array_equal(np.asarray(one), allt[2, 1])


def test_device_output_needs_block_mode(cyc):
    """Per-frame estimators scale on the host, so a device `out` is refused."""
    import torch
    x = rand_c(4096, 201)
    est = cyc.CyclicCorrelator(full_cfg(cyc, 256, [0, 1]))
    est.push(x)
    dev = torch.empty(2 * 256, dtype=torch.complex128, device="cuda")
    with pytest.raises(cyc.UsageError, match="device-memory output"):
        est.average(out=dev)


# BASELINE configs at reduced sizes (full sizes run in bench.py --config cN)
def test_c5_geometry_vs_oracle(cyc, oracle):
    """Config 5: 8192-bin grid x lags 0..255, both flags (2^20 samples; oracle on 24 bins)."""
    from paper_2405_16911_b200 import siggen
    x = siggen.c5_record(n=1 << 20)
    est = cyc.CyclicCorrelator(full_cfg(cyc, 8192, list(range(256)), flags=cyc.Flags.BOTH, emit_frames=False))
    est.push(x)
    F = est.frames_emitted()
    bins = np.array([0, 1, 2, 7, 100, 1147, 1148, 2000, 2294, 4095, 4096, 5000, 6000, 7000, 7045, 8191,
                     3, 8190, 1802, 6389, 12, 33, 4444, 8000])
    cv, cj = oracle.block_fold(x, x, bins, 8192, list(range(256)), 0, F * 8192)
    mp = mean_power(x)
    got = est.average_all()  # [1, 2, 256 * 8192]
    for fi, want in ((0, cv), (1, cj)):
        g = got[0, fi].reshape(256, 8192)[:, bins]
        assert_parity(g, want.T, mp, what=f"C5 flag {fi}")


def test_c3_geometry_vs_oracle(cyc, oracle):
    """Config 3: recursive lambda = 1 - 2^-12, 256 alphas m/1024 x lags 0..31, emit every 2^16
    (2^18 samples in 8192-sample calls; oracle on 6 alphas)."""
    from paper_2405_16911_b200 import siggen
    x = siggen.gmsk(1 << 18, 0.3, 8, 0.02, 3).astype(np.complex64)
    alphas = [m / 1024 for m in range(-128, 128)]
    cfg = cyc.EstimatorConfig(mode=cyc.Mode.Recursive, win_len=1 << 16, alphas=alphas,
                              lag_spec=cyc.LagSpec.Explicit(range(32)), lam=1 - 2 ** -12)
    est = cyc.CyclicCorrelator(cfg)
    frames = []
    for off in range(0, len(x), 8192):
        frames += est.push(x[off:off + 8192])
    assert len(frames) == (len(x) - (1 << 16) - 31) // (1 << 16) + 1
    pick = [0, 5, 100, 128, 200, 255]
    want = oracle.recursive(x.astype(complex), x.astype(complex), [alphas[i] for i in pick], list(range(32)), 0,
                            1 - 2 ** -12, 1 << 16)
    got = np.array([f.values.reshape(256, 32)[pick] for f in frames])
    assert_parity(got, want, mean_power(x), what="C3")


def test_c1_geometry_vs_oracle(cyc, oracle):
    """Config 1: Set N=4096, Symmetric(15), conj alphas 0.1 + k/16 (P = 80), 4096-sample pushes."""
    from paper_2405_16911_b200 import siggen
    x = siggen.c1_record(n=1 << 16)
    for conj, al in ((False, [k / 8 for k in range(-2, 3)]), (True, [0.1 + k / 16 for k in range(-2, 3)])):
        est = cyc.CyclicCorrelator(set_cfg(cyc, 4096, 15, al, conj))
        frames = []
        for off in range(0, len(x), 4096):
            frames += est.push(x[off:off + 4096])
        want = oracle.stream(0, conj, 4096, x.astype(complex), x.astype(complex), alphas=al, max_lag=15)
        assert len(frames) == len(want)
        assert_parity(frames_array(frames), want, mean_power(x), what=f"C1 conj={conj}")


def test_multichannel_tensor_core_fold_batches(cyc):
    """20 channels of device-resident block folds: the tensor-core launches
    are batched 16 segments at a time (tensor maps per segment); every
    channel equals its own single-channel estimator."""
    import torch
    C_, N, L = 20, 1024, 1024 * 220
    xs = np.stack([rand_c(L, 300 + c) for c in range(C_)])
    lags = list(range(64))
    multi = cyc.CyclicCorrelator(full_cfg(cyc, N, lags, flags=cyc.Flags.BOTH, emit_frames=False, channels=C_))
    d = torch.from_numpy(xs).cuda()
    multi.push_device(d.data_ptr(), L)
    allt = multi.average_all()
    for c in (0, 7, 15, 16, 19):
        one = cyc.CyclicCorrelator(full_cfg(cyc, N, lags, flags=cyc.Flags.BOTH, emit_frames=False))
        dc = torch.from_numpy(np.ascontiguousarray(xs[c])).cuda()
        one.push_device(dc.data_ptr(), L)
        mp = mean_power(xs[c])
        for fi, fl in ((0, cyc.Flags.CONV), (1, cyc.Flags.CONJ)):
            assert np.max(np.abs(allt[c, fi] - one.average(flag=fl))) <= 1e-6 * mp, (c, fl)


@pytest.mark.parametrize("kind", ["pinned", "device", "pageable"])
def test_multichannel_first_bad_sample(cyc, kind):
    """The finite scan covers every channel (one launch over all channel rows):
    the error names the first offender in (index, x-before-y, channel) order
    and leaves the estimator unchanged."""
    import torch
    C_, L = 5, 3 << 20
    xs = np.stack([rand_c(L, 400 + c) for c in range(C_)])
    xs[3, 2_000_123] = np.nan
    xs[1, 2_500_000] = np.inf
    cfg = full_cfg(cyc, 1024, list(range(32)), emit_frames=False, channels=C_)
    est = cyc.CyclicCorrelator(cfg)
    good = np.stack([rand_c(4096, 500 + c) for c in range(C_)])
    est.push(good)
    c0 = est.consumed()
    if kind == "pinned":
        p = cyc.host_alloc(xs.shape)
        p[:] = xs
        call = lambda: est.push(p)
    elif kind == "device":
        d = torch.from_numpy(xs).cuda()
        call = lambda: est.push_device(d.data_ptr(), L)
    else:
        call = lambda: est.push(xs)
    with pytest.raises(cyc.DataError, match=f"index {c0 + 2_000_123} in x stream of channel 3") as ei:
        call()
    assert ei.value.index == c0 + 2_000_123
    assert est.consumed() == c0


# proj/src/fft.cpp:72-87: non-power-of-two N takes the direct DFT -- on the GPU
# the exact-index DFT finalize over Pf = lcm(N, 128)
@pytest.mark.parametrize("N", [1000, 768])
def test_full_mode_non_pow2_window_vs_oracle(cyc, oracle, N):
    x = rand_c(N * 9 + 17, 940 + N)
    lags = [-2, 0, 3, 7]
    mp = mean_power(x)
    for conj in (False, True):
        est = cyc.CyclicCorrelator(full_cfg(cyc, N, lags, conj))
        frames = est.push(x)
        want = oracle.stream(1, conj, N, x.astype(complex), x.astype(complex), lags=lags)
        assert len(frames) == len(want) >= 8
        assert_parity(frames_array(frames), want, mp, what=f"Full N={N} conj={conj} frames")
        # block mode: the coherent average from one fold
        blk = cyc.CyclicCorrelator(full_cfg(cyc, N, lags, conj, emit_frames=False))
        blk.push(x)
        assert_parity(blk.average(), want.mean(axis=0), mp, what=f"Full N={N} conj={conj} block")


def test_offgrid_direct_block_average_long_record(cyc, oracle):
    """Alphas off any rational grid (direct kernel) averaged over 2^22 samples:
    the long per-thread sums stay within the north-star tolerance of the fp64
    literal sum (proj/src/reference.cpp:11-32 summed over the block)."""
    L = 1 << 22
    x = rand_c(L, 950)
    alphas = [0.1234507, -0.3141592653]
    est = cyc.CyclicCorrelator(set_cfg(cyc, 4096, 2, alphas, emit_frames=False))
    assert est.algorithm() == "direct"
    est.push(x)
    F = est.frames_emitted()
    got = est.average().reshape(len(alphas), 5)
    want = oracle.block_direct(x.astype(complex), x.astype(complex), alphas, [-2, -1, 0, 1, 2], False, 2, F * 4096)
    # the reference's frames carry e^{-j 2 pi alpha k0} with k0 = m_minus + f N (absolute anchor): the block
    # sum over [m_minus, m_minus + F N) equals the mean of the frames
    assert_parity(got, want, mean_power(x), what="off-grid direct block average")


def test_estimators_on_two_devices(cyc, oracle):
    """Handles on different devices of one process: each
    device gets its kernels' shared-memory opt-in (kernels.cuh first_on_device)."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    x = rand_c(1024 * 300 + 5, 960)
    N, lags = 1024, list(range(64))
    outs = []
    for d in (0, 1):
        est = cyc.CyclicCorrelator(full_cfg(cyc, N, lags, flags=cyc.Flags.BOTH, emit_frames=False, device=d))
        dx = torch.from_numpy(x.view(np.float32)).to(f"cuda:{d}")
        est.push_device(dx.data_ptr(), len(x))
        outs.append(est.average_all())
    F = (len(x) - N - 63) // N + 1
    cv, cj = oracle.block_fold(x, x, np.arange(0, N, 37), N, lags, 0, F * N)
    for o in outs:
        assert_parity(o[0, 0].reshape(64, N)[:, ::37], cv.T, mean_power(x))
        assert_parity(o[0, 1].reshape(64, N)[:, ::37], cj.T, mean_power(x))


def test_block_average_device_matches_separate_calls(cyc, oracle):
    """cyc_block_average_device = reset + push_device + average_all (one host
    synchronisation), against the oracle; a rejected chunk raises DataError with
    the chunk's index and leaves the reset state."""
    import torch
    N, lags = 1024, list(range(64))
    x = rand_c(N * 300 + 17, 77)
    cfg = cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=N, lag_spec=cyc.LagSpec.Explicit(lags),
                              flags=cyc.Flags.BOTH, emit_frames=False)
    est = cyc.CyclicCorrelator(cfg)
    d = torch.from_numpy(x.view(np.float32)).cuda()
    out = torch.empty((1, 2, len(lags) * N), dtype=torch.complex128, device="cuda")
    for _ in range(2):  # the second call replays the captured push
        est.block_average_device(d.data_ptr(), len(x), out)
    got = out.cpu().numpy()
    ref = cyc.CyclicCorrelator(cfg)
    ref.push_device(d.data_ptr(), len(x))
    want = ref.average_all()
    assert np.array_equal(got, want)
    F = est.frames_emitted()
    bins = np.array([0, 5, 511, 1023])
    cv, cj = oracle.block_fold(x, x, bins, N, lags, 0, F * N)
    for fi, w in ((0, cv), (1, cj)):
        assert_parity(got[0, fi].reshape(len(lags), N)[:, bins], w.T, mean_power(x), what=f"flag {fi}")
    bad = x.copy()
    bad[4321] = np.nan
    db = torch.from_numpy(bad.view(np.float32)).cuda()
    with pytest.raises(cyc.DataError) as ei:
        est.block_average_device(db.data_ptr(), len(bad), out)
    assert ei.value.index == 4321
    assert est.consumed() == 0 and est.frames_emitted() == 0
