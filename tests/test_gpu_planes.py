"""GPU parity of the planes path (fold_tc.cu: split_planes_kernel +
fold_tcp_kernel): device-resident block pushes whose lag span covers several
64-lag blocks fold from bf16 hi/lo planes split once per sample.  Against the
fp64 oracle at the north-star tolerance, plus the reference's chunk-rejection
contract (proj/src/estimator.cpp:41-52) for the split's fused finite scan."""
import numpy as np
import pytest

from conftest import assert_parity, mean_power, rand_c

pytestmark = pytest.mark.gpu


def cfg(cyc, N, lags, channels=1):
    return cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=N, lag_spec=cyc.LagSpec.Explicit(lags),
                               flags=cyc.Flags.BOTH, emit_frames=False, channels=channels)


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a).view(np.float32)).cuda()


@pytest.mark.parametrize("lags", [list(range(128)), list(range(5, 205)), list(range(256)), list(range(0, 384, 3)), list(range(32, 160))])
def test_planes_fold_vs_oracle(cyc, oracle, lags):
    N = 1024
    x = rand_c(N * 700 + 333, 901)
    est = cyc.CyclicCorrelator(cfg(cyc, N, lags))
    est.profile(True)
    d = dev(x)
    est.push_device(d.data_ptr(), len(x))
    assert est.profile_read_ex()["tensor_launches"] > 0
    F = est.frames_emitted()
    bins = np.array([0, 1, 2, 100, 511, 512, 777, 1023])
    cv, cj = oracle.block_fold(x, x, bins, N, lags, 0, F * N)
    got = est.average_all()[0]
    for fi, want in ((0, cv), (1, cj)):
        g = got[fi].reshape(len(lags), N)[:, bins]
        assert_parity(g, want.T, mean_power(x), what=f"planes {len(lags)} lags flag {fi}")


def test_planes_unaligned_chunk_and_channels(cyc, oracle):
    """Second chunk starting at an odd absolute sample (planes base realigned),
    three channels folded in one launch."""
    N, lags, C_ = 512, list(range(160)), 3
    L1, L2 = 1001, 512 * 400 + 77
    xs = np.stack([rand_c(L1 + L2, 910 + c) for c in range(C_)])
    est = cyc.CyclicCorrelator(cfg(cyc, N, lags, channels=C_))
    a = dev(xs[:, :L1])
    est.push_device(a.data_ptr(), L1)
    b = dev(xs[:, L1:])
    est.push_device(b.data_ptr(), L2)
    F = est.frames_emitted()
    bins = np.array([0, 3, 255, 256, 400, 511])
    got = est.average_all()
    for c in range(C_):
        cv, cj = oracle.block_fold(xs[c], xs[c], bins, N, lags, 0, F * N)
        for fi, want in ((0, cv), (1, cj)):
            g = got[c, fi].reshape(len(lags), N)[:, bins]
            assert_parity(g, want.T, mean_power(xs[c]), what=f"planes channel {c} flag {fi}")


@pytest.mark.parametrize("where", [0, 12345, 700 * 1024 - 1])
def test_planes_split_rejects_chunk(cyc, where):
    """A non-finite sample anywhere in the chunk: DataError naming the absolute
    index, state unchanged (the next good chunk gives the same tables as an
    estimator that never saw the bad one)."""
    N, lags = 1024, list(range(192))
    good = rand_c(N * 300, 920)
    more = rand_c(N * 400, 921)
    bad = rand_c(N * 700, 922)
    bad[where] = np.inf if where % 2 else np.nan
    ref_est, est = cyc.CyclicCorrelator(cfg(cyc, N, lags)), cyc.CyclicCorrelator(cfg(cyc, N, lags))
    g, m, b = dev(good), dev(more), dev(bad)
    ref_est.push_device(g.data_ptr(), len(good))
    est.push_device(g.data_ptr(), len(good))
    c0 = est.consumed()
    with pytest.raises(cyc.DataError) as ei:
        est.push_device(b.data_ptr(), len(bad))
    assert ei.value.index == c0 + where
    assert est.consumed() == c0
    ref_est.push_device(m.data_ptr(), len(more))
    est.push_device(m.data_ptr(), len(more))
    for fl in (cyc.Flags.CONV, cyc.Flags.CONJ):
        assert np.max(np.abs(est.average(flag=fl) - ref_est.average(flag=fl))) <= 1e-12


def test_planes_fresh_state_rejection_leaves_zeros(cyc):
    """After reset the planes reduce overwrites the state instead of clearing
    it first; a rejected first chunk must still leave the reset (zero) state:
    the next chunk then gives the tables of an estimator that only saw it.
    (Two 64-lag blocks: the planes path; three would take the fused kernel.)"""
    N, lags = 1024, list(range(128))
    good = rand_c(N * 300, 930)
    more = rand_c(N * 400, 931)
    bad = rand_c(N * 700, 932)
    bad[4321] = np.nan
    ref_est, est = cyc.CyclicCorrelator(cfg(cyc, N, lags)), cyc.CyclicCorrelator(cfg(cyc, N, lags))
    g, m, b = dev(good), dev(more), dev(bad)
    # both accumulator buffers (reset alternates them) hold sums, and the
    # reset's clear is due
    est.push_device(g.data_ptr(), len(good))
    est.reset()
    est.push_device(g.data_ptr(), len(good))
    est.reset()
    with pytest.raises(cyc.DataError) as ei:
        est.push_device(b.data_ptr(), len(bad))
    assert ei.value.index == 4321 and est.consumed() == 0
    est.push_device(m.data_ptr(), len(more))
    ref_est.push_device(m.data_ptr(), len(more))
    for fl in (cyc.Flags.CONV, cyc.Flags.CONJ):
        assert np.max(np.abs(est.average(flag=fl) - ref_est.average(flag=fl))) <= 1e-12
    # and the accepted fresh path (reset + one chunk) equals a new estimator's
    est.reset()
    est.push_device(m.data_ptr(), len(more))
    for fl in (cyc.Flags.CONV, cyc.Flags.CONJ):
        assert np.max(np.abs(est.average(flag=fl) - ref_est.average(flag=fl))) <= 1e-12


def test_planes_matches_fused_converters(cyc):
    """The planes path and the fused-converter path compute the same products
    (same split arithmetic); tile boundaries differ, so they agree to fp32
    partial-sum rounding."""
    import os
    N, lags = 2048, list(range(128))
    x = rand_c(N * 500 + 5, 930)
    d = dev(x)
    a = cyc.CyclicCorrelator(cfg(cyc, N, lags))
    a.push_device(d.data_ptr(), len(x))
    b = cyc.CyclicCorrelator(cfg(cyc, N, lags))
    p = cyc.host_alloc(x.shape)
    p[:] = x
    b.push(p)  # pinned host pieces: ring segments, fused converters
    mp = mean_power(x)
    for fl in (cyc.Flags.CONV, cyc.Flags.CONJ):
        assert np.max(np.abs(a.average(flag=fl) - b.average(flag=fl))) <= 2e-6 * mp


def test_planes_two_cta_variant():
    """The cta_group::2 planes fold (opt-in, CYC_PLANES2=1) passes the same
    oracle checks; run in a child process because the knob is read once."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, CYC_PLANES2="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_planes.py"), "-k", "not two_cta"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
