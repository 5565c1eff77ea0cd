"""the cf32 interchange format (proj/src/io.cpp:74-103) pushed
straight from a file, and the CFO estimator (proj/src/impair.cpp:45-115) built
on the conjugate Full-mode scan.  Cases follow proj/tests/test_impair.cpp:141-172
and proj/tests/test_io.cpp; the estimates are compared with the reference's own
estimate_cfo_ccf (oracle/_ref) on the same records."""
import os

import numpy as np
import pytest

from conftest import assert_parity, mean_power, rand_c

N = 1024
FRAMES = 16
BETA = 0.0625


# ---- CPU: argument guards that need no device (impair.cpp:47-49) ----

def test_cfo_guards_before_device(cyc):
    x = np.zeros(4096, np.complex64)
    with pytest.raises(cyc.UsageError, match="at least one frame"):
        cyc.estimate_cfo_ccf(x, BETA, N, 0)
    with pytest.raises(cyc.UsageError, match=r"\[-1/2, 1/2\)"):
        cyc.estimate_cfo_ccf(x, 0.75, N, 4)


def test_write_cf32_rejects_non_finite(cyc, tmp_path):
    x = np.ones(8, np.complex64)
    x[5] = np.nan
    with pytest.raises(cyc.DataError, match="index 5"):
        cyc.write_cf32(str(tmp_path / "a.cf32"), x)


def test_no_feature_error_is_a_data_error(cyc):
    assert issubclass(cyc.NoFeatureError, cyc.DataError)


# ---- GPU: the estimator against the reference ----

@pytest.mark.gpu
def test_cfo_recovers_offsets_like_reference(cyc, ref):
    """test_impair.cpp:141-157: within one bin spacing, and equal to the
    reference's own estimate on the same record."""
    x = ref.cpm(FRAMES * N + 8, h=0.5, seed=77)
    e0 = cyc.estimate_cfo_ccf(x, BETA, N, FRAMES)
    assert abs(e0) <= 0.5 / N
    assert abs(e0 - ref.estimate_cfo_ccf(x, BETA, N, FRAMES)) <= 1e-7
    for eps in (-0.01, 0.003, 0.02):
        y = ref.apply_cfo(x, eps, 0.4)
        est = cyc.estimate_cfo_ccf(y, BETA, N, FRAMES)
        assert abs(est - eps) <= 1.0 / N, (eps, est)
        assert abs(est - ref.estimate_cfo_ccf(y, BETA, N, FRAMES)) <= 1e-7, eps


@pytest.mark.gpu
@pytest.mark.parametrize("beta,eps", [(-0.0625, 0.005), (0.0625, -0.004)])
def test_cfo_mirror_feature_matches_reference(cyc, ref, beta, eps):
    """Either mirror of the GMSK conjugate pair (beta = +-1/(2 sps))."""
    x = ref.apply_cfo(ref.cpm(FRAMES * N, h=0.5, seed=5), eps, 0.1)
    want = ref.estimate_cfo_ccf(x, beta, N, FRAMES)
    got = cyc.estimate_cfo_ccf(x, beta, N, FRAMES)
    assert abs(got - want) <= 1e-7


@pytest.mark.gpu
def test_cfo_refuses_signals_without_feature(cyc, ref):
    """test_impair.cpp:160-166: h=0.7 CPM (proper) and white noise."""
    x = ref.cpm(16 * N + 8, h=0.7, seed=88)
    with pytest.raises(LookupError):
        ref.estimate_cfo_ccf(x, BETA, N, 16)
    with pytest.raises(cyc.NoFeatureError, match="no feature detected"):
        cyc.estimate_cfo_ccf(x, BETA, N, 16)
    noise = ref.awgn(16 * N + 8, 1.0, 9)
    with pytest.raises(cyc.NoFeatureError):
        cyc.estimate_cfo_ccf(noise, BETA, N, 16)


@pytest.mark.gpu
def test_cfo_argument_guards(cyc, ref):
    """test_impair.cpp:168-172."""
    x = ref.cpm(4096, h=0.5, seed=1)
    with pytest.raises(cyc.UsageError):
        cyc.estimate_cfo_ccf(x, BETA, N, 0)
    with pytest.raises(cyc.UsageError, match="too short"):
        cyc.estimate_cfo_ccf(x, BETA, N, 8)
    with pytest.raises(cyc.UsageError):
        cyc.estimate_cfo_ccf(x, 0.75, N, 4)
    with pytest.raises(cyc.ConfigError):  # N validated by the estimator (impair.cpp:56)
        cyc.estimate_cfo_ccf(x, BETA, 1, 4)


@pytest.mark.gpu
def test_cfo_non_finite_tail_is_a_data_error(cyc, ref):
    """The reference pushes the whole record, so a NaN past the last scanned
    frame still raises DataError (estimator.cpp:44-51), not NoFeatureError."""
    x = ref.cpm(FRAMES * N + 8, h=0.5, seed=77)
    x[FRAMES * N + 3] = np.nan
    with pytest.raises(cyc.DataError, match=str(FRAMES * N + 3)) as ei:
        cyc.estimate_cfo_ccf(x, BETA, N, FRAMES)
    assert not isinstance(ei.value, cyc.NoFeatureError)


# ---- GPU: cf32 file ingest ----

def _set_cfg(cyc, n=256, m=3, alphas=(0.0, 0.125, -0.25), conj=False):
    return cyc.EstimatorConfig(mode=cyc.Mode.Set, conj=conj, win_len=n, alphas=list(alphas),
                               lag_spec=cyc.LagSpec.Symmetric(m))


@pytest.mark.gpu
@pytest.mark.parametrize("conj", [False, True])
def test_push_file_matches_reference(cyc, ref, tmp_path, conj):
    """read_cf32 + push (io.cpp:90-103 + tools/main.cpp:212-214): frames equal
    the reference's on the same (float-exact) samples and the array push."""
    x = rand_c(256 * 12 + 5, 31)
    path = str(tmp_path / "rec.cf32")
    assert cyc.write_cf32(path, x) == 8 * x.size
    a = cyc.CyclicCorrelator(_set_cfg(cyc, conj=conj))
    fr = a.push_file(path)
    b = cyc.CyclicCorrelator(_set_cfg(cyc, conj=conj))
    fb = b.push(x, x)
    want, starts = ref.stream(0, int(conj), 256, x.astype(complex), x.astype(complex), alphas=(0.0, 0.125, -0.25), max_lag=3)
    assert len(fr) == len(fb) == len(want)
    mp = mean_power(x)
    for f, g, w, s in zip(fr, fb, want, starts):
        assert f.start_abs == s
        assert_parity(f.values, w, mp, what="file")
        np.testing.assert_allclose(f.values, g.values, rtol=0, atol=1e-6 * mp)
    assert a.consumed() == x.size


@pytest.mark.gpu
def test_push_file_streams_across_calls(cyc, tmp_path):
    """Two files pushed back to back behave as one stream (frames straddle)."""
    x = rand_c(256 * 6, 32)
    p1, p2 = str(tmp_path / "a.cf32"), str(tmp_path / "b.cf32")
    cyc.write_cf32(p1, x[:700])
    cyc.write_cf32(p2, x[700:])
    a = cyc.CyclicCorrelator(_set_cfg(cyc))
    frames = a.push_file(p1) + a.push_file(p2)
    b = cyc.CyclicCorrelator(_set_cfg(cyc))
    whole = b.push(x, x)
    assert [f.start_abs for f in frames] == [f.start_abs for f in whole]
    for f, g in zip(frames, whole):
        np.testing.assert_allclose(f.values, g.values, rtol=0, atol=1e-6)


@pytest.mark.gpu
def test_push_file_errors(cyc, tmp_path):
    """io.cpp:92-100: unreadable -> IoError; length % 8 != 0 -> FormatError
    (an IoError); non-finite -> DataError with the absolute index and nothing
    consumed."""
    a = cyc.CyclicCorrelator(_set_cfg(cyc))
    with pytest.raises(cyc.IoError, match="cannot open"):
        a.push_file(str(tmp_path / "missing.cf32"))
    bad = tmp_path / "trunc.cf32"
    bad.write_bytes(b"\0" * 12)
    with pytest.raises(cyc.FormatError, match="truncated"):
        a.push_file(str(bad))
    x = rand_c(1000, 33)
    x[417] = np.inf
    p = tmp_path / "nan.cf32"
    p.write_bytes(x.astype("<c8").tobytes())
    with pytest.raises(cyc.DataError) as ei:
        a.push_file(str(p))
    assert ei.value.index == 417
    assert a.consumed() == 0
    empty = tmp_path / "empty.cf32"
    empty.write_bytes(b"")
    assert a.push_file(str(empty)) == []
    assert a.consumed() == 0
    # the estimator stays usable after the errors
    x[417] = 0
    q = str(tmp_path / "ok.cf32")
    cyc.write_cf32(q, x)
    assert len(a.push_file(q)) == 3


@pytest.mark.gpu
def test_push_file_block_mode_large(cyc, ref, tmp_path):
    """A multi-MiB file through the block (emit_frames=False) path: the
    coherent average equals the reference's block average."""
    n = 2048
    x = rand_c(n * 600, 34)
    path = str(tmp_path / "big.cf32")
    cyc.write_cf32(path, x)
    cfg = _set_cfg(cyc, n=n, m=4, alphas=(0.0, 0.25, 1.0 / 8))
    cfg.emit_frames = False
    a = cyc.CyclicCorrelator(cfg)
    assert a.push_file(path) == []
    got = a.average(cyc.AverageMode.Coherent)
    want, nf = ref.block_average(0, 0, n, x, x, alphas=(0.0, 0.25, 1.0 / 8), max_lag=4)
    assert nf == 599  # the last frame waits for m lookahead samples
    assert_parity(got, want, mean_power(x), what="block file")
