"""Fused finite check and CUDA-graph replay of device-resident block pushes.

A device chunk whose folds are one tensor-core launch is validated inside that
launch (each staged sample of the covered periods checked once) plus a small
scan of the rest; the reference's push semantics (estimator.cpp:43-52: the
first non-finite sample rejects the whole chunk, state unchanged) must hold
exactly as with the stand-alone scan.  Repeated pushes of the same buffer at
the same stream position replay a captured CUDA graph: results and verdicts
must not change.
"""
import numpy as np
import pytest

from conftest import rand_c

pytestmark = pytest.mark.gpu

W, LAGS = 1024, list(range(64))  # tensor-core geometry: Pf = 1024, one 64-lag block


def block_cfg(cyc, channels=1):
    return cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=W, lag_spec=cyc.LagSpec.Explicit(LAGS),
                               flags=cyc.Flags.BOTH, emit_frames=False, channels=channels)


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


N = 1 << 20
# covered periods are [0, 1023) x 1024 for this geometry; the rest is scanned
FUSED_POS = [0, 5000, 500 * W + 127, 500 * W + 128, 700 * W + 1023, 1022 * W + 1023]
REST_POS = [1023 * W, N - 1024, N - 1]


@pytest.mark.parametrize("pos", FUSED_POS + REST_POS)
@pytest.mark.parametrize("bad", ["inf_re", "nan_im", "ninf_im"])
def test_fused_check_names_the_offender(cyc, pos, bad):
    x = rand_c(N, 11)
    if bad == "inf_re":
        x[pos] = complex(np.inf, x[pos].imag)
    elif bad == "nan_im":
        x[pos] = complex(x[pos].real, np.nan)
    else:
        x[pos] = complex(x[pos].real, -np.inf)
    est = cyc.CyclicCorrelator(block_cfg(cyc))
    d = dev(x)
    with pytest.raises(cyc.DataError, match=f"non-finite sample at absolute index {pos} in x stream") as ei:
        est.push_device(d.data_ptr(), N)
    assert ei.value.index == pos
    assert est.consumed() == 0 and est.frames_emitted() == 0


def test_fused_check_first_of_many(cyc):
    """The lowest index wins across the fused ranges and the scanned rest."""
    x = rand_c(N, 12)
    for p in (N - 3, 1023 * W + 7, 900 * W + 200, 611_111, 611_112):
        x[p] = np.nan
    est = cyc.CyclicCorrelator(block_cfg(cyc))
    d = dev(x)
    with pytest.raises(cyc.DataError) as ei:
        est.push_device(d.data_ptr(), N)
    assert ei.value.index == 611_111


def test_fused_check_cross_and_channels(cyc):
    """x before y at one index; the lowest channel at one (index, stream)."""
    x, y = rand_c(N, 13), rand_c(N, 14)
    y[300_000] = np.inf
    est = cyc.CyclicCorrelator(block_cfg(cyc))
    dx, dy = dev(x), dev(y)
    with pytest.raises(cyc.DataError, match="index 300000 in y stream"):
        est.push_device(dx.data_ptr(), N, dy.data_ptr())
    x[300_000] = np.nan
    dx = dev(x)
    with pytest.raises(cyc.DataError, match="index 300000 in x stream"):
        est.push_device(dx.data_ptr(), N, dy.data_ptr())
    C = 3
    xs = np.stack([rand_c(N, 20 + c) for c in range(C)])
    xs[2, 400_000] = np.nan
    xs[0, 400_001] = np.nan
    xs[1, 1023 * W + 1] = np.inf
    est = cyc.CyclicCorrelator(block_cfg(cyc, channels=C))
    d = dev(xs)
    with pytest.raises(cyc.DataError, match="index 400000 in x stream of channel 2"):
        est.push_device(d.data_ptr(), N)
    assert est.consumed() == 0


def test_fused_check_accepts_huge_finite_values(cyc):
    """A finite value whose bf16 split overflows is only a hint: the exact
    re-check accepts it (the reference accepts every finite float)."""
    x = rand_c(N, 15)
    x[123_456] = complex(3.4e38, -3.4e38)
    est = cyc.CyclicCorrelator(block_cfg(cyc))
    d = dev(x)
    est.push_device(d.data_ptr(), N)
    assert est.consumed() == N


def test_rejected_chunk_leaves_state_and_replays_identically(cyc):
    """Same buffer, same position: the second and later pushes replay a captured
    graph.  Results are bit-identical to the direct pushes, a poisoned replay
    is rejected with the exact index and changes nothing, and the good replay
    afterwards still matches."""
    import torch
    x = rand_c(N, 16)
    d = dev(x)
    ref = cyc.CyclicCorrelator(block_cfg(cyc))
    ref.push_device(d.data_ptr(), N)
    want = ref.average_all()
    est = cyc.CyclicCorrelator(block_cfg(cyc))
    out = torch.empty(want.shape, dtype=torch.complex128, device="cuda")
    for it in range(4):
        est.reset()
        est.push_device(d.data_ptr(), N)
        est.average_all(out=out)
        assert np.array_equal(out.cpu().numpy(), want), it
    for pos in (777_777, N - 5):
        d[pos] = complex(np.nan, 0.0)  # same buffer: a replay of the captured push
        est.reset()
        with pytest.raises(cyc.DataError) as ei:
            est.push_device(d.data_ptr(), N)
        assert ei.value.index == pos and est.consumed() == 0
        d[pos] = torch.tensor(x[pos], dtype=torch.complex64)
    est.push_device(d.data_ptr(), N)
    est.average_all(out=out)
    assert np.array_equal(out.cpu().numpy(), want)


def test_device_push_orders_after_default_stream_producer(cyc):
    """The chunk is read after work the caller queued on the default stream,
    and the caller's later default-stream writes wait for the fold."""
    import torch
    x = rand_c(N, 17)
    src = dev(x)
    ref = cyc.CyclicCorrelator(block_cfg(cyc))
    ref.push_device(src.data_ptr(), N)
    want = ref.average_all()
    est = cyc.CyclicCorrelator(block_cfg(cyc))
    d = torch.empty_like(src)
    for _ in range(3):
        est.reset()
        d.zero_()
        torch.cuda._sleep(2_000_000)  # a slow producer on the default stream
        d.copy_(src)
        est.push_device(d.data_ptr(), N)
        d.zero_()  # ordered after the fold by the push's fence
        got = est.average_all()
        assert np.array_equal(got, want)


def test_chunked_device_pushes_match_one_push(cyc):
    """Unequal device chunks (frames straddling chunk boundaries read the ring,
    so only the first push takes the fused check and the graph) give the one-push
    tables within the north-star tolerance; repeating the whole sequence after a
    reset replays identically."""
    from conftest import assert_parity, mean_power
    x = rand_c(3 * N, 18)
    cuts = [0, 700_001, 1_900_000, 3 * N]
    d = dev(x)
    one = cyc.CyclicCorrelator(block_cfg(cyc))
    one.push_device(d.data_ptr(), 3 * N)
    want = one.average_all()
    est = cyc.CyclicCorrelator(block_cfg(cyc))
    first = None
    for rep in range(3):
        est.reset()
        for a, b in zip(cuts[:-1], cuts[1:]):
            est.push_device(d.data_ptr() + 8 * a, b - a)
        got = est.average_all()
        assert est.frames_emitted() == one.frames_emitted()
        for fl in range(2):
            assert_parity(got[0, fl], want[0, fl], mean_power(x), rel_l2=1e-5, what=f"flag {fl}")
        if first is None:
            first = got
        assert np.array_equal(got, first), rep


@pytest.mark.parametrize("pos", [0, 333_333, (1 << 21) - 1, (1 << 21) - 3000])
def test_fused_check_multi_launch_plan(cyc, pos):
    """Three 64-lag blocks (lb 0 self, lb 1-2 not): several tensor-core launches,
    the first of which holds every lb = 0 group and checks the chunk.  Verdicts
    are exact, and a clean chunk matches the pinned-host path's tables."""
    from conftest import assert_parity, mean_power
    n = 1 << 21
    cfg = cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=2048, lag_spec=cyc.LagSpec.Explicit(range(192)),
                              flags=cyc.Flags.BOTH, emit_frames=False)
    x = rand_c(n, 30)
    est = cyc.CyclicCorrelator(cfg)
    d = dev(x)
    est.push_device(d.data_ptr(), n)
    host = cyc.CyclicCorrelator(cfg)
    p = cyc.host_alloc(x.shape)
    p[:] = x
    host.push(p)
    got, want = est.average_all(), host.average_all()
    for fl in range(2):
        assert_parity(got[0, fl], want[0, fl], mean_power(x), rel_l2=1e-5, what=f"flag {fl}")
    bad = x.copy()
    bad[pos] = np.nan
    est.reset()
    db = dev(bad)
    with pytest.raises(cyc.DataError) as ei:
        est.push_device(db.data_ptr(), n)
    assert ei.value.index == pos and est.consumed() == 0


def test_fused_check_many_channel_batches(cyc):
    """C4-like (Full N=256, lags 0..31) with 20 channels: two segment batches,
    so the folds land in the pending accumulator and a gated add commits them.
    Clean chunks match the pinned-host path; a bad sample in the second batch
    rejects the chunk (exact channel and index) and commits nothing."""
    from conftest import assert_parity, mean_power
    C, n = 20, 1 << 17
    cfg = cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=256, lag_spec=cyc.LagSpec.Explicit(range(32)),
                              flags=cyc.Flags.BOTH, emit_frames=False, channels=C)
    xs = np.stack([rand_c(n, 40 + c) for c in range(C)])
    est, host = cyc.CyclicCorrelator(cfg), cyc.CyclicCorrelator(cfg)
    d = dev(xs)
    p = cyc.host_alloc(xs.shape)
    p[:] = xs
    for rep in range(3):  # direct, captured and replayed pushes
        est.reset()
        est.push_device(d.data_ptr(), n)
        got = est.average_all()
        if rep == 0:
            host.push(p)
            want = host.average_all()
            first = got
        assert np.array_equal(got, first)
    for c in (0, 17, 19):
        for fl in range(2):
            assert_parity(got[c, fl], want[c, fl], mean_power(xs[c]), rel_l2=1e-5, what=f"ch {c} flag {fl}")
    bad = xs.copy()
    bad[18, 70_000] = np.nan
    bad[3, 90_000] = np.inf
    est.reset()
    db = dev(bad)
    with pytest.raises(cyc.DataError, match="index 70000 in x stream of channel 18"):
        est.push_device(db.data_ptr(), n)
    assert est.consumed() == 0
    est.push_device(d.data_ptr(), n)  # the state was untouched: same tables as before
    assert np.array_equal(est.average_all(), first)
