"""Pipelined emission (cyc_set_emit_pipeline / cyc_flush_frames): frames leave one
call later than under the reference's synchronous push() (estimator.cpp:59-82)
but are the same frames -- same order, indices, start_abs and values bit for
bit -- and still match the oracle."""
import numpy as np
import pytest

from conftest import assert_parity, mean_power, rand_c

pytestmark = pytest.mark.gpu


def run_stream(cyc, cfg, x, chunk, depth, y=None):
    est = cyc.CyclicCorrelator(cfg)
    est.set_emit_pipeline(depth)
    frames, per_push = [], []
    for o in range(0, len(x), chunk):
        got = est.push(x[o:o + chunk], None if y is None else y[o:o + chunk])
        per_push.append(len(got))
        frames += got
    tail = est.flush_frames()
    assert est.flush_frames() == []  # nothing left in flight
    return frames + tail, per_push, len(tail), est


def same_frames(a, b):
    assert len(a) == len(b) > 0
    for fa, fb in zip(a, b):
        assert (fa.frame_index, fa.start_abs, fa.flag, fa.channel) == (fb.frame_index, fb.start_abs, fb.flag, fb.channel)
        assert np.array_equal(np.asarray(fa.values), np.asarray(fb.values))


def test_recursive_small_calls_pipelined(cyc, oracle):
    # the C3 call pattern in miniature: E = 8 calls
    x = rand_c(40_000, 7)
    alphas = [m / 64 for m in range(-8, 8)]
    lags = list(range(8))
    lam, E = 1 - 2 ** -8, 4096
    cfg = cyc.EstimatorConfig(mode=cyc.Mode.Recursive, win_len=E, alphas=alphas,
                              lag_spec=cyc.LagSpec.Explicit(lags), lam=lam)
    sync, pp0, tail0, _ = run_stream(cyc, cfg, x, 512, 0)
    pipe, pp1, tail1, _ = run_stream(cyc, cfg, x, 512, 1)
    assert tail0 == 0
    same_frames(pipe, sync)
    same_frames(run_stream(cyc, cfg, x, 512, 2)[0], sync)
    # no pipelined push returns a frame earlier than the push that completes it
    assert all(sum(pp1[:i + 1]) <= sum(pp0[:i + 1]) for i in range(len(pp0)))
    want = oracle.recursive(x.astype(complex), x.astype(complex), alphas, lags, False, lam, E)
    got = np.array([f.values for f in pipe]).reshape(want.shape)
    assert_parity(got, want, mean_power(x), what="recursive pipelined")


@pytest.mark.parametrize("depth", [1, 2])
@pytest.mark.parametrize("chunk", [64, 100, 1000])
def test_set_frames_pipelined(cyc, oracle, chunk, depth):
    # the C1 call pattern: one Set frame per push (chunk == N), ragged and multi-frame pushes
    x = rand_c(3000, 11)
    y = rand_c(3000, 12)
    alphas = [3 / 64, 0.0, -0.21, 0.1234507]
    cfg = cyc.EstimatorConfig(mode=cyc.Mode.Set, win_len=64, alphas=alphas, lag_spec=cyc.LagSpec.Symmetric(3),
                              flags=cyc.Flags.BOTH)
    sync, _, _, e0 = run_stream(cyc, cfg, x, chunk, 0, y)
    pipe, _, _, e1 = run_stream(cyc, cfg, x, chunk, depth, y)
    same_frames(pipe, sync)
    for conj, flag in ((False, cyc.Flags.CONV), (True, cyc.Flags.CONJ)):
        want = oracle.stream(0, conj, 64, x.astype(complex), y.astype(complex), alphas=alphas, max_lag=3)
        got = np.array([f.values for f in pipe if f.flag == flag])
        assert_parity(got, want, mean_power(x) ** 0.5 * mean_power(y) ** 0.5, what="set pipelined")
        # the running average_frames sums do not depend on when frames are delivered
        assert np.array_equal(e0.average(cyc.AverageMode.Coherent, flag), e1.average(cyc.AverageMode.Coherent, flag))


def test_full_frames_pipelined_and_depth_switch(cyc):
    x = rand_c(1 << 13, 21)
    cfg = cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=256, lag_spec=cyc.LagSpec.Explicit([-2, 0, 3]))
    sync, _, _, _ = run_stream(cyc, cfg, x, 256, 0)
    est = cyc.CyclicCorrelator(cfg)
    est.set_emit_pipeline(1)
    frames = []
    for i, o in enumerate(range(0, len(x), 256)):
        if i == 10:
            est.set_emit_pipeline(0)  # the batch in flight is kept and delivered by the next push
        if i == 20:
            est.set_emit_pipeline(2)
        if i == 26:
            est.set_emit_pipeline(1)
        frames += est.push(x[o:o + 256])
    frames += est.flush_frames()
    same_frames(frames, sync)


def test_reset_drops_the_batch_in_flight(cyc):
    x = rand_c(1024, 3)
    cfg = cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=256, lag_spec=cyc.LagSpec.Explicit([0, 1]))
    est = cyc.CyclicCorrelator(cfg)
    est.set_emit_pipeline(1)
    first = est.push(x[:300])
    assert first == []  # enqueued, not delivered
    est.reset()
    assert est.flush_frames() == []
    again = est.push(x[:300]) + est.flush_frames()
    ref, _, _, _ = run_stream(cyc, cfg, x[:300], 300, 0)
    same_frames(again, ref)
    with pytest.raises(cyc.UsageError):
        est.set_emit_pipeline(3)


def test_c1_geometry_depth_two(cyc):
    # BASELINE C1's call pattern (4096-sample pushes, union alpha set, both flags): direct per-frame kernel
    x = rand_c(40 * 4096, 31)
    alphas = [k / 8 for k in range(-2, 3)] + [0.1 + k / 16 for k in range(-2, 3)]
    cfg = cyc.EstimatorConfig(mode=cyc.Mode.Set, win_len=4096, alphas=alphas, lag_spec=cyc.LagSpec.Symmetric(15),
                              flags=cyc.Flags.BOTH)
    sync, _, _, e0 = run_stream(cyc, cfg, x, 4096, 0)
    pipe, pp, tail, e2 = run_stream(cyc, cfg, x, 4096, 2)
    same_frames(pipe, sync)
    assert tail >= 2  # frames were still in flight at the end (both flags of at least one batch)
    assert np.array_equal(e0.average(cyc.AverageMode.Coherent, cyc.Flags.CONV),
                          e2.average(cyc.AverageMode.Coherent, cyc.Flags.CONV))


def test_direct_side_copy_growth_and_depth_switch(cyc):
    # depth-2 direct frames leave through a side-stream copy of alternating device tables:
    # growing batches reallocate those tables with copies in flight, depth switches move
    # between the side copy and the mapped stores, and a reset drops what is in flight
    x = rand_c(60 * 256, 41)
    alphas = [0.1234507, -0.3141, 1 / 7]
    cfg = cyc.EstimatorConfig(mode=cyc.Mode.Set, win_len=256, alphas=alphas, lag_spec=cyc.LagSpec.Symmetric(5),
                              flags=cyc.Flags.BOTH)
    sync = run_stream(cyc, cfg, x, 256, 0)[0]
    est = cyc.CyclicCorrelator(cfg)
    est.set_emit_pipeline(2)
    est.push(x[:700])
    est.reset()  # frames in flight belong to the old stream
    frames, o = [], 0
    sizes = [256, 256, 256, 512, 256, 1024, 256, 256, 2048, 300, 212, 256, 256]
    for i, n in enumerate(sizes * 2):
        if o + n > len(x):
            break
        if i == 5:
            est.set_emit_pipeline(1)
        if i == 8:
            est.set_emit_pipeline(2)
        if i == 14:
            est.set_emit_pipeline(0)
        if i == 16:
            est.set_emit_pipeline(2)
        frames += est.push(x[o:o + n])
        o += n
    frames += est.flush_frames()
    same_frames(frames, [f for f in sync if f.start_abs + 256 + 5 <= o])
