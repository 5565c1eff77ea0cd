"""Multi-GPU plans on CPU: world_size-2 gloo runs of the time-sharded block
average (the exchange step is a sum all-reduce of per-shard folds) against the
whole-record oracle, plus the pure plan invariants."""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import rand_c

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_time_shards_cover_the_frame_grid():
    from paper_2405_16911_b200.shard import frames_total, time_shards
    for L, N, mp_, mm, W in [(1 << 20, 1024, 63, 0, 8), (100_000, 256, 31, 0, 3), (5000, 64, 3, 3, 2), (10, 64, 0, 0, 4)]:
        F = frames_total(L, N, mp_, mm)
        sh = time_shards(L, N, mp_, mm, W)
        assert sum(s.frames for s in sh) == F
        assert sh[0].frame0 == 0 and sh[-1].frame1 == F
        for a, b in zip(sh, sh[1:]):
            assert a.frame1 == b.frame0
        for s in sh:
            assert s.sample1 <= L
            if s.frames:  # the shard's own emission rule yields exactly its frames
                assert frames_total(s.sample1 - s.sample0, N, mp_, mm) == s.frames


def test_channel_shards():
    from paper_2405_16911_b200.shard import channel_shards
    sh = channel_shards(64, 3)
    assert sh[0][0] == 0 and sh[-1][1] == 64 and sum(b - a for a, b in sh) == 64


class FoldModel:
    """CPU model of a block-mode estimator's fold state in the product's layout
    ([channel][lag][residue][xr*yr, xi*yr, xr*yi, xi*yi], residues of ABSOLUTE
    sample indices -- what cyc_fold_state exposes, include/cycb200.h), for a
    time shard whose first sample is absolute index `origin`."""

    def __init__(self, x_local, origin, N, lags, frames):
        import torch
        self.N, self.T = N, len(lags)
        n = frames * N
        y = x_local[:n].astype(np.complex128)
        r = (origin + np.arange(n)) % N  # absolute residues: the shards sum without re-anchoring
        S = np.zeros((self.T, N, 4))
        for ti, lag in enumerate(lags):
            xs = x_local[lag:lag + n].astype(np.complex128)
            for comp, v in enumerate((xs.real * y.real, xs.imag * y.real, xs.real * y.imag, xs.imag * y.imag)):
                S[ti, :, comp] = np.bincount(r, weights=v, minlength=N)
        self.S = torch.from_numpy(S.reshape(-1).copy())
        self.frames = frames

    def fold_tensor(self):
        return self.S

    def fold_set_frames(self, frames):
        self.frames = frames

    def set_lag_slice(self, begin=0, end=0):
        self.lag_slice = (begin, end)

    def tables(self, bins):
        """Coherent averages (conv, conj) [bins, lags] from the fold state."""
        S = self.S.numpy().reshape(self.T, self.N, 4)
        conv = (S[..., 0] + S[..., 3]) + 1j * (S[..., 1] - S[..., 2])  # x * conj(y)
        conj = (S[..., 0] - S[..., 3]) + 1j * (S[..., 1] + S[..., 2])  # x * y
        w = np.exp(-2j * np.pi * np.outer(bins, np.arange(self.N)) / self.N)
        scale = 1.0 / (self.frames * self.N)
        return (w @ conv.T) * scale, (w @ conj.T) * scale


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    from paper_2405_16911_b200.shard import exchange_time_shards, gather_channel_tables, time_shards
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x = rand_c(1 << 16, 5)
    N, lags = 512, list(range(16))
    sh = time_shards(len(x), N, 15, 0, world)[rank]
    # each rank sees ONLY its samples; absolute indices are carried by `origin`
    m = FoldModel(x[sh.sample0:sh.sample1], sh.origin, N, lags, sh.frames)
    F = sum(s.frames for s in time_shards(len(x), N, 15, 0, world))
    exchange_time_shards(m, F, dist)  # the product's exchange step (bench.py)
    bins = np.array([0, 1, 5, 100, 255, 256, 511])
    cv, cj = m.tables(bins)
    # channel shards: 6 channels, 3 per rank, tables gathered in channel order
    chans = [rank * 3 + c for c in range(3)]
    local = torch.from_numpy(np.stack([np.full((2, 4), float(c)) + 1j * c for c in chans]))
    full = gather_channel_tables(local, world, dist)
    if rank == 0:
        q.put((cv, cj, m.frames, full.numpy()))
    dist.destroy_process_group()


def test_gloo_time_shard_exchange_equals_whole_record():
    """world-2 gloo run of shard.exchange_time_shards (the bench's NCCL step)
    over per-shard fold states: equals the whole record's oracle tables."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    cv, cj, F, full = q.get()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from oracle.oracle import Oracle
    o = Oracle()
    x = rand_c(1 << 16, 5)
    bins = np.array([0, 1, 5, 100, 255, 256, 511])
    wv, wj = o.block_fold(x, x, bins, 512, list(range(16)), 0, F * 512)
    assert np.max(np.abs(cv - wv)) <= 1e-12
    assert np.max(np.abs(cj - wj)) <= 1e-12
    assert full.shape == (6, 2, 4)
    assert np.array_equal(full.real[:, 0, 0], np.arange(6.0))


def _worker_lags(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    from paper_2405_16911_b200.shard import exchange_lag_slices, gather_lag_tables, time_shards
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x = rand_c(1 << 16, 7)
    N, T = 256, 16
    sh = time_shards(len(x), N, T - 1, 0, world)[rank]
    m = FoldModel(x[sh.sample0:sh.sample1], sh.origin, N, list(range(T)), sh.frames)
    F = sum(s.frames for s in time_shards(len(x), N, T - 1, 0, world))
    t0, t1 = exchange_lag_slices(m, F, T, T, world, rank, dist)  # the bench's exchange step
    assert (t0, t1) == (T * rank // world, T * (rank + 1) // world) and m.lag_slice == (t0, t1)
    cv, cj = m.tables(np.arange(N))  # [bins, lags]
    # Full-mode tables [1, flags, T * N] (lag-major): this rank fills only its
    # finalized slice (the rest NaN), then the lag slices are all-gathered
    out = torch.full((1, 2, T * N), float("nan"), dtype=torch.complex128)
    for f, tab in enumerate((cv, cj)):
        rows = out[0, f].view(T, N)
        rows[t0:t1] = torch.from_numpy(np.ascontiguousarray(tab.T[t0:t1]))
    gather_lag_tables(out, t0, t1, T, world, dist)
    if rank == 0:
        q.put((out.numpy(), m.frames))
    dist.destroy_process_group()


def test_gloo_lag_slice_exchange_and_gather_equal_whole_record():
    """world-2 gloo run of shard.exchange_lag_slices (reduce-scatter by lag rows;
    gloo takes the all-reduce branch) + gather_lag_tables: the assembled
    tables equal the whole record's oracle tables for every lag."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = 30500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker_lags, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out, F = q.get()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from oracle.oracle import Oracle
    x = rand_c(1 << 16, 7)
    N, T = 256, 16
    wv, wj = Oracle().block_fold(x, x, np.arange(N), N, list(range(T)), 0, F * N)
    for f, want in ((0, wv), (1, wj)):
        got = out[0, f].reshape(T, N)
        assert not np.isnan(got).any()
        assert np.max(np.abs(got - want.T)) <= 1e-12


def test_lag_slice_plan():
    from paper_2405_16911_b200.shard import lag_slice
    for T, W in [(256, 8), (64, 4), (30, 4)]:
        sl = [lag_slice(T, W, r) for r in range(W)]
        assert sl[0][0] == 0 and sl[-1][1] == T and all(a[1] == b[0] for a, b in zip(sl, sl[1:]))


@pytest.mark.gpu
def test_lag_slice_finalize_matches_full_average(cyc):
    """cyc_set_lag_slice: average_all finalizes only the slice's lags (device and
    host outputs), the other rows untouched, the slice's rows equal to the full
    average; (0, 0) restores every lag."""
    import torch
    x = rand_c(1 << 20, 8)
    N, T = 1024, 64
    est = cyc.CyclicCorrelator(cyc.EstimatorConfig(mode=cyc.Mode.Full, win_len=N, lag_spec=cyc.LagSpec.Explicit(range(T)),
                                                   flags=cyc.Flags.BOTH, emit_frames=False))
    est.push(x)
    full = est.average_all()  # [1, 2, T * N]
    for t0, t1 in [(16, 32), (0, 8), (48, 64)]:
        est.set_lag_slice(t0, t1)
        host = np.full_like(full, np.nan)
        est.average_all(out=host)
        dev = torch.full(full.shape, float("nan"), dtype=torch.complex128, device="cuda")
        est.average_all(out=dev)
        torch.cuda.synchronize()
        for got in (host, dev.cpu().numpy()):
            g = got.reshape(2, T, N)
            f = full.reshape(2, T, N)
            assert np.array_equal(g[:, t0:t1], f[:, t0:t1])
            assert np.isnan(np.delete(g, np.s_[t0:t1], axis=1)).all()
    est.set_lag_slice(0, 0)
    assert np.array_equal(est.average_all(), full)
    with pytest.raises(Exception):
        est.set_lag_slice(10, 70)


@pytest.mark.gpu
def test_lag_slice_finalize_set_mode_alpha_major(cyc):
    """The lag slice in the alpha-major Set layout ([alpha][lag]): the host copy
    is a strided column band; rows of other lags untouched."""
    x = rand_c(1 << 18, 9)
    alphas = [k / 64 for k in range(-8, 8)]
    est = cyc.CyclicCorrelator(cyc.EstimatorConfig(mode=cyc.Mode.Set, win_len=256, alphas=alphas,
                                                   lag_spec=cyc.LagSpec.Symmetric(7), flags=cyc.Flags.BOTH,
                                                   emit_frames=False))
    est.push(x)
    full = est.average_all()  # [1, 2, A * (2M + 1)] alpha-major
    A, T = len(alphas), 15
    est.set_lag_slice(3, 9)
    host = np.full_like(full, np.nan)
    est.average_all(out=host)
    g, f = host.reshape(2, A, T), full.reshape(2, A, T)
    assert np.array_equal(g[:, :, 3:9], f[:, :, 3:9])
    assert np.isnan(g[:, :, :3]).all() and np.isnan(g[:, :, 9:]).all()


@pytest.mark.gpu
def test_time_shards_on_device_sum_to_whole_record(cyc):
    """Single-GPU emulation of the NCCL exchange: per-shard estimators with
    origin, fold states summed with torch, frames added."""
    import torch
    from paper_2405_16911_b200.shard import DeviceArray, time_shards
    x = rand_c(1 << 20, 6)
    N, lags = 1024, list(range(64))
    mk = lambda origin: cyc.CyclicCorrelator(cyc.EstimatorConfig(
        mode=cyc.Mode.Full, win_len=N, lag_spec=cyc.LagSpec.Explicit(lags), flags=cyc.Flags.BOTH,
        emit_frames=False, origin=origin))
    whole = mk(0)
    whole.push(x)
    shards = time_shards(len(x), N, 63, 0, 4)
    ests = []
    for s in shards:
        e = mk(s.origin)
        e.push(x[s.sample0:s.sample1])
        assert e.frames_emitted() == s.frames
        ests.append(e)
    ptr0, n0, _ = ests[0].fold_state()
    acc = torch.as_tensor(DeviceArray(ptr0, n0), device="cuda")
    for e in ests[1:]:
        p, n, _ = e.fold_state()
        acc += torch.as_tensor(DeviceArray(p, n), device="cuda")
    torch.cuda.synchronize()
    ests[0].fold_set_frames(sum(s.frames for s in shards))
    # identical up to fp32 partial-sum grouping (tiles split the periods differently)
    for fl in (cyc.Flags.CONV, cyc.Flags.CONJ):
        a, b = ests[0].average(flag=fl), whole.average(flag=fl)
        assert np.linalg.norm(a - b) <= 1e-6 * np.linalg.norm(b)
        assert np.max(np.abs(a - b)) <= 1e-6 * 2.0  # mean power of x is 2; north star is 1e-5
