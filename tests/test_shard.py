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


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    from oracle.oracle import Oracle
    from paper_2405_16911_b200.shard import time_shards
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle()
    x = rand_c(1 << 16, 5)
    N, lags = 512, list(range(16))
    sh = time_shards(len(x), N, 15, 0, world)[rank]
    # each rank sees ONLY its samples; absolute indices are carried by `origin`
    xs = x[sh.sample0:sh.sample1]
    cv, cj = o.block_fold(xs, xs, np.arange(N), N, lags, 0, sh.frames * N)
    # re-anchor: block_fold anchors phases at the local index; the engine uses origin
    k = np.arange(N)
    ph = np.exp(-2j * np.pi * (k * sh.origin % N) / N)[:, None]
    part = np.stack([cv * ph, cj * ph]) * (sh.frames * N)
    t = torch.from_numpy(part.view(np.float64).copy())
    dist.all_reduce(t)
    fr = torch.tensor([sh.frames], dtype=torch.float64)
    dist.all_reduce(fr)
    if rank == 0:
        q.put((t.numpy().view(np.complex128) / (fr.item() * N), int(fr.item())))
    dist.destroy_process_group()


def test_gloo_time_shard_allreduce_equals_whole_record():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, F = q.get()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from oracle.oracle import Oracle
    o = Oracle()
    x = rand_c(1 << 16, 5)
    cv, cj = o.block_fold(x, x, np.arange(512), 512, list(range(16)), 0, F * 512)
    assert np.max(np.abs(got[0] - cv)) <= 1e-12
    assert np.max(np.abs(got[1] - cj)) <= 1e-12


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
