"""Multi-GPU sharding plans for the cyclic-ACF path.

* time shards (one record, strong scaling): GPU g folds frames
  [F*g/G, F*(g+1)/G) of the global frame grid from an estimator created with
  origin = first_frame * win_len (its phases stay anchored to absolute sample
  0, estimator.hpp:87-93), pushing only its samples plus the lag halo; the
  per-GPU fold accumulators are then summed (NCCL all-reduce of
  channels x t_pad x Pf x 4 fp64 -- 2 MiB at C2, 64 MiB at C5) and the frame
  counts added.  Exact: the coherent average is linear in the frames.
* channel shards (C4): independent streams; the (channel, flag) tables are
  all-gathered at the end (no collective on the data path).
* replicas (C1, C3: the small-call paths do not shard): every GPU its own record.

With one channel and the lag list 0..T-1, the bench reduce-scatters the states
by lag rows instead (exchange_lag_slices: each GPU then finalizes only its
T/G lags) and all-gathers the tables (gather_lag_tables).

The exchange steps below are what bench.py runs between the push and the
finalize; they take any estimator-like object with fold_tensor(),
fold_set_frames() (time shards) and any torch.distributed group (NCCL on the
GPUs; gloo in the CPU tests, tests/test_shard.py).
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class TimeShard:
    rank: int
    frame0: int      # first global frame of the shard
    frame1: int      # one past the last
    sample0: int     # first absolute sample the shard pushes (= origin)
    sample1: int     # one past the last sample it needs

    @property
    def frames(self) -> int:
        return self.frame1 - self.frame0

    @property
    def origin(self) -> int:
        return self.sample0


def frames_total(L: int, win_len: int, m_plus: int, m_minus: int) -> int:
    """Emission rule of the reference (proj/src/estimator.cpp:20, test_estimator.cpp:202-204)."""
    need = win_len + m_plus + m_minus
    return (L - need) // win_len + 1 if L >= need else 0


def time_shards(L: int, win_len: int, m_plus: int, m_minus: int, world: int) -> list:
    F = frames_total(L, win_len, m_plus, m_minus)
    out = []
    for r in range(world):
        f0, f1 = F * r // world, F * (r + 1) // world
        # frame f covers x over [f*N, f*N + N + m_plus + m_minus)
        s0 = f0 * win_len
        s1 = f1 * win_len + m_plus + m_minus if f1 > f0 else s0
        out.append(TimeShard(r, f0, f1, s0, s1))
    return out


def channel_shards(channels: int, world: int) -> list:
    """Contiguous channel ranges per rank."""
    return [(channels * r // world, channels * (r + 1) // world) for r in range(world)]


class DeviceArray:
    """Zero-copy view of a device buffer for torch/NCCL (__cuda_array_interface__)."""

    def __init__(self, ptr: int, count: int, typestr: str = "<f8"):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def exchange_time_shards(est, frames_total: int, dist, group=None):
    """Time shards: sum every rank's fp64 fold state in place (all-reduce) and
    set the record's frame count -- afterwards each rank's average() is the
    whole record's (the states are indexed by absolute residue, so no phase
    re-anchoring is needed).  Returns the summed state tensor."""
    t = est.fold_tensor()  # synchronizes the estimator's fold before the collective reads it
    dist.all_reduce(t, group=group)
    est.fold_set_frames(frames_total)
    return t


def lag_slice(T: int, world: int, rank: int):
    """Contiguous lag range [t0, t1) of the lag list owned by `rank`."""
    return T * rank // world, T * (rank + 1) // world


def exchange_lag_slices(est, frames_total: int, T: int, t_pad: int, world: int, rank: int, dist, group=None):
    """Time shards, lag-sliced: reduce-scatter the fp64 fold states by lag rows
    (rank r ends up with the whole record's state for its lags T r/G .. T (r+1)/G
    only -- each rank sends and receives (G-1)/G of one slice instead of an
    all-reduce's two passes over the whole state) and point the estimator's
    finalize at that slice (set_lag_slice), so each rank transforms 1/G of the
    tables.  Needs one channel, the lag list 0..T-1 with T == t_pad (state rows =
    lags) and T % G == 0; otherwise the states are all-reduced and every lag is
    finalized.  Backends without a reduce-scatter (gloo) all-reduce instead --
    the same sums.  Returns the rank's lag range [t0, t1)."""
    if world == 1 or T != t_pad or T % world or est_channels(est) != 1:
        exchange_time_shards(est, frames_total, dist, group)
        return 0, T
    t0, t1 = lag_slice(T, world, rank)
    t = est.fold_tensor()  # [t_pad][Pf][4] for one channel
    mine = t.view(t_pad, -1)[t0:t1].reshape(-1)
    try:
        dist.reduce_scatter_tensor(mine, t, group=group)
    except (RuntimeError, AttributeError, NotImplementedError, ValueError):
        dist.all_reduce(t, group=group)
    est.fold_set_frames(frames_total)
    est.set_lag_slice(t0, t1)
    return t0, t1


def est_channels(est) -> int:
    cfg = getattr(est, "_cfg", None)
    return getattr(cfg, "channels", 1) if cfg is not None else getattr(est, "channels", 1)


def gather_lag_tables(out, t0: int, t1: int, T: int, world: int, dist, group=None):
    """All-gather the lag slices of a Full-mode table [1, flags, T * N]
    (lag-major) in place: rank r contributes rows [T r/G, T (r+1)/G)."""
    if world == 1:
        return out
    import torch
    flags = out.shape[1]
    n = out.shape[2] // T
    for f in range(flags):
        full = out[0, f].view(T, n)
        local = full[t0:t1].contiguous()
        try:
            dist.all_gather_into_tensor(full.view(-1), local.view(-1), group=group)
        except (RuntimeError, AttributeError, ValueError):
            parts = [torch.empty_like(local) for _ in range(world)]
            dist.all_gather(parts, local, group=group)
            full.copy_(torch.cat(parts))
    return out


def gather_channel_tables(local, world: int, dist, group=None):
    """Channel shards: all-gather [channels/world, flags, layout] tables into
    [channels, flags, layout] (rank order = channel order)."""
    import torch
    if world == 1:
        return local
    out = torch.empty((world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    try:
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
    except (RuntimeError, AttributeError):  # backends without the fused form
        parts = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(parts, local.contiguous(), group=group)
        out = torch.cat(parts)
    return out
