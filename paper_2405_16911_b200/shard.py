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
