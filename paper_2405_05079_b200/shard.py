"""Landmark sharding for multi-GPU runs.

Each rank owns a contiguous landmark range with (nearly) equal observation
counts; cameras are replicated.  Per power-series term the camera-sized
partial S'.v vectors are summed with one NCCL allreduce inside libpovar.so
(n_p x 12 fp64); per LM iteration U/b_p, costs and flags are allreduced as
well, so every rank takes identical accept/reject and stop decisions.

The reference has no distributed path; this module is
the host-side plan + NCCL id plumbing.  ``torch.distributed`` (gloo) carries
the control plane (id broadcast, barriers, timing max); NCCL carries the data.
"""

from __future__ import annotations

import numpy as np


def plan_shards(problem, world: int) -> list[tuple[int, int]]:
    """Split [0, n_l) into ``world`` contiguous ranges of ~equal observation count.

    Boundaries are the landmark prefix-sum positions closest to k/world of the
    total; every rank gets a (possibly empty) range and the ranges tile
    [0, n_l) exactly.
    """
    if world < 1:
        raise ValueError("world must be >= 1")
    n_l = problem.num_landmarks
    counts = np.bincount(np.asarray(problem.landmark_indices, dtype=np.int64), minlength=n_l)
    prefix = np.concatenate([[0], np.cumsum(counts)])
    total = int(prefix[-1])
    bounds = [0]
    for k in range(1, world):
        target = total * k / world
        j = int(np.searchsorted(prefix, target, side="left"))
        if j > 0 and abs(prefix[j - 1] - target) <= abs(prefix[min(j, n_l)] - target):
            j -= 1
        bounds.append(min(max(j, bounds[-1]), n_l))
    bounds.append(n_l)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def shard_observation_counts(problem, plan) -> list[int]:
    li = np.asarray(problem.landmark_indices, dtype=np.int64)
    return [int(((li >= b) & (li < e)).sum()) for b, e in plan]


def broadcast_nccl_id(rank: int, world: int) -> bytes:
    """Rank 0 creates the NCCL unique id; torch.distributed broadcasts it."""
    import torch.distributed as dist

    from . import _lib

    obj = [None]
    if rank == 0:
        buf = (b"\0" * 128)
        import ctypes
        raw = ctypes.create_string_buffer(128)
        _lib.check(_lib.load().pv_nccl_unique_id(raw))
        buf = raw.raw
        obj = [buf]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def loopback_id(world: int) -> bytes:
    """An in-process loopback communicator for ``world`` contexts on ONE device, each driven
    by its own host thread (``pv_loopback_id``): the sharded code path -- split camera
    kernels, replicated epilogue, collective flags -- without a multi-GPU node."""
    import ctypes

    from . import _lib
    raw = ctypes.create_string_buffer(128)
    _lib.check(_lib.load().pv_loopback_id(int(world), raw))
    return raw.raw


def merge_states(states, plan):
    """Whole-problem state from per-rank results: the (replicated) cameras of rank 0 and
    each rank's own landmark range [begin, end) (a rank's ``get_state`` only updates the
    landmarks it owns)."""
    from .types import ProjectiveState
    lms = np.array(states[0].landmarks, copy=True)
    for st, (b, e) in zip(states, plan):
        lms[b:e] = st.landmarks[b:e]
    return ProjectiveState(states[0].cameras, lms)
