"""Multi-GPU plumbing: scenario sharding and the episode-stats all-reduce.

The batch is sharded, not split by any data-path collective:
rank r of N simulates the contiguous rows [lo, hi) of the global scenario
set.  The only cross-GPU exchange is one all-reduce (sum) of the int64
episode-stats vector per rollout; integer sums are exact, so the result does
not depend on the reduction order (the fixed-order contract of the
reference's AllReducer, transport.hpp:59-61).
"""
from __future__ import annotations

import numpy as np

STATS_FIELDS = ("rows", "done", "collision", "off_route", "red_light", "stop_line", "goal_reached",
                "progress_sum_um")


def shard_rows(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous slice of `total` rows owned by `rank` (sizes differ by <= 1)."""
    if not (0 <= rank < world) or total < 0:
        raise ValueError("bad shard request")
    lo = total * rank // world
    hi = total * (rank + 1) // world
    return lo, hi


def stats_from_host_state(events: np.ndarray, done: np.ndarray, proj_s: np.ndarray,
                          initial_s: np.ndarray) -> np.ndarray:
    """Host statement of the int64 episode-stats vector that the device
    kernel k_episode_stats produces (zsim_episode_stats in include/zsim_gpu.h)."""
    ev = events.astype(np.int64)
    out = np.zeros(len(STATS_FIELDS), np.int64)
    out[0] = len(events)
    out[1] = int((done != 0).sum())
    for k in range(5):
        out[2 + k] = int(((ev >> k) & 1).sum())
    out[7] = int(np.rint((proj_s - initial_s) * 1e6).astype(np.int64).sum())
    return out


def allreduce_stats(stats, group=None):
    """Sum a stats vector (torch int64 tensor) over all ranks in place."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=group)
    return stats
