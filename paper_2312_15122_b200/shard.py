"""Multi-GPU plumbing: scenario sharding, the episode-stats all-reduce and the
episode-metrics gather.

The batch is sharded, not split by any data-path collective:
rank r of N simulates the contiguous rows [lo, hi) of the global scenario
set.  The only cross-GPU exchange is one all-reduce (sum) of the int64
episode-stats vector per rollout; integer sums are exact, so the result does
not depend on the reduction order (the fixed-order contract of the
reference's AllReducer, transport.hpp:59-61).  The fp64 metric sums
(zsim_episode_metrics) are all-gathered instead and summed in rank order, so
the aggregate is reproducible for a given sharding.
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


def metric_sums_host(s: np.ndarray, a_lat: np.ndarray, a_lon: np.ndarray, mask: np.ndarray, events: np.ndarray,
                     initial_s: np.ndarray, logged: np.ndarray, dt: float, bounds=(0.8, 0.05, 0.5, 0.5, 0.5, 0.8),
                     w_accel: float = 0.1, w_jerk: float = 0.05) -> np.ndarray:
    """Host statement of zsim_episode_metrics' Aggregate partial sums
    (metrics::score_episode, metrics.cpp:54-95, summed over rows in order)."""
    out = np.zeros(12)
    B, T = s.shape
    for b in range(B):
        lg = float(logged[b])
        live_t = np.nonzero(mask[b])[0]
        init = float(initial_s[b])
        final_s = float(s[b, live_t[-1]]) if len(live_t) else init
        if lg <= 0.1:
            out[1] += 1
            continue
        raw = (final_s - init) / lg
        rel = min(max(raw, 0.0), 1.0)
        ev = int(events[b])
        coll, off, light, stop = [0.0 if ev & m else 1.0 for m in (1, 2, 4, 8)]
        acc, live, prev = 0.0, 0, None
        for t in range(T):
            if not mask[b, t]:
                break
            al, ao = float(a_lat[b, t]), float(a_lon[b, t])
            jl = jo = 0.0
            if prev is not None:
                jl, jo = (al - prev[0]) / dt, (ao - prev[1]) / dt
            acc += w_accel * (al * al + ao * ao) + w_jerk * (jl * jl + jo * jo)
            prev, live = (al, ao), live + 1
        comfort = 1.0 if live == 0 else float(np.exp(-acc / live))
        score = 1.0
        for v, l in zip((rel, coll, off, stop, light, comfort), bounds):
            score *= v * (1.0 - l) + l
        out += [1, 0, score, rel, raw, coll, off, stop, light, comfort, 1.0 if (coll == 0 or off == 0) else 0.0,
                1.0 if ev & 16 else 0.0]
    return out


def gather_metric_sums(sums, group=None) -> np.ndarray:
    """All-gather every rank's fp64 metric partial sums (torch tensor [12]);
    returns [world][12] in rank order for aggregate_finalize."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return sums.detach().cpu().numpy()[None, :]
    parts = [torch.zeros_like(sums) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, sums, group=group)
    return np.stack([p.cpu().numpy() for p in parts])


class StatsComm:
    """The C-ABI NCCL communicator (zsim_comm_*, include/zsim_gpu.h) used for
    the one per-rollout exchange: the int64 stats all-reduce and the fp64
    metric-sums all-gather.  The 128-byte NCCL id is made by rank 0 and
    broadcast over the caller's torch.distributed group (plumbing only)."""

    def __init__(self, rank: int, world: int, device: int):
        import ctypes as C

        import torch.distributed as dist

        from ._abi import check, lib
        self._lib, self._check, self.rank, self.world = lib, check, rank, world
        idb = (C.c_uint8 * 128)()
        if rank == 0:
            check(lib.zsim_comm_unique_id(idb))
        obj = [bytes(idb)]
        if dist.is_available() and dist.is_initialized() and world > 1:
            dist.broadcast_object_list(obj, src=0)
        idb = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        h = C.c_void_p()
        check(lib.zsim_comm_init_rank(idb, int(world), int(rank), int(device), C.byref(h)))
        self.handle = h.value

    def allreduce_stats(self, stats, stream=None):
        """In place over a torch int64 device tensor."""
        import ctypes as C
        from .env import _stream
        self._check(self._lib.zsim_stats_allreduce(self.handle, C.cast(stats.data_ptr(), C.POINTER(C.c_int64)),
                                                   int(stats.numel()), _stream(stream)))
        return stats

    def gather_metric_sums(self, sums, stream=None) -> np.ndarray:
        """[world][n] fp64 in rank order from every rank's device sums[n]."""
        import ctypes as C

        import torch
        from .env import _stream
        out = torch.zeros(self.world * sums.numel(), dtype=torch.float64, device=sums.device)
        self._check(self._lib.zsim_metric_sums_allgather(
            self.handle, C.cast(sums.data_ptr(), C.POINTER(C.c_double)), int(sums.numel()),
            C.cast(out.data_ptr(), C.POINTER(C.c_double)), _stream(stream)))
        torch.cuda.synchronize(sums.device)
        return out.cpu().numpy().reshape(self.world, -1)

    def check(self) -> None:
        """Surface an NCCL asynchronous error (ncclCommGetAsyncError)."""
        self._check(self._lib.zsim_comm_check(self.handle))

    def close(self) -> None:
        if getattr(self, "handle", None):
            self._lib.zsim_comm_destroy(self.handle)
            self.handle = None
