"""The N>1 data path with the device kernels (GPU): two ranks (processes),
each simulating its own scenario shard on the device with the real kernels
(Env.from_stress shard, fused step+observe rollout, k_episode_stats,
recorded rollout + k_episode_metrics), then the rollout exchange over a gloo
group -- the int64 stats all-reduce and the rank-ordered all-gather of the
fp64 metric partial sums.  The result must equal one process simulating the
whole batch: stats bit-exact, aggregate identical to the rank-ordered sum.

Only one GPU exists here, so both ranks share it; their kernels never wait on
each other (the only exchange is host-side gloo).  NCCL itself is exercised
by tests/test_gpu_comm.py (one rank) and bench.py at N > 1 on a multi-GPU box.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOTAL, STEPS = 24, 40
SHAPE = dict(agents=20, road_points=700)


def _shard_run(lo: int, hi: int):
    import torch

    import paper_2312_15122_b200 as z
    env = z.Env.from_stress(z.StressConfig(count=hi - lo, first_index=lo, **SHAPE), 7,
                            config=z.SimConfig(disable_dones=False))
    A, S = z.random_actions(STEPS, TOTAL, seed=11)
    dA = torch.from_numpy(np.ascontiguousarray(A[:, lo:hi])).cuda()
    dS = torch.from_numpy(np.ascontiguousarray(S[:, lo:hi])).cuda()
    s0, s1, so, ob = env.device_state(), env.device_state(), env.device_stepout(), env.device_obs()
    env.reset_device(42, s0)
    for t in range(STEPS):
        env.step_observe_device(s0, dA[t].data_ptr(), dS[t].data_ptr(), s1, so, ob)
        s0, s1 = s1, s0
    stats = torch.zeros(8, dtype=torch.int64, device="cuda")
    env.episode_stats(s0, stats.data_ptr())
    # recorded rollout of the same shard -> per-GPU metric partial sums
    ep = env.device_episode(STEPS)
    env.rollout_device(42, STEPS, dA.data_ptr(), dS.data_ptr(), STEPS, episode=ep)
    _, sums = env.episode_metrics(ep, rows=False)
    torch.cuda.synchronize()
    return stats.cpu(), sums


def _worker(rank: int, world: int, port: int, q) -> None:
    import torch
    import torch.distributed as dist

    from paper_2312_15122_b200.shard import allreduce_stats, gather_metric_sums, shard_rows
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard_rows(TOTAL, world, rank)
        stats, sums = _shard_run(lo, hi)
        allreduce_stats(stats)
        parts = gather_metric_sums(torch.as_tensor(np.asarray(sums), dtype=torch.float64))
        q.put((rank, (stats.numpy().tolist(), parts.tolist())))
    finally:
        dist.destroy_process_group()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_device_shards_equal_single_process():
    import torch.multiprocessing as mp

    import paper_2312_15122_b200 as z
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want_stats, want_sums = _shard_run(0, TOTAL)
    assert got[0][0] == want_stats.numpy().tolist() and got[1][0] == got[0][0]
    assert got[0][1] == got[1][1]
    agg = z.aggregate_finalize(np.array(got[0][1]))
    whole = z.aggregate_finalize(np.asarray(want_sums)[None, :])
    assert agg["scenarios"] == whole["scenarios"] == TOTAL
    for k in agg:
        assert abs(agg[k] - whole[k]) <= 1e-12 * max(1.0, abs(whole[k])), (k, agg[k], whole[k])
