"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 host path:
contiguous scenario shards generated in closed form per global index, each
rank simulating its shard (with the C restatement standing in for the device
on this CPU-only box), and the int64 episode-stats all-reduce.  The result
must equal the single-process statistics of the whole batch exactly."""
from __future__ import annotations

import os
import socket

import numpy as np
import torch.multiprocessing as mp

import paper_2312_15122_b200 as z
from paper_2312_15122_b200.shard import (allreduce_stats, gather_metric_sums, metric_sums_host, shard_rows,
                                         stats_from_host_state)

TOTAL, STEPS = 10, 25
SHAPE = dict(agents=6, road_points=200, lane_vertices=20)


def _simulate(lo: int, hi: int) -> np.ndarray:
    from oracle import portpy
    zsim = z.stress_scenarios(z.StressConfig(count=hi - lo, first_index=lo, **SHAPE), seed=5)
    env = portpy.PortEnv(zsim, config=z.SimConfig(disable_dones=True))
    A, S = z.random_actions(STEPS, TOTAL, seed=17)
    st = env.init_state(42)
    for t in range(STEPS):
        st, _ = env.step(st, A[t, lo:hi], S[t, lo:hi])
    _, init_s, _ = env.scalars()
    return stats_from_host_state(st.events, st.done, st.proj_s, init_s)


def _worker(rank: int, world: int, port: int, q) -> None:
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_rows(TOTAL, world, rank)
    stats = torch.from_numpy(_simulate(lo, hi))
    allreduce_stats(stats)
    # metric partial sums: dyadic per-rank values, gathered in rank order
    sums = torch.full((12,), float(rank + 1) * 0.25, dtype=torch.float64)
    parts = gather_metric_sums(sums)
    q.put((rank, (stats.numpy().tolist(), parts.tolist())))
    dist.destroy_process_group()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_rows_partition():
    for total in (0, 1, 7, 4096, 131072):
        for world in (1, 2, 3, 8):
            spans = [shard_rows(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def test_sharded_generation_concatenates_to_global_set():
    from tests.zsim_py import read_zsim
    full = read_zsim(z.stress_scenarios(z.StressConfig(count=TOTAL, **SHAPE), seed=5))
    parts = []
    for r in range(3):
        lo, hi = shard_rows(TOTAL, 3, r)
        parts += read_zsim(z.stress_scenarios(z.StressConfig(count=hi - lo, first_index=lo, **SHAPE), seed=5))
    assert [s["id"] for s in full] == [s["id"] for s in parts]
    assert all(np.array_equal(a["ego"]["x"], b["ego"]["x"]) for a, b in zip(full, parts))


def test_two_rank_gloo_stats_allreduce_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = _simulate(0, TOTAL).tolist()
    assert got[0][0] == want and got[1][0] == want
    assert want[0] == TOTAL
    # every rank sees the same rank-ordered metric partials
    assert got[0][1] == got[1][1] == [[0.25] * 12, [0.5] * 12]
    assert z.aggregate_finalize(np.array(got[0][1]))["scenarios"] == 0.75


def test_metric_sums_host_matches_reference_aggregate():
    from oracle import refpy
    if not refpy.available():
        import pytest
        pytest.skip("oracle/_ref not built")
    zsim = z.stress_scenarios(z.StressConfig(count=8, **SHAPE), seed=5)
    A, S = z.random_actions(40, 8, seed=3)
    ep = refpy.RefEnv(zsim, config=z.SimConfig(disable_dones=False)).rollout(40, A.T, S.T, 42)
    sums = metric_sums_host(ep["s"], ep["a_lat"], ep["a_lon"], ep["mask"], ep["events"], ep["initial_s"],
                            ep["logged_progress"], 0.1)
    got = z.aggregate_finalize(sums)
    ref = refpy.aggregate(ep["s"], ep["a_lat"], ep["a_lon"], ep["mask"], ep["events"], ep["initial_s"],
                          ep["logged_progress"], 0.1)
    for k, v in enumerate(got.values()):
        assert abs(v - ref[k]) <= 1e-12 * max(1.0, abs(ref[k])), (k, v, ref[k])
