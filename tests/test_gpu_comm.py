"""The C-ABI NCCL path (zsim_comm_*) on one GPU: a 1-rank
communicator's stats all-reduce and metric all-gather are identities, the
device stats of a rollout survive the exchange bit-exactly, and async errors
are surfaced (none here).  The multi-rank host logic is covered on CPU by
tests/test_multiprocess_gloo.py; only one GPU exists in this environment."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

import paper_2312_15122_b200 as z

pytestmark = pytest.mark.gpu


def test_comm_available_and_unique_id():
    assert z.lib.zsim_comm_available() == 1
    a, b = (C.c_uint8 * 128)(), (C.c_uint8 * 128)()
    assert z.lib.zsim_comm_unique_id(a) == 0 and z.lib.zsim_comm_unique_id(b) == 0
    assert bytes(a) != bytes(b)


def test_single_rank_stats_allreduce_and_gather():
    import torch

    from paper_2312_15122_b200.shard import StatsComm
    zsim = z.stress_scenarios(z.StressConfig(count=8, agents=8, road_points=300), 3)
    env = z.Env(zsim, config=z.SimConfig(disable_dones=True), device=0)
    A, S = z.random_actions(20, env.batch_size(), seed=4)
    dA, dS = torch.from_numpy(A).cuda(), torch.from_numpy(S).cuda()
    s0, s1, so, ob = env.device_state(), env.device_state(), env.device_stepout(), env.device_obs()
    env.reset_device(42, s0)
    for t in range(20):
        env.step_observe_device(s0, dA[t].data_ptr(), dS[t].data_ptr(), s1, so, ob)
        s0, s1 = s1, s0
    stats = torch.zeros(8, dtype=torch.int64, device="cuda")
    env.episode_stats(s0, stats.data_ptr())
    torch.cuda.synchronize()
    before = stats.cpu().numpy().copy()
    comm = StatsComm(0, 1, 0)
    try:
        comm.allreduce_stats(stats)
        torch.cuda.synchronize()
        comm.check()
        assert np.array_equal(stats.cpu().numpy(), before)
        sums = torch.arange(12, dtype=torch.float64, device="cuda") * 0.25
        g = comm.gather_metric_sums(sums)
        assert g.shape == (1, 12) and np.array_equal(g[0], np.arange(12) * 0.25)
    finally:
        comm.close()
    assert before[0] == env.batch_size()


def test_comm_rejects_bad_arguments():
    h = C.c_void_p()
    idb = (C.c_uint8 * 128)()
    assert z.lib.zsim_comm_init_rank(idb, 2, 5, 0, C.byref(h)) == 1  # rank >= nranks: invalid_argument
    assert z.lib.zsim_stats_allreduce(None, None, 8, None) == 1


def _python_stats(count, agents, points, steps, controlled=False):
    import torch
    env = z.Env.from_stress(z.StressConfig(count=count, agents=agents, road_points=points,
                                           flags=z.STRESS_C2 if controlled else 0), 7,
                            config=z.SimConfig(disable_dones=True), controlled=controlled)
    B = env.batch_size()
    A, S = z.random_actions(91, B, seed=123)
    dA, dS = torch.from_numpy(A).cuda(), torch.from_numpy(S).cuda()
    s0, s1, so, ob = env.device_state(), env.device_state(), env.device_stepout(), env.device_obs()
    for k in range(steps):
        if k % 91 == 0:
            env.reset_device(42, s0)
        env.step_observe_device(s0, dA[k % 91].data_ptr(), dS[k % 91].data_ptr(), s1, so, ob)
        s0, s1 = s1, s0
    stats = torch.zeros(8, dtype=torch.int64, device="cuda")
    env.episode_stats(s0, stats.data_ptr())
    torch.cuda.synchronize()
    return stats.cpu().tolist()


@pytest.mark.parametrize("controlled", [False, True])
def test_single_process_multi_gpu_driver(controlled):
    """csrc/zsim_multi_gpu.cpp (host C++ over the C-ABI: ncclCommInitAll, one
    thread + stream per GPU, stats all-reduce) on every visible GPU (one here):
    its all-reduced stats equal the Python device path over the same set."""
    import json
    import subprocess
    from pathlib import Path
    exe = Path(z.__file__).resolve().parent / "zsim_multi_gpu"
    assert exe.exists(), "build() compiles paper_2312_15122_b200/zsim_multi_gpu"
    args = ["20", "120", "16", "600", "1"] if controlled else ["64", "120", "24", "900", "0"]
    r = subprocess.run([str(exe), "1", *args], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    count, steps, agents, points = int(args[0]), int(args[1]), int(args[2]), int(args[3])
    assert out["ndev"] == 1 and out["steps"] == steps
    assert out["stats"] == _python_stats(count, agents, points, steps, controlled)
