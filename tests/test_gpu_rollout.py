"""Device rollout recording and episode metrics.

zsim_rollout = Env::rollout with the reference ScriptedPolicy
(simcore.cpp:554-618, 69-84) recorded into a device EpisodeBatch;
zsim_episode_metrics = metrics::score_episode + aggregate
(metrics.cpp:29-131).  Compared field by field with the reference compiled
in place (oracle/_ref): integer / flag fields bit-exact, fp fields within the
north_star tolerance, metrics within fp64 round-off (different summation
order, device exp)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2312_15122_b200 as z
from oracle import refpy

needs_ref = pytest.mark.skipif(not refpy.available(), reason="oracle/_ref not built")
RTOL, ATOL = 1e-5, 1e-6


def test_aggregate_finalize_sums_parts_in_order():
    parts = np.array([[3, 1, 1.5, 2.0, 2.2, 3, 2, 3, 3, 2.4, 1, 1], [1, 0, 0.5, 1.0, 1.0, 1, 1, 1, 0, 0.9, 0, 0]])
    a = z.aggregate_finalize(parts)
    t = parts.sum(0)
    assert a["scenarios"] == 4 and a["degenerate"] == 1
    assert a["mean_score"] == t[2] / 4 and a["failure_rate"] == t[10] / 4 and a["goal_rate"] == t[11] / 4
    assert z.aggregate_finalize(np.zeros(12))["mean_score"] == 0.0


def _device_rollout(env, horizon, A, S, seed=42, obs=False):
    import torch
    dA = torch.from_numpy(np.ascontiguousarray(A)).cuda()
    dS = torch.from_numpy(np.ascontiguousarray(S)).cuda()
    ep = env.device_episode(horizon)
    ob = [env.device_obs() for _ in range(horizon + 1)] if obs else None
    env.rollout_device(seed, horizon, dA.data_ptr(), dS.data_ptr(), A.shape[0], episode=ep, obs=ob)
    torch.cuda.synchronize()
    return ep, ob


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("src,dones_off,script", [("stress", True, 91), ("stress", False, 91), ("gen", False, 91),
                                                  ("stress", False, 40)])
def test_device_rollout_matches_reference_rollout(src, dones_off, script):
    zsim = z.stress_scenarios(z.StressConfig(count=16), 7) if src == "stress" else refpy.generate(16, seed=9)
    cfg = z.SimConfig(disable_dones=dones_off)
    env = z.Env(zsim, config=cfg)
    B = env.info.batch
    A, S = z.random_actions(script, B, seed=17)  # [script][B]; a short script ends in zero actions
    ep, _ = _device_rollout(env, 91, A, S)
    got = env.download_episode(ep)
    ref = refpy.RefEnv(zsim, config=cfg).rollout(91, A.T, S.T, 42)
    for f in ("accel_idx", "steer_idx", "done", "mask", "terminal", "events"):
        assert np.array_equal(got[f], ref[f]), f
    for f in ("logp", "value", "reward", "s", "a_lat", "a_lon", "v", "bootstrap", "initial_s", "logged_progress"):
        np.testing.assert_allclose(got[f], ref[f], rtol=RTOL, atol=ATOL, err_msg=f)
    if not dones_off:
        assert (ref["mask"] == 0).any()  # rows do terminate: masks and frozen t are exercised


@pytest.mark.gpu
def test_device_rollout_records_the_observations():
    zsim = z.stress_scenarios(z.StressConfig(count=8), 5)
    env = z.Env(zsim, config=z.SimConfig(disable_dones=False))
    A, S = z.random_actions(12, 8, seed=3)
    _, obs = _device_rollout(env, 12, A, S, obs=True)
    st = env.init_state(42)
    for t in range(13):
        want = env.observe(st)
        have = env.download_obs(obs[t])
        for f in ("active", "agents", "road", "route", "value_only"):
            assert np.array_equal(getattr(want, f), getattr(have, f)), (t, f)
        if t < 12:
            # ScriptedPolicy reads the script at each row's t (frozen once done)
            a = np.array([A[min(tt, 11)][b] for b, tt in enumerate(st.t)], dtype=np.int32)
            s = np.array([S[min(tt, 11)][b] for b, tt in enumerate(st.t)], dtype=np.int32)
            st, _ = env.step(st, a, s)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("dones_off", [True, False])
def test_device_metrics_match_reference(dones_off):
    zsim = z.stress_scenarios(z.StressConfig(count=32), 11)
    cfg = z.SimConfig(disable_dones=dones_off)
    env = z.Env(zsim, config=cfg)
    A, S = z.random_actions(91, 32, seed=23)
    ep, _ = _device_rollout(env, 91, A, S)
    rows, sums = env.episode_metrics(ep)
    got = z.aggregate_finalize(sums)
    h = env.download_episode(ep)
    ref = refpy.aggregate(h["s"], h["a_lat"], h["a_lon"], h["mask"], h["events"], h["initial_s"],
                          h["logged_progress"], env.info.dt)
    for k, (name, v) in enumerate(got.items()):
        assert abs(v - ref[k]) <= 1e-12 * max(1.0, abs(ref[k])), (name, v, ref[k])
    # per-row reports are consistent with the aggregate
    live = rows["degenerate"] == 0
    assert abs(rows["scenario_score"][live].mean() - got["mean_score"]) <= 1e-12
    assert set(np.unique(rows["collision_free"])) <= {0.0, 1.0}


@pytest.mark.gpu
def test_device_metric_sums_match_host_statement():
    from paper_2312_15122_b200.shard import metric_sums_host
    zsim = z.stress_scenarios(z.StressConfig(count=24), 13)
    env = z.Env(zsim, config=z.SimConfig(disable_dones=False))
    A, S = z.random_actions(91, 24, seed=29)
    ep, _ = _device_rollout(env, 91, A, S)
    _, sums = env.episode_metrics(ep, rows=False)
    h = env.download_episode(ep)
    want = metric_sums_host(h["s"], h["a_lat"], h["a_lon"], h["mask"], h["events"], h["initial_s"],
                            h["logged_progress"], env.info.dt)
    np.testing.assert_allclose(sums, want, rtol=1e-12, atol=1e-12)


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("seq_len,dones", [(16, False), (10, True), (1, True), (91, True)])
def test_cut_sequences_matches_reference(seq_len, dones):
    """zsim_cut_sequences = train::cut_sequences (replay.cpp:8-52) over a
    recorded device episode, against the REFERENCE's cut of its own rollout:
    sequence count, order (row, t0), per-step actions / done / mask bit-exact,
    logmu / reward / bootstrap / observations within the north_star tolerance."""
    B, T = 12, 40
    zsim = z.stress_scenarios(z.StressConfig(count=B, agents=10, road_points=500), seed=21)
    cfg = z.SimConfig(disable_dones=not dones)
    env = z.Env(zsim, config=cfg, device=0)
    A, S = z.random_actions(T, B, seed=17)
    ep, ob = _device_rollout(env, T, A, S, obs=True)
    got = env.cut_sequences_device(ep, ob, seq_len)
    import torch
    torch.cuda.synchronize()
    n = int(got["count"].item())
    ref = refpy.RefEnv(zsim, config=cfg).rollout_cut(T, A.T.copy(), S.T.copy(), seq_len)
    assert n == ref["count"] and n > 0
    g = {k: v[:n].cpu().numpy() for k, v in got.items() if k != "count"}
    np.testing.assert_array_equal(g["row"], ref["row"])
    for k in ("accel_idx", "steer_idx", "done", "mask"):
        np.testing.assert_array_equal(g[k], ref[k], err_msg=k)
    for k in ("logmu", "reward", "bootstrap", "obs_active", "obs_agents", "obs_road", "obs_route", "obs_value_only"):
        np.testing.assert_allclose(g[k], ref[k], rtol=RTOL, atol=ATOL, err_msg=k)
    assert (g["t0"] % seq_len == 0).all()


@pytest.mark.gpu
def test_cut_sequences_rejects_bad_seq_len():
    env = z.Env(z.stress_scenarios(z.StressConfig(count=2, agents=4, road_points=100), seed=2), device=0)
    A, S = z.random_actions(5, 2, seed=1)
    ep, ob = _device_rollout(env, 5, A, S, obs=True)
    with pytest.raises(z.ZsimError) as e:
        env.cut_sequences_device(ep, ob, 0)
    assert e.value.kind == "invalid_argument"
