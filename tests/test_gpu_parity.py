"""GPU parity suite: the sm_100a kernels (through the C-ABI) against the
reference simulator compiled in place (oracle/_ref) on identical scenarios
and actions.  Contract (BASELINE.json north_star): flags, reasons, events,
done, top-k membership bit-exact; fp outputs within 1e-5 rel / 1e-6 abs on
every step of a 91-step rollout."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2312_15122_b200 as z
from tests.parity import compare_obs, compare_state, compare_stepout

pytestmark = pytest.mark.gpu

from oracle import portpy, refpy

needs_ref = pytest.mark.skipif(not refpy.available(), reason="oracle/_ref not built")


def _oracle(zsim, cfg):
    """The compiled reference when present, else the C restatement (pinned to
    the reference by tests/test_oracle.py and the golden fixtures)."""
    return refpy.RefEnv(zsim, config=cfg) if refpy.available() else portpy.PortEnv(zsim, config=cfg)


@pytest.fixture(scope="module")
def stress16():
    return z.stress_scenarios(z.StressConfig(count=16), seed=7)


@pytest.fixture(scope="module")
def generated32():
    if not refpy.available():
        from tests.golden_check import GOLDEN
        return (GOLDEN / "gen8.zsim").read_bytes()
    return refpy.generate(32, seed=7, num_steps=92)


def _rollout_vs_ref(zsim, cfg, accel, steer, steps, resync=False):
    genv = z.Env(zsim, config=cfg)
    renv = _oracle(zsim, cfg)
    errs = []
    g, i, l = renv.scalars()
    if not (np.array_equal(g, genv._goal_s) and np.array_equal(i, genv._initial_s)
            and np.array_equal(l, genv._logged)):
        errs.append("staged goal_s / initial_s / logged_progress differ from the reference")
    sg, sr = genv.init_state(42), renv.init_state(42)
    errs += compare_state(sg, sr, "reset ")
    for t in range(steps):
        og, orf = genv.observe(sr if resync else sg), renv.observe(sr)
        errs += compare_obs(og, orf, f"t{t} ")
        ng, sog = genv.step(sr if resync else sg, accel[t], steer[t])
        nr, sor = renv.step(sr, accel[t], steer[t])
        errs += compare_state(ng, nr, f"t{t} ")
        errs += compare_stepout(sog, sor, f"t{t} ")
        sg, sr = ng, nr
        if len(errs) > 20:
            break
    og, orf = genv.observe(sg), renv.observe(sr)
    errs += compare_obs(og, orf, "final ")
    return errs, sg, sr


@pytest.mark.parametrize("dones_off", [True, False])
def test_stress_rollout_matches_reference(stress16, dones_off):
    cfg = z.SimConfig(disable_dones=dones_off)
    A, S = z.random_actions(91, 16, seed=123)
    errs, sg, _ = _rollout_vs_ref(stress16, cfg, A, S, 91)
    assert not errs, "\n".join(errs[:20])
    if dones_off:
        assert sg.events.any()  # the random policy does trigger latched events


def test_stress_rollout_resynced_matches_reference(stress16):
    cfg = z.SimConfig(disable_dones=True)
    A, S = z.random_actions(91, 16, seed=321)
    errs, _, _ = _rollout_vs_ref(stress16, cfg, A, S, 91, resync=True)
    assert not errs, "\n".join(errs[:20])


@pytest.mark.parametrize("dones_off", [True, False])
def test_generated_random_rollout_matches_reference(generated32, dones_off):
    cfg = z.SimConfig(disable_dones=dones_off)
    B = z.Env(generated32).batch_size()
    A, S = z.random_actions(91, B, seed=99)
    errs, _, _ = _rollout_vs_ref(generated32, cfg, A, S, 91)
    assert not errs, "\n".join(errs[:20])


@needs_ref
@pytest.mark.parametrize("dones_off", [True, False])
def test_generated_logged_replay_is_clean(generated32, dones_off):
    """Generator soundness (scenario_gen.cpp:528-549) on the device: replaying
    the recovered logged actions triggers nothing and lands on the log."""
    B = 32
    acts = [refpy.recover_actions(generated32, b) for b in range(B)]
    T = len(acts[0][0])
    A = np.stack([a for a, _ in acts], 1).astype(np.int32)
    S = np.stack([s for _, s in acts], 1).astype(np.int32)
    cfg = z.SimConfig(disable_dones=dones_off)
    env = z.Env(generated32, config=cfg)
    st = env.init_state(1)
    for t in range(T):
        env.observe(st)
        st, so = env.step(st, A[t], S[t])
        assert not st.done.any(), f"t={t}: done rows {np.nonzero(st.done)[0]}"
    assert not st.events.any()
    logged = env._logged
    ratio = (so.s.astype(np.float64) - env._initial_s) / logged
    assert np.all(np.abs(ratio - 1.0) <= 1e-6), ratio
    errs, _, _ = _rollout_vs_ref(generated32, cfg, A, S, T)
    assert not errs, "\n".join(errs[:20])


def _device_rollout(env, A, S, steps, fused, seed=42):
    import torch
    dA = torch.from_numpy(A).cuda()
    dS = torch.from_numpy(S).cuda()
    s0, s1 = env.device_state(), env.device_state()
    so, ob = env.device_stepout(), env.device_obs()
    stream = torch.cuda.current_stream()
    env.reset_device(seed, s0, stream)
    obs_hist, so_hist = [], []
    for t in range(steps):
        a, s = dA[t].data_ptr(), dS[t].data_ptr()
        if fused:
            env.step_observe_device(s0, a, s, s1, so, ob, stream)
        else:
            env.step_device(s0, a, s, s1, so, stream)
            env.observe_device(s1, ob, stream)
        obs_hist.append(env.download_obs(ob, stream=stream))
        so_hist.append(env.download_stepout(so, stream=stream))
        torch.cuda.synchronize()
        s0, s1 = s1, s0
    st = env.download_state(s0, stream=stream)
    torch.cuda.synchronize()
    return st, obs_hist, so_hist


def test_fused_step_observe_is_bit_identical_to_separate(stress16):
    env = z.Env(stress16, config=z.SimConfig(disable_dones=True))
    A, S = z.random_actions(30, 16, seed=5)
    st1, ob1, so1 = _device_rollout(env, A, S, 30, fused=True)
    st2, ob2, so2 = _device_rollout(env, A, S, 30, fused=False)
    for f in ("x", "y", "heading", "v", "steering", "proj_s", "events", "rng", "stopped_flags"):
        assert np.array_equal(getattr(st1, f), getattr(st2, f)), f
    for a, b in zip(ob1, ob2):
        for f in ("active", "agents", "road", "route", "value_only"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), f
    for a, b in zip(so1, so2):
        assert np.array_equal(a.reward, b.reward)


def test_device_path_matches_host_path(stress16):
    env = z.Env(stress16, config=z.SimConfig(disable_dones=False))
    A, S = z.random_actions(20, 16, seed=8)
    st_dev, ob_dev, so_dev = _device_rollout(env, A, S, 20, fused=True)
    st = env.init_state(42)
    for t in range(20):
        st, so = env.step(st, A[t], S[t])
        ob = env.observe(st)
        assert np.array_equal(ob.road, ob_dev[t].road)
        assert np.array_equal(so.reward, so_dev[t].reward)
    assert np.array_equal(st.x, st_dev.x) and np.array_equal(st.events, st_dev.events)


def test_batch_equivalence_bit_exact(stress16):
    """env_step(B scenarios) == B x env_step(1 scenario), bit-exact."""
    cfg = z.SimConfig(disable_dones=True)
    A, S = z.random_actions(12, 16, seed=11)
    env = z.Env(stress16, config=cfg)
    st = env.init_state(42)
    obs_b = []
    for t in range(12):
        obs_b.append(env.observe(st))
        st, _ = env.step(st, A[t], S[t])
    for b in (0, 5, 15):
        e1 = z.Env(stress16, indices=[b], config=cfg)
        s1 = e1.init_state(42)
        s1.rng[...] = env.init_state(42).rng[b]  # rng split depends on the row index (simcore.cpp:261)
        for t in range(12):
            o1 = e1.observe(s1)
            assert np.array_equal(o1.road[0], obs_b[t].road[b])
            assert np.array_equal(o1.agents[0], obs_b[t].agents[b])
            s1, _ = e1.step(s1, A[t, b:b + 1], S[t, b:b + 1])
        assert s1.x[0] == st.x[b] and s1.events[0] == st.events[b]


def test_determinism(stress16):
    env = z.Env(stress16, config=z.SimConfig(disable_dones=True))
    A, S = z.random_actions(15, 16, seed=2)
    r1 = _device_rollout(env, A, S, 15, fused=True)
    r2 = _device_rollout(env, A, S, 15, fused=True)
    assert np.array_equal(r1[0].x, r2[0].x)
    assert all(np.array_equal(a.road, b.road) for a, b in zip(r1[1], r2[1]))


def test_bad_action_index_raises_invalid_argument(stress16):
    env = z.Env(stress16)
    st = env.init_state(42)
    A = np.zeros(16, np.int32)
    S = np.zeros(16, np.int32)
    A[3] = 7  # 7 accel bins: 0..6
    with pytest.raises(z.ZsimError) as ei:
        env.step(st, A, S)
    assert ei.value.kind == "invalid_argument" and "out of range" in str(ei.value)
    with pytest.raises(z.ZsimError):
        env.step(st, A[:5], S[:5])


def test_device_error_word_reports_bad_action(stress16):
    import torch
    env = z.Env(stress16)
    s0, s1, so = env.device_state(), env.device_state(), env.device_stepout()
    env.reset_device(42, s0)
    A = torch.zeros(16, dtype=torch.int32, device="cuda")
    S = torch.zeros(16, dtype=torch.int32, device="cuda")
    S[2] = -1
    env.step_device(s0, A.data_ptr(), S.data_ptr(), s1, so)
    with pytest.raises(z.ZsimError) as ei:
        env.check_errors()
    assert ei.value.kind == "invalid_argument"
    env.check_errors()  # cleared


def test_device_error_word_reports_non_finite_state(stress16):
    """Failure detection: a NaN ego state is flagged (ZSIM_RUNTIME) while the
    step itself stays the reference's (the NaN propagates, other rows exact)."""
    import torch
    env = z.Env(stress16, config=z.SimConfig(disable_dones=True))
    st = env.init_state(42)
    st.v[5] = np.nan
    s0, s1, so = env.device_state(), env.device_state(), env.device_stepout()
    env.upload_state(st, s0)
    A = torch.zeros(16, dtype=torch.int32, device="cuda")
    S = torch.zeros(16, dtype=torch.int32, device="cuda")
    env.step_device(s0, A.data_ptr(), S.data_ptr(), s1, so)
    with pytest.raises(z.ZsimError) as ei:
        env.check_errors()
    assert ei.value.kind == "runtime" and "non-finite" in str(ei.value)
    env.check_errors()  # cleared
    host = env.download_state(s1)
    ref, _ = env.step(st, np.zeros(16, np.int32), np.zeros(16, np.int32))
    assert np.isnan(host.x[5]) and np.array_equal(np.delete(host.x, 5), np.delete(ref.x, 5))


def test_all_done_batch_is_absorbing(stress16):
    """all scenarios already done -> state unchanged, rewards 0."""
    env = z.Env(stress16)
    st = env.init_state(42)
    st.done[:] = 1
    st.reason[:] = 2
    nxt, so = env.step(st, np.full(16, 6, np.int32), np.full(16, 4, np.int32))
    for f in ("x", "y", "heading", "v", "steering", "t", "proj_s", "events"):
        assert np.array_equal(getattr(nxt, f), getattr(st, f)), f
    assert (so.reward == 0).all() and (so.event == 0).all()
    ob = env.observe(nxt)
    assert not ob.road.any() and not ob.active.any()


@pytest.mark.parametrize("controlled", [False, True])
def test_split_observation_kernels_equal_fused(controlled):
    """zsim_set_launch_policy: the split kernel arrangement (step + agents,
    then road/route top-k) is bit-identical to the fused kernel."""
    import torch
    if controlled:
        zsim = z.stress_scenarios(z.StressConfig(count=3, agents=40, road_points=512, flags=z.STRESS_C2), 9)
    else:
        zsim = z.stress_scenarios(z.StressConfig(count=24), 9)
    outs = []
    for policy in (1, 2):
        env = z.Env(zsim, config=z.SimConfig(disable_dones=False), controlled=controlled)
        env.set_launch_policy(policy)
        B = env.info.batch
        A, S = z.random_actions(40, B, seed=2)
        dA, dS = torch.from_numpy(A).cuda(), torch.from_numpy(S).cuda()
        s0, s1, so, ob = env.device_state(), env.device_state(), env.device_stepout(), env.device_obs()
        env.reset_device(42, s0)
        rec = []
        for t in range(40):
            env.step_observe_device(s0, dA[t].data_ptr(), dS[t].data_ptr(), s1, so, ob)
            s0, s1 = s1, s0
            o = env.download_obs(ob)
            rec.append([getattr(o, f).copy() for f in ("active", "agents", "road", "route", "value_only")])
        env.observe_device(s0, ob)  # observe-only arrangement too
        o = env.download_obs(ob)
        rec.append([getattr(o, f).copy() for f in ("active", "agents", "road", "route", "value_only")])
        st = env.download_state(s0)
        rec.append([st.x.copy(), st.done.copy(), st.events.copy()])
        outs.append(rec)
    for a, b in zip(*outs):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


def test_in_place_step_matches_out_of_place(stress16):
    """zsim_step's `out` may alias `in` (include/zsim_gpu.h): a rollout that
    steps one device state in place equals the ping-pong rollout bit for bit
    (stopped flags included: the pre-step flags are read before they are
    overwritten)."""
    import torch
    env = z.Env(stress16, config=z.SimConfig(disable_dones=False))
    A, S = z.random_actions(60, 16, seed=99)
    dA, dS = torch.from_numpy(A).cuda(), torch.from_numpy(S).cuda()
    s0, s1, sp = env.device_state(), env.device_state(), env.device_state()
    so, ob = env.device_stepout(), env.device_obs()
    env.reset_device(42, s0)
    env.reset_device(42, sp)
    for t in range(60):
        env.step_observe_device(s0, dA[t].data_ptr(), dS[t].data_ptr(), s1, so, ob)
        s0, s1 = s1, s0
        env.step_observe_device(sp, dA[t].data_ptr(), dS[t].data_ptr(), sp, so, ob)
    torch.cuda.synchronize()
    a, b = env.download_state(s0), env.download_state(sp)
    for name in ("x", "y", "heading", "v", "steering", "t", "done", "reason", "events", "proj_s", "stopped_flags"):
        assert np.array_equal(getattr(a, name), getattr(b, name)), name


@pytest.mark.parametrize("count", [16, 2100])
def test_step_observe_host_equals_step_then_observe(count):
    """zsim_step_observe_host (one call, row chunks streamed back from 2048
    rows on) gives exactly step_host followed by observe_host."""
    zsim = z.stress_scenarios(z.StressConfig(count=count, agents=12, road_points=300), 5)
    env = z.Env(zsim, config=z.SimConfig(disable_dones=False))
    A, S = z.random_actions(12, count, seed=4)
    s_a = env.init_state(42)
    s_b = env.init_state(42)
    for t in range(12):
        n_a, so_a = env.step(s_a, A[t], S[t])
        ob_a = env.observe(n_a)
        n_b, so_b, ob_b = env.step_observe(s_b, A[t], S[t])
        for f in ("x", "y", "heading", "v", "steering", "t", "done", "reason", "rng", "proj_s", "events",
                  "stopped_flags"):
            assert np.array_equal(getattr(n_a, f), getattr(n_b, f)), (t, f)
        for f in ("reward", "event", "s", "v"):
            assert np.array_equal(getattr(so_a, f), getattr(so_b, f)), (t, f)
        for f in ("active", "agents", "road", "route", "value_only"):
            assert np.array_equal(getattr(ob_a, f), getattr(ob_b, f)), (t, f)
        s_a, s_b = n_a, n_b
    with pytest.raises(z.ZsimError):
        env.step_observe(s_b, A[0][:-1], S[0][:-1])
