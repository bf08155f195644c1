"""On-device policy inference: NNPolicy::act over
forward_row (train/policy.hpp:27-58, nn/model.hpp:464-585) against the float64
numpy restatement in oracle/policy_oracle.py.

Tolerances against the float64 oracle (the reference itself computes in
float32 with Eigen's summation order, so it sits within the fp32 bound too):
  precision "fp32" (the default: every contraction on the FP32 pipe): logits / value within
      1e-5 absolute + 1e-4 relative, log-probs within 2e-5 (measured: 4e-7);
  precision "tf32" (opt-in: the ten 128x128 projections on tcgen05 with
      tf32 operands, fp32 accumulation): logits / value within 1e-3 absolute +
      5e-3 relative, log-probs within 2e-3 (measured: 1.8e-4).
Sampled / argmax indices must be identical wherever the oracle's decision
margin exceeds the path's margin (1e-4 fp32, 2e-3 tf32; a closer call may
legitimately flip under rounding on either side); rng streams advance
bit-exactly."""
import ctypes as C

import numpy as np
import pytest

from oracle import policy_oracle as po
from oracle import refpy

TOL = {"fp32": dict(atol=1e-5, rtol=1e-4, logp=2e-5, margin=1e-4),
       "tf32": dict(atol=1e-3, rtol=5e-3, logp=2e-3, margin=2e-3)}


def test_init_params_bit_exact_vs_oracle():
    import paper_2312_15122_b200 as z
    for seed in (0, 7):
        a = z.init_params(z.ModelConfig(), seed)
        b = po.init_params(po.ModelConfig(), seed)
        assert a.dtype == np.float32 and a.size == b.size == 425837
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_param_layout_matches_reference_order():
    ix = po.param_index(po.ModelConfig())
    names = [e.name for e in ix.entries]
    assert names[:4] == ["emb.agents.w", "emb.agents.b", "emb.road.w", "emb.road.b"]
    assert names[-2:] == ["value.head.w", "value.head.b"]
    assert ix.by_name["enc.self.wq"].rows == 128 and ix.by_name["value.in.w"].cols == 160


def test_config_errors():
    import paper_2312_15122_b200 as z
    with pytest.raises(z.ZsimError) as e:
        z.ModelConfig(latent=96, heads=5).param_count()
    assert e.value.kind == "config"
    with pytest.raises(z.ZsimError) as e:
        z.ModelConfig(latent=64).param_count()
    assert e.value.kind == "config"
    with pytest.raises(z.ZsimError) as e:
        z.ModelConfig(trunk_blocks=0).param_count()
    assert e.value.kind == "config"


def random_obs(B, rng):
    """Observation rows with the value ranges the simulator produces, plus
    all-zero (done) rows and partially masked token sets."""
    obs = {
        "active": rng.normal(0, 3, (B, 9)).astype(np.float32),
        "agents": rng.normal(0, 20, (B, 16, 6)).astype(np.float32),
        "road": rng.normal(0, 30, (B, 128, 12)).astype(np.float32),
        "route": rng.normal(0, 30, (B, 64, 5)).astype(np.float32),
        "value_only": np.abs(rng.normal(0, 50, (B, 2))).astype(np.float32),
    }
    obs["agents"][..., 5] = rng.random((B, 16)) < 0.7
    obs["road"][..., 2:11] = rng.random((B, 128, 9)) < 0.3
    obs["road"][..., 11] = rng.random((B, 128)) < 0.8
    obs["route"][..., 2:4] = rng.random((B, 64, 2)) < 0.5
    obs["route"][..., 4] = rng.random((B, 64)) < 0.9
    for k in obs:
        obs[k][1] = 0.0  # a done row
    obs["agents"][2, :, 5] = 0.0  # no valid agents: only the null latent token
    obs["road"][3, :, 11] = 0.0  # no valid road tokens
    return obs


def run_device(pol, obs, rng_state, B):
    import torch
    from paper_2312_15122_b200._abi import ObsView
    dev = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in obs.items()}
    view = ObsView()
    for k, t in dev.items():
        setattr(view, k, C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_float)))
    rng = torch.from_numpy(rng_state.view(np.int64).copy()).cuda()
    accel = torch.zeros(B, dtype=torch.int32, device="cuda")
    steer = torch.zeros_like(accel)
    logp = torch.zeros(B, dtype=torch.float32, device="cuda")
    value = torch.zeros_like(logp)
    na, ns = pol.cfg.n_accel, pol.cfg.n_steer
    logits = torch.zeros(B, na + ns, dtype=torch.float32, device="cuda")
    pol.act_device(view, B, rng.data_ptr(), accel.data_ptr(), steer.data_ptr(), logp.data_ptr(), value.data_ptr(),
                   logits.data_ptr())
    torch.cuda.synchronize()
    return dict(accel=accel.cpu().numpy(), steer=steer.cpu().numpy(), logp=logp.cpu().numpy(),
                value=value.cpu().numpy(), rng=rng.cpu().numpy().view(np.uint64),
                logits=logits.cpu().numpy())


def margins_ok(logits, u, use_argmax, margin):
    """Decision margin of the oracle: top-2 logit gap (argmax) or the distance
    of u to the nearest CDF boundary (sampling)."""
    if use_argmax:
        s = np.sort(logits)
        return s[-1] - s[-2] > margin
    p = np.exp(po.log_softmax(logits))
    return np.min(np.abs(np.cumsum(p) - u)) > margin


def check_against_oracle(cfg_o, params, obs, B, use_argmax, precision, seed=3):
    import paper_2312_15122_b200 as z
    tol = TOL[precision]
    rng0 = np.array([(0x1234567 * (b + 1) + seed) & ((1 << 64) - 1) for b in range(B)], np.uint64)
    pol = z.NNPolicy(z.ModelConfig(), params, use_argmax=use_argmax, precision=precision)
    got = run_device(pol, obs, rng0, B)
    ref = po.act(po.Model(cfg_o, params), obs, rng0, use_argmax)
    na = cfg_o.n_accel
    err = max(np.abs(got["logits"][:, :na] - ref["logits_accel"]).max(),
              np.abs(got["logits"][:, na:] - ref["logits_steer"]).max(), np.abs(got["value"] - ref["value"]).max())
    print(f"{precision}: max |logit / value error| = {err:.3g}")
    np.testing.assert_allclose(got["logits"][:, :na], ref["logits_accel"], atol=tol["atol"], rtol=tol["rtol"])
    np.testing.assert_allclose(got["logits"][:, na:], ref["logits_steer"], atol=tol["atol"], rtol=tol["rtol"])
    np.testing.assert_allclose(got["value"], ref["value"], atol=tol["atol"], rtol=tol["rtol"])
    checked = 0
    for b in range(B):
        if margins_ok(ref["logits_accel"][b], ref["u"][b][0], use_argmax, tol["margin"]) and \
                margins_ok(ref["logits_steer"][b], ref["u"][b][1], use_argmax, tol["margin"]):
            assert got["accel"][b] == ref["accel"][b] and got["steer"][b] == ref["steer"][b], b
            assert abs(got["logp"][b] - ref["logp"][b]) < tol["logp"], b
            checked += 1
    assert checked >= (9 * B) // 10, (checked, B)  # decisive-margin rows: actions and logp must match
    if not use_argmax:
        assert np.array_equal(got["rng"], ref["rng"])  # two draws per row
    return got, ref


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["tf32", "fp32"])
@pytest.mark.parametrize("use_argmax", [True, False])
def test_policy_act_random_obs(use_argmax, precision):
    cfg_o = po.ModelConfig()
    params = po.init_params(cfg_o, 11)
    B = 17  # the last CTA is partial for both row groupings (7 and 3 rows per CTA)
    obs = random_obs(B, np.random.default_rng(5))
    check_against_oracle(cfg_o, params, obs, B, use_argmax, precision)


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["tf32", "fp32"])
def test_policy_act_on_simulator_observations(precision):
    import torch

    import paper_2312_15122_b200 as z
    zsim = z.stress_scenarios(z.StressConfig(count=16, agents=20, road_points=900), seed=3)
    env = z.Env(zsim, config=z.SimConfig(disable_dones=False), device=0)
    st, nxt, so, ob = env.device_state(), env.device_state(), env.device_stepout(), env.device_obs()
    env.reset_device(4, st)
    A, S = z.random_actions(5, 16, seed=9)
    for t in range(5):
        a, s = torch.from_numpy(A[t]).cuda(), torch.from_numpy(S[t]).cuda()
        env.step_observe_device(st, a.data_ptr(), s.data_ptr(), nxt, so, ob)
        st, nxt = nxt, st
    torch.cuda.synchronize()
    h = env.download_obs(ob)
    obs = {k: getattr(h, k).copy() for k in ("active", "agents", "road", "route", "value_only")}
    cfg_o = po.ModelConfig()
    check_against_oracle(cfg_o, po.init_params(cfg_o, 2), obs, 16, False, precision)


@pytest.mark.gpu
@pytest.mark.skipif(not refpy.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("precision", ["fp32", "tf32"])
@pytest.mark.parametrize("use_argmax", [True, False])
def test_policy_act_vs_reference_nnpolicy(use_argmax, precision):
    """The device NNPolicy against the reference's own NNPolicy::act
    (policy.hpp:27-58 over model.hpp's Model<float>, compiled unchanged in
    oracle/_ref with oracle/eigen_mini): actions identical wherever the
    decision margin exceeds the precision's, rng streams bit-identical, value
    and log-prob within the precision's tolerance."""
    import paper_2312_15122_b200 as z
    tol = TOL[precision]
    params = refpy.policy_init(None, 13)
    B = 40
    obs = random_obs(B, np.random.default_rng(17))
    rng0 = (np.arange(1, B + 1, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)) ^ np.uint64(99)
    ref = refpy.policy_act(params, obs, B, rng0, use_argmax)
    logits64, _ = refpy.policy_forward(params, obs, B, double=True)
    pol = z.NNPolicy(z.ModelConfig(), params, use_argmax=use_argmax, precision=precision)
    got = run_device(pol, obs, rng0.copy(), B)
    np.testing.assert_allclose(got["value"], ref["value"], atol=tol["atol"], rtol=tol["rtol"])
    # decision margins from the reference's float64 logits and the sampled u
    ora = po.act(po.Model(po.ModelConfig(), params), obs, rng0.copy(), use_argmax)
    checked = 0
    for b in range(B):
        if margins_ok(logits64[b, :7], ora["u"][b][0], use_argmax, tol["margin"]) and \
                margins_ok(logits64[b, 7:], ora["u"][b][1], use_argmax, tol["margin"]):
            assert got["accel"][b] == ref["accel"][b] and got["steer"][b] == ref["steer"][b], b
            assert abs(got["logp"][b] - ref["logp"][b]) < tol["logp"], b
            checked += 1
    assert checked >= (9 * B) // 10, (checked, B)
    if not use_argmax:
        assert np.array_equal(got["rng"], ref["rng"])


@pytest.mark.gpu
def test_policy_errors():
    import paper_2312_15122_b200 as z
    p = po.init_params(po.ModelConfig(), 1)
    with pytest.raises(z.ZsimError) as e:
        z.NNPolicy(z.ModelConfig(), p[:-1])
    assert e.value.kind == "invalid_argument"


def _oracle_env(zsim, cfg):
    from oracle import portpy, refpy
    return refpy.RefEnv(zsim, config=cfg) if refpy.available() else portpy.PortEnv(zsim, config=cfg)


@pytest.mark.gpu
@pytest.mark.parametrize("use_argmax", [True, False])
def test_policy_rollout_matches_oracle_loop(use_argmax):
    """zsim_rollout_policy = Env::rollout with NNPolicy (simcore.cpp:554-618,
    train/policy.hpp:27-58) against the oracle loop observe -> act -> step
    (the reference Env + the float64 policy oracle).  fp32 precision; a row is
    compared up to the first step whose policy decision margin is below 1e-4
    (past a legitimately flipped near-tie the trajectories diverge)."""
    import torch

    import paper_2312_15122_b200 as z
    zsim = z.stress_scenarios(z.StressConfig(count=6, agents=12, road_points=600), seed=4)
    cfg = z.SimConfig(disable_dones=False)
    env = z.Env(zsim, config=cfg, device=0)
    cfg_o = po.ModelConfig()
    params = po.init_params(cfg_o, 9)
    pol = z.NNPolicy(z.ModelConfig(), params, use_argmax=use_argmax, precision="fp32")
    H, B = 12, 6
    ep = env.device_episode(H)
    env.rollout_policy_device(pol, 42, H, episode=ep)
    torch.cuda.synchronize()
    got = env.download_episode(ep)

    ref = _oracle_env(zsim, cfg)
    model = po.Model(cfg_o, params)
    st = ref.init_state(42)
    live = np.ones(B, bool)
    for t in range(H):
        o = ref.observe(st)
        obs = {k: getattr(o, k) for k in ("active", "agents", "road", "route", "value_only")}
        out = po.act(model, obs, st.rng, use_argmax)
        for b in range(B):
            if live[b] and not (margins_ok(out["logits_accel"][b], out["u"][b][0], use_argmax, 1e-4) and
                                margins_ok(out["logits_steer"][b], out["u"][b][1], use_argmax, 1e-4)):
                live[b] = False
        st.rng[:] = out["rng"]
        mask = 1 - st.done.astype(np.int32)
        nst, so = ref.step(st, out["accel"], out["steer"])
        for b in np.nonzero(live)[0]:
            assert got["accel_idx"][b, t] == out["accel"][b] and got["steer_idx"][b, t] == out["steer"][b], (b, t)
            assert got["mask"][b, t] == mask[b] and got["done"][b, t] == nst.done[b], (b, t)
            assert abs(got["logp"][b, t] - out["logp"][b]) < 2e-5, (b, t)
            assert abs(got["value"][b, t] - out["value"][b]) < 1e-5 + 1e-4 * abs(out["value"][b]), (b, t)
            for f in ("reward", "s", "v"):
                np.testing.assert_allclose(got[f][b, t], getattr(so, f)[b], rtol=1e-5, atol=1e-6)
        st = nst
    assert live.sum() >= B // 2
    # bootstrap = the policy's value on the final observation (0 for done rows)
    o = ref.observe(st)
    out = po.act(model, {k: getattr(o, k) for k in ("active", "agents", "road", "route", "value_only")}, st.rng,
                 use_argmax)
    for b in np.nonzero(live)[0]:
        want = 0.0 if st.done[b] else out["value"][b]
        assert abs(got["bootstrap"][b] - want) < 1e-5 + 1e-4 * abs(want)
        assert got["terminal"][b] == st.reason[b] and got["events"][b] == st.events[b]


@pytest.mark.gpu
def test_policy_act_host_matches_device_path():
    """zsim_policy_act_host (the RolloutPolicy-shaped host entry point behind
    the C++ drop-in zsim::gpu::NNPolicy) equals the device entry point."""
    import paper_2312_15122_b200 as z
    from paper_2312_15122_b200._abi import ObsView, lib
    cfg_o = po.ModelConfig()
    params = po.init_params(cfg_o, 4)
    B = 9
    obs = random_obs(B, np.random.default_rng(8))
    rng0 = np.arange(1, B + 1, dtype=np.uint64) * np.uint64(977)
    for use_argmax in (True, False):
        pol = z.NNPolicy(z.ModelConfig(), params, use_argmax=use_argmax)
        dev = run_device(pol, obs, rng0.copy(), B)
        host = {k: np.ascontiguousarray(v, dtype=np.float32) for k, v in obs.items()}
        v = ObsView()
        for k, a in host.items():
            setattr(v, k, a.ctypes.data_as(C.POINTER(C.c_float)))
        rng = rng0.copy()
        acc, ste = np.zeros(B, np.int32), np.zeros(B, np.int32)
        lp, val = np.zeros(B, np.float32), np.zeros(B, np.float32)
        P = lambda a: C.c_void_p(a.ctypes.data)  # noqa: E731
        assert lib.zsim_policy_act_host(pol.handle, C.byref(v), B, P(rng), int(use_argmax), P(acc), P(ste), P(lp),
                                        P(val)) == 0
        np.testing.assert_array_equal(acc, dev["accel"])
        np.testing.assert_array_equal(ste, dev["steer"])
        np.testing.assert_array_equal(lp, dev["logp"])
        np.testing.assert_array_equal(val, dev["value"])
        if not use_argmax:
            np.testing.assert_array_equal(rng, dev["rng"])


def test_policy_oracle_attention_invariances():
    """CPU check of the float64 policy oracle's attention semantics
    (model.hpp:326-367): masked key tokens receive probability exactly 0, so
    their feature values cannot change any output, and cross attention is
    invariant to the order of the key tokens."""
    cfg = po.ModelConfig()
    m = po.Model(cfg, po.init_params(cfg, 6))
    obs = random_obs(4, np.random.default_rng(3))
    base = po.forward_row(m, obs, 0)
    o2 = {k: v.copy() for k, v in obs.items()}
    masked = o2["road"][0, :, 11] <= 0.5
    o2["road"][0, masked, :11] = 123.0  # garbage in masked road tokens
    o2["route"][0, o2["route"][0, :, 4] <= 0.5, :4] = -55.0
    got = po.forward_row(m, o2, 0)
    for a, b in zip(base[:2], got[:2]):
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-12)
    assert abs(base[2] - got[2]) < 1e-12
    perm = np.random.default_rng(1).permutation(128)
    o3 = {k: v.copy() for k, v in obs.items()}
    o3["road"][0] = obs["road"][0][perm]
    got = po.forward_row(m, o3, 0)
    np.testing.assert_allclose(base[0], got[0], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(base[1], got[1], rtol=1e-12, atol=1e-12)
