"""C2 "all agents controlled".

The reference has no such mode; the row of actor j of a scenario is defined
as a reference Env row over zsim_controlled_expand's scenario for it
(include/zsim_gpu.h).  CPU tests pin the expansion itself (and that the
reference accepts every expanded scenario); GPU tests run the controlled
device Env -- scenario data staged once and shared by its rows -- against
the reference Env over the expanded scenarios, and against the ego-mode
device Env over the same expanded bytes (bit-identical)."""
from __future__ import annotations

import math

import numpy as np
import pytest

import paper_2312_15122_b200 as z
from oracle import refpy
from tests.parity import compare_obs, compare_state, compare_stepout
from tests.zsim_py import read_zsim


def _eq(a, b) -> bool:
    """Deep bitwise equality of decoded ZSIM records (dicts / lists / arrays)."""
    if isinstance(a, dict):
        return isinstance(b, dict) and a.keys() == b.keys() and all(_eq(a[k], b[k]) for k in a)
    if isinstance(a, (list, tuple)):
        return isinstance(b, (list, tuple)) and len(a) == len(b) and all(_eq(x, y) for x, y in zip(a, b))
    if isinstance(a, np.ndarray):
        return isinstance(b, np.ndarray) and a.dtype == b.dtype and a.tobytes() == b.tobytes()
    return a == b


def _c2(count=3, agents=6, seed=11):
    return z.stress_scenarios(z.StressConfig(count=count, agents=agents, road_points=256, flags=z.STRESS_C2), seed)


def test_expand_rows_and_actor_logs():
    src = _c2()
    scen = read_zsim(src)
    exp = read_zsim(z.controlled_expand(src))
    assert len(exp) == sum(1 + len(s["agents"]) for s in scen)  # C2 actors are valid at every step
    cfg = z.SimConfig()
    k = 0
    for s in scen:
        A = 1 + len(s["agents"])
        for j in range(A):
            e = exp[k]
            k += 1
            assert e["id"] == f"{s['id']}#{j}"
            assert _eq(e["lanes"], s["lanes"]) and _eq(e["features"], s["features"]) and _eq(e["lights"], s["lights"])
            assert len(e["agents"]) == A - 1
            if j == 0:
                assert _eq(e["ego"], s["ego"]) and _eq(e["agents"], s["agents"])
                assert (e["goal_x"], e["goal_y"]) == (s["goal_x"], s["goal_y"])
                continue
            ag = s["agents"][j - 1]
            assert _eq(e["ego"]["x"], ag["x"]) and _eq(e["ego"]["heading"], ag["heading"])
            assert _eq(e["ego"]["v"], ag["speed"])
            # the logged ego replays as agent 0 with the SimConfig ego box, centred ahead of its logged point
            ea = e["agents"][0]
            assert ea["length"] == np.float32(cfg.ego_length) and ea["width"] == np.float32(cfg.ego_width)
            h0 = float(s["ego"]["heading"][0])
            assert ea["x"][0] == np.float32(float(s["ego"]["x"][0]) + math.cos(h0) * cfg.ego_center_offset)
            # the other agents keep actor order
            assert _eq(e["agents"][1:], [a for i, a in enumerate(s["agents"]) if i != j - 1])
            h = float(ag["heading"][-1])
            assert e["goal_x"] == np.float32(float(ag["x"][-1]) + 4.0 * math.cos(h))


def test_only_fully_valid_agents_are_controllable():
    src = z.stress_scenarios(z.StressConfig(count=6, agents=8, road_points=128), 3)  # 15% invalid windows
    scen = read_zsim(src)
    want = sum(1 + sum(all(a["valid"][:s["num_steps"]]) for a in s["agents"]) for s in scen)
    assert len(read_zsim(z.controlled_expand(src))) == want
    assert want < sum(1 + len(s["agents"]) for s in scen)


@pytest.mark.skipif(not refpy.available(), reason="oracle/_ref not built")
def test_reference_accepts_expanded_scenarios():
    exp = z.controlled_expand(_c2())
    for i in range(len(read_zsim(exp))):
        assert refpy.validate(exp, i) == ""


@pytest.mark.gpu
@pytest.mark.parametrize("dones_off,agents", [(True, 8), (False, 8), (True, 40)])
def test_controlled_env_matches_reference(dones_off, agents):
    """agents=40: more than 32 agents per row (the chunked agent ordering)."""
    src = _c2(count=3, agents=agents)
    exp = z.controlled_expand(src)
    cfg = z.SimConfig(disable_dones=dones_off)
    genv = z.Env(src, config=cfg, controlled=True)
    assert genv.info.controlled == 1 and genv.info.scenarios == 3 and genv.info.batch == 3 * agents
    assert list(genv.row_scenario) == [s for s in range(3) for _ in range(agents)]
    assert list(genv.row_actor) == list(range(agents)) * 3
    renv = refpy.RefEnv(exp, config=cfg) if refpy.available() else None
    if renv is None:
        from oracle import portpy
        renv = portpy.PortEnv(exp, config=cfg)
    g, i, l = renv.scalars()
    assert np.array_equal(g, genv._goal_s) and np.array_equal(i, genv._initial_s) and np.array_equal(l, genv._logged)
    B = genv.info.batch
    steps = 91 if agents <= 8 else 30
    A, S = z.random_actions(steps, B, seed=5)
    sg, sr = genv.init_state(42), renv.init_state(42)
    errs = compare_state(sg, sr, "reset ")
    for t in range(steps):
        errs += compare_obs(genv.observe(sg), renv.observe(sr), f"t{t} ")
        ng, sog = genv.step(sg, A[t], S[t])
        nr, sor = renv.step(sr, A[t], S[t])
        errs += compare_state(ng, nr, f"t{t} ") + compare_stepout(sog, sor, f"t{t} ")
        sg, sr = ng, nr
        if len(errs) > 20:
            break
    assert not errs, "\n".join(errs[:20])


@pytest.mark.gpu
def test_controlled_env_equals_ego_env_on_expanded_rows():
    src = _c2(count=2, agents=12, seed=4)
    exp = z.controlled_expand(src)
    cfg = z.SimConfig(disable_dones=True)
    c_env, e_env = z.Env(src, config=cfg, controlled=True), z.Env(exp, config=cfg)
    B = c_env.info.batch
    assert e_env.info.batch == B and c_env.info.static_bytes < e_env.info.static_bytes
    A, S = z.random_actions(30, B, seed=8)
    sc, se = c_env.init_state(42), e_env.init_state(42)
    for t in range(30):
        oc, oe = c_env.observe(sc), e_env.observe(se)
        for f in ("active", "agents", "road", "route", "value_only"):
            assert np.array_equal(getattr(oc, f), getattr(oe, f)), (t, f)
        sc, _ = c_env.step(sc, A[t], S[t])
        se, _ = e_env.step(se, A[t], S[t])
        for f in ("x", "y", "heading", "v", "proj_s", "events"):
            assert np.array_equal(getattr(sc, f), getattr(se, f)), (t, f)
