"""Known-answer cases from the reference's SPEC examples (SPEC.md [OP]
sections; the reference ships no test cases), run against any
implementation with the Env host API (GPU Env, C restatement, compiled
reference).  Each case builds a crafted straight-road scenario
(tests/zsim_py.straight_scenario) and checks the documented outcome."""
from __future__ import annotations

import math

import numpy as np

import paper_2312_15122_b200 as z
from tests.zsim_py import straight_scenario, write_zsim

ZERO_A, ZERO_S = 3, 2  # indices of 0.0 in ActionTable::defaults (dynamics.cpp:21-26)


def _one_step(make_env, sc, dones_off=False, accel=ZERO_A, steer=ZERO_S):
    env = make_env(write_zsim([sc]), z.SimConfig(disable_dones=dones_off))
    st = env.init_state(42)
    ob = env.observe(st)
    nxt, so = env.step(st, np.array([accel], np.int32), np.array([steer], np.int32))
    return st, ob, nxt, so


def kat_straight_line(make_env):
    """v=10, delta=0, theta=0, dt=0.1 => x += 1.0, y += 0."""
    st, _, nxt, so = _one_step(make_env, straight_scenario(v=10.0))
    assert nxt.x[0] == st.x[0] + 1.0 and nxt.y[0] == st.y[0]
    assert nxt.heading[0] == 0.0 and nxt.v[0] == 10.0 and nxt.t[0] == 1
    assert so.event[0] == 0 and not nxt.done[0]


def kat_rest_state(make_env):
    """v=0, a=0 => position and heading unchanged."""
    st, _, nxt, _ = _one_step(make_env, straight_scenario(v=0.0))
    assert nxt.x[0] == st.x[0] and nxt.y[0] == st.y[0] and nxt.heading[0] == st.heading[0]


def kat_speed_penalty(make_env):
    """v = v_limit + 1, w_s = 0.1, dt = 0.1 => -0.01 speed term."""
    _, _, nxt, so = _one_step(make_env, straight_scenario(v=11.0, limit=10.0))
    progress = nxt.proj_s[0] - 0.0
    assert abs(float(so.reward[0]) - (progress - 0.01)) < 1e-6
    assert abs(progress - 1.1) < 1e-9


def kat_collision(make_env):
    """identical boxes => collision; priority over off-route."""
    sc = straight_scenario(v=10.0, agents=[{"x": 2.5, "y": 0.0, "length": 4.7, "width": 1.9}])
    _, _, nxt, so = _one_step(make_env, sc)
    assert so.event[0] == 1 and nxt.done[0] == 1 and nxt.reason[0] == 1 and nxt.events[0] == 1
    assert abs(float(so.reward[0]) - (nxt.proj_s[0] - 10.0)) < 1e-5  # terminal penalty
    _, _, nxt, so = _one_step(make_env, sc, dones_off=True)
    assert so.event[0] == 1 and nxt.done[0] == 0 and nxt.events[0] & 1


def kat_off_route(make_env):
    """ego centre 3 m laterally off a single 3.5 m lane => off_route."""
    sc = straight_scenario(v=5.0)
    sc["ego"]["y"] = np.full(sc["num_steps"], 3.0)
    _, _, nxt, so = _one_step(make_env, sc)
    assert so.event[0] == 2 and nxt.reason[0] == 2


def kat_red_light(make_env):
    """crossing a red signal's stop point => red_light."""
    n = 20
    sc = straight_scenario(v=10.0, lights=[{"stop_x": 0.5, "stop_y": 0.0, "state": np.zeros(n, np.uint8)}])
    _, ob, nxt, so = _one_step(make_env, sc)
    assert so.event[0] == 3
    assert ob.active[0, 3] == 1.0 and abs(ob.active[0, 7] - 0.5) < 1e-6  # red one-hot, distance to light
    sc["lights"][0]["state"] = np.full(n, 2, np.uint8)  # green: no event
    _, ob, _, so = _one_step(make_env, sc)
    assert so.event[0] == 0 and ob.active[0, 5] == 1.0


def kat_stop_line(make_env):
    """SPEC.md:345 stop-line semantics: crossing above 0.5 m/s without a stop => stop_line;
    stop_info distance."""
    sc = straight_scenario(v=10.0, stops=[{"xy": [0.5, -1.75, 0.5, 1.75], "pos_x": 0.5, "pos_y": 0.0}])
    _, ob, _, so = _one_step(make_env, sc)
    assert so.event[0] == 4 and abs(ob.active[0, 2] - 0.5) < 1e-6
    sc = straight_scenario(v=10.0, stops=[{"xy": [50.0, -1.75, 50.0, 1.75], "pos_x": 50.0, "pos_y": 0.0}])
    _, ob, _, so = _one_step(make_env, sc)
    assert so.event[0] == 0 and abs(ob.active[0, 2] - 50.0) < 1e-5


def kat_goal(make_env):
    """goal termination carries zero terminal reward."""
    sc = straight_scenario(v=10.0, goal=(2.0, 0.0))
    _, _, nxt, so = _one_step(make_env, sc)
    assert so.event[0] == 5 and nxt.done[0] == 1
    assert abs(float(so.reward[0]) - nxt.proj_s[0]) < 1e-6


def kat_agent_ahead_frame(make_env):
    """agent directly 5 m ahead, ego heading pi/2 => relative (5, 0)."""
    sc = straight_scenario(v=0.0, heading=math.pi / 2,
                           agents=[{"x": 0.0, "y": 5.0, "heading": math.pi / 2, "length": 4.0, "width": 2.0}])
    _, ob, _, _ = _one_step(make_env, sc, dones_off=True)
    f = ob.agents[0, 0]
    assert abs(f[0] - 5.0) < 1e-5 and abs(f[1]) < 1e-5 and f[5] == 1.0
    assert ob.agents[0, 1, 5] == 0.0  # one agent only


def kat_parallel_box_distance(make_env):
    """SPEC.md:321 analogue -- parallel boxes offset laterally: distance = gap
    (ego box 4.7 x 1.9 centred 1.5 m ahead; agent 4 x 2 at y = 3 => 3 - 0.95 - 1.0)."""
    sc = straight_scenario(v=0.0, agents=[{"x": 1.5, "y": 3.0, "length": 4.0, "width": 2.0}])
    _, ob, _, _ = _one_step(make_env, sc, dones_off=True)
    assert abs(ob.agents[0, 0, 4] - 1.05) < 1e-6


def kat_no_features_in_radius(make_env):
    """no features in radius => all road slots invalid."""
    far = np.array([500.0, 500.0, 502.0, 500.0])
    sc = straight_scenario(v=0.0, features=[{"kind": 4, "dir": 0, "xy": far}])
    _, ob, _, _ = _one_step(make_env, sc, dones_off=True)
    assert not ob.road.any()


def kat_single_feature(make_env):
    """one feature point at 2 m => that point, kind/dir one-hot."""
    sc = straight_scenario(v=0.0, features=[{"kind": 2, "dir": 3, "xy": np.array([2.0, 0.0, 150.0, 0.0])}])
    _, ob, _, _ = _one_step(make_env, sc, dones_off=True)
    f = ob.road[0, 0]
    assert abs(f[0] - 2.0) < 1e-6 and f[1] == 0.0 and f[2 + 2] == 1.0 and f[7 + 3] == 1.0 and f[11] == 1.0
    assert ob.road[0, 1, 11] == 0.0  # the second point is 150 m away: outside the radius


ALL = [kat_straight_line, kat_rest_state, kat_speed_penalty, kat_collision, kat_off_route, kat_red_light,
       kat_stop_line, kat_goal, kat_agent_ahead_frame, kat_parallel_box_distance, kat_no_features_in_radius,
       kat_single_feature]
