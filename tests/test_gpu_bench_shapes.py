"""Parity at the BASELINE shapes, through the exact launches bench.py times.

Each test builds the benchmark's Env (Env.from_stress: the same scenario set,
seed, action tensor and reset seed as bench.py), runs the fused
step+observe launch over the WHOLE batch for a 91-step rollout, and every step
compares sampled rows against the reference simulator (oracle/_ref) stepping
only those rows.  Rows are independent (batch equivalence), so
the reference Env over a block of scenarios reproduces the block's rows once
its rng words are set to the full batch's (the split depends on the global
row index, simcore.cpp:261).

* C1: 4096 scenarios x 32 agents x 2048 points, one wave (the headline launch);
* C3 / C4: the per-GPU shards (8192 x 64 x 4096 and 16384 x 128 x 8192) that
  run with agent pruning and chunked agent ordering;
* C2: 128 controlled actors per scenario x 8192 points,
  the split arrangement forced (as at the benchmark's 524,288 rows) and the
  fused one, vs the reference over the expanded per-actor scenarios.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

import paper_2312_15122_b200 as z
from oracle import refpy
from oracle.hostio import OracleConfig
from tests.parity import compare_obs, compare_state, compare_stepout

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not refpy.available(), reason="oracle/_ref not built")]

EPISODE = 91
STATE_F = (("x", "<f8"), ("y", "<f8"), ("heading", "<f8"), ("v", "<f8"), ("steering", "<f8"), ("t", "<i4"),
           ("done", "|u1"), ("reason", "|u1"), ("rng", "<u8"), ("proj_s", "<f8"), ("proj_d", "<f8"),
           ("proj_in_corridor", "|u1"), ("events", "|u1"), ("stopped_flags", "|u1"))
STEPOUT_F = (("reward", "<f4"), ("event", "|u1"), ("s", "<f4"), ("a_lat", "<f4"), ("a_lon", "<f4"), ("v", "<f4"))


class _DevArray:
    """A device allocation of the library as a torch tensor (no copy)."""

    def __init__(self, ptr, shape, typestr):
        addr = C.cast(ptr, C.c_void_p).value
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (addr, False),
                                         "version": 2}


class _Rows:
    """Host copy of some rows of a device batch (attribute access like the
    oracle containers)."""


def _fetch(view, fields, B, rows, shapes=None):
    import torch
    out = _Rows()
    idx = torch.from_numpy(rows).cuda()
    for name, ts in fields:
        shape = (B,) + (shapes[name] if shapes else ())
        t = torch.as_tensor(_DevArray(getattr(view, name), shape, ts), device="cuda")
        setattr(out, name, t.index_select(0, idx).cpu().numpy())
    return out


def _fetch_obs(env, ob, rows):
    c = env.config()
    shapes = {"active": (9,), "agents": (c.n_agents, 6), "road": (c.n_road, 12), "route": (c.n_route, 5),
              "value_only": (2,)}
    return _fetch(ob.v, [(k, "<f4") for k in shapes], env.batch_size(), rows, shapes)


def _blocks(n_scen, width):
    """Three scenario blocks: start, middle, end of the batch."""
    mid = (n_scen // 2) - width // 2
    return [(0, width), (mid, mid + width), (n_scen - width, n_scen)]


def _run(shape: dict, n_scen: int, width: int, dones_off: bool, controlled: bool = False, launch_policy: int = 0,
         steps: int = EPISODE):
    import torch
    cfg = z.SimConfig(disable_dones=dones_off)
    A_, P = shape["agents"], shape["road_points"]
    env = z.Env.from_stress(z.StressConfig(count=n_scen, agents=A_, road_points=P,
                                           flags=z.STRESS_C2 if controlled else 0), 7, config=cfg,
                            controlled=controlled)
    if launch_policy:
        env.set_launch_policy(launch_policy)
    rpr = A_ if controlled else 1
    B = env.batch_size()
    assert B == n_scen * rpr and env.total_stop_lines == B  # one stop line per row: flags index by row
    accel, steer = z.random_actions(EPISODE, B, seed=123)
    dA, dS = torch.from_numpy(accel).cuda(), torch.from_numpy(steer).cuda()
    cur, nxt, so, ob = env.device_state(), env.device_state(), env.device_stepout(), env.device_obs()
    env.reset_device(42, cur)
    # reference blocks
    refs = []
    for lo, hi in _blocks(n_scen, width):
        img = refpy.stress(hi - lo, A_, P, seed=7, first_index=lo, c2=controlled)
        if controlled:
            img = refpy.controlled_expand(img)
        renv = refpy.RefEnv(img, config=OracleConfig(disable_dones=dones_off))
        rows = np.arange(lo * rpr, hi * rpr, dtype=np.int64)
        refs.append((renv, rows))
    rows_all = np.concatenate([r for _, r in refs])
    torch.cuda.synchronize()
    g0 = _fetch(cur.v, STATE_F, B, rows_all)
    rstates, errs, off = [], [], 0
    for renv, rows in refs:
        sr = renv.init_state(42)
        n = len(rows)
        sr.rng[...] = g0.rng[off:off + n]
        gsub = _Rows()
        for f, _ in STATE_F:
            setattr(gsub, f, getattr(g0, f)[off:off + n])
        errs += compare_state(gsub, sr, f"rows {rows[0]}.. reset ")
        rstates.append(sr)
        off += n
    for t in range(steps):
        env.step_observe_device(cur, dA[t].data_ptr(), dS[t].data_ptr(), nxt, so, ob)
        cur, nxt = nxt, cur
        torch.cuda.synchronize()
        gs, gso, gob = _fetch(cur.v, STATE_F, B, rows_all), _fetch(so.v, STEPOUT_F, B, rows_all), \
            _fetch_obs(env, ob, rows_all)
        off = 0
        for i, (renv, rows) in enumerate(refs):
            n = len(rows)
            nr, sor = renv.step(rstates[i], accel[t, rows], steer[t, rows])
            orf = renv.observe(nr)
            rstates[i] = nr
            sub = lambda o, fs: _sub(o, fs, off, n)  # noqa: E731
            tag = f"t{t} rows {rows[0]}.. "
            errs += compare_state(sub(gs, [f for f, _ in STATE_F]), nr, tag)
            errs += compare_stepout(sub(gso, [f for f, _ in STEPOUT_F]), sor, tag)
            errs += compare_obs(sub(gob, ["active", "agents", "road", "route", "value_only"]), orf, tag)
            off += n
        if len(errs) > 10:
            break
    env.check_errors()
    return errs, env


def _sub(o, fields, off, n):
    s = _Rows()
    for f in fields:
        setattr(s, f, getattr(o, f)[off:off + n])
    return s


@pytest.mark.parametrize("dones_off", [True, False])
def test_c1_full_launch_sampled_rows(dones_off):
    """The headline launch: 4096 rows, one wave; 3 x 86 = 258 rows checked every step."""
    errs, env = _run(dict(agents=32, road_points=2048), 4096, 86, dones_off)
    assert env.info.step_observe_kernels == 1
    assert not errs, "\n".join(errs[:10])


@pytest.mark.parametrize("dones_off", [True, False])
def test_c3_shard_sampled_rows(dones_off):
    errs, _ = _run(dict(agents=64, road_points=4096), 8192, 24, dones_off)
    assert not errs, "\n".join(errs[:10])


def test_c4_shard_sampled_rows():
    """The 8-GPU C4 shard (16,384 rows, ~4 waves): deeper than three waves,
    so the automatic launch policy runs the split kernels (step + agents,
    then road / route top-k)."""
    errs, env = _run(dict(agents=128, road_points=8192), 16384, 16, True)
    assert env.info.step_observe_kernels == 2
    assert not errs, "\n".join(errs[:10])


@pytest.mark.parametrize("launch_policy", [1, 2])
@pytest.mark.parametrize("dones_off", [True, False])
def test_c2_controlled_128_actors_8k_points(dones_off, launch_policy):
    """SURVEY 8a row 20 at the C2 shape: 4 scenarios x 128 controlled actors x
    8192 points, all 512 rows vs the reference over the expanded scenarios;
    launch_policy 2 forces the split kernels the 524,288-row benchmark runs."""
    errs, env = _run(dict(agents=128, road_points=8192), 4, 1, dones_off, controlled=True,
                     launch_policy=launch_policy)
    assert env.info.step_observe_kernels == (1 if launch_policy == 1 else 2)
    assert not errs, "\n".join(errs[:10])


def test_c2_benchmark_batch_sampled_rows():
    """The C2 benchmark batch itself (4096 scenarios = 524,288 controlled rows,
    split kernels chosen automatically): 2 scenarios' 256 rows at each end
    and the middle, 20 steps."""
    errs, env = _run(dict(agents=128, road_points=8192), 4096, 1, True, controlled=True, steps=20)
    assert env.info.step_observe_kernels == 2
    assert not errs, "\n".join(errs[:10])


def test_from_stress_matches_zsim_image():
    """Env.from_stress stages exactly what Env(stress_scenarios(...)) stages."""
    sc = z.StressConfig(count=6, agents=20, road_points=700, first_index=33)
    e1 = z.Env.from_stress(sc, 7)
    e2 = z.Env(z.stress_scenarios(sc, 7))
    assert e1.info.static_bytes == e2.info.static_bytes
    assert np.array_equal(e1._goal_s, e2._goal_s) and np.array_equal(e1._initial_s, e2._initial_s)
    s1, s2 = e1.init_state(42), e2.init_state(42)
    A, S = z.random_actions(5, 6, seed=1)
    for t in range(5):
        o1, o2 = e1.observe(s1), e2.observe(s2)
        assert np.array_equal(o1.road, o2.road) and np.array_equal(o1.agents, o2.agents)
        s1, _ = e1.step(s1, A[t], S[t])
        s2, _ = e2.step(s2, A[t], S[t])
    assert np.array_equal(s1.x, s2.x)
