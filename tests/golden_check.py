"""Replay a golden fixture (tests/golden/golden.npz, produced by the reference
via tests/golden/make_golden.py) through any Env implementation."""
from __future__ import annotations

from pathlib import Path

import numpy as np

import paper_2312_15122_b200 as z
from tests.parity import compare_obs, compare_state, compare_stepout

GOLDEN = Path(__file__).resolve().parent / "golden"
STATE_F = ("x", "y", "heading", "v", "steering", "t", "done", "reason", "rng", "proj_s", "proj_d", "proj_in_corridor",
           "events", "stopped_flags")
STEPOUT_F = ("reward", "event", "s", "a_lat", "a_lon", "v")
OBS_F = ("active", "agents", "road", "route", "value_only")
CASES = [(name, mode) for name in ("gen8", "stress4") for mode in ("off", "on")]


def load():
    return dict(np.load(GOLDEN / "golden.npz"))


class _Obj:
    pass


def _state_at(g, key, k):
    o = _Obj()
    for f in STATE_F:
        setattr(o, f, g[f"{key}/state/{f}"][k])
    return o


def replay(make_env, name: str, mode: str, g=None, exact: bool = False):
    """Returns (errors, bit_identical_fraction).  `exact` demands bit-equality
    of every state / StepOut array (valid for another glibc-based build)."""
    g = g if g is not None else load()
    key = f"{name}_{mode}"
    zsim = (GOLDEN / f"{name}.zsim").read_bytes()
    env = make_env(zsim, z.SimConfig(disable_dones=(mode == "off")))
    A, S = g[f"{key}/accel"], g[f"{key}/steer"]
    errs = []
    same = total = 0
    st = env.init_state(42)
    errs += compare_state(st, _state_at(g, key, 0), "reset ")
    for t in range(A.shape[0]):
        if t in (0, 1, 30, 60, 90):
            ob = env.observe(st)
            ref = _Obj()
            for f in OBS_F:
                setattr(ref, f, g[f"{key}/obs{t}/{f}"])
            errs += compare_obs(ob, ref, f"t{t} ")
            for f in OBS_F:
                same += int(np.array_equal(getattr(ob, f), getattr(ref, f)))
                total += 1
        st, so = env.step(st, A[t], S[t])
        rs = _state_at(g, key, t + 1)
        errs += compare_state(st, rs, f"t{t} ")
        rso = _Obj()
        for f in STEPOUT_F:
            setattr(rso, f, g[f"{key}/stepout/{f}"][t])
        errs += compare_stepout(so, rso, f"t{t} ")
        for f in STATE_F:
            eq = np.array_equal(getattr(st, f), getattr(rs, f))
            same += int(eq)
            total += 1
            if exact and not eq:
                errs.append(f"t{t} state.{f} not bit-identical")
        for f in STEPOUT_F:
            eq = np.array_equal(getattr(so, f), getattr(rso, f))
            same += int(eq)
            total += 1
            if exact and not eq:
                errs.append(f"t{t} stepout.{f} not bit-identical")
        if len(errs) > 20:
            break
    return errs, same / max(total, 1)
