"""Generate the golden fixtures in tests/golden/ from the REFERENCE simulator
(oracle/_ref, compiled in place from /root/reference by oracle/build_oracle.py).

    python tests/golden/make_golden.py

Fixtures (small; committed):
  gen8.zsim      8 scenarios from the reference generator generate_synthetic
                 (scenario_gen.cpp:601-634; straight / curve / junction with
                 stop lines), seed 2, 92 logged steps.
  stress4.zsim   4 stress scenarios from our generator at reduced shape
                 (8 agents, 256 road points) -- checked against the
                 reference's validate (scenario_io.cpp:193-271).
  golden.npz     for each file and for dones on/off: the reference's
                 init_state(42), then 91 steps of observe+step with fixed
                 actions (random seed 5 for stress4; the recovered logged
                 actions, simcore.cpp:629-652, for gen8): every state and
                 StepOut, and the observation at steps 0, 1, 30, 60, 90.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import paper_2312_15122_b200 as z  # noqa: E402
from oracle import refpy  # noqa: E402

OUT = Path(__file__).resolve().parent
OBS_STEPS = (0, 1, 30, 60, 90)
STATE_F = ("x", "y", "heading", "v", "steering", "t", "done", "reason", "rng", "proj_s", "proj_d", "proj_in_corridor",
           "events", "stopped_flags")
STEPOUT_F = ("reward", "event", "s", "a_lat", "a_lon", "v")
OBS_F = ("active", "agents", "road", "route", "value_only")


def actions_for(name: str, zsim: bytes, B: int):
    if name == "stress4":
        return z.random_actions(91, B, seed=5)
    acts = [refpy.recover_actions(zsim, b) for b in range(B)]
    return (np.stack([a for a, _ in acts], 1).astype(np.int32), np.stack([s for _, s in acts], 1).astype(np.int32))


def record(name: str, zsim: bytes, dones_off: bool, out: dict) -> None:
    cfg = z.SimConfig(disable_dones=dones_off)
    env = refpy.RefEnv(zsim, config=cfg)
    B = env.batch_size()
    A, S = actions_for(name, zsim, B)
    key = f"{name}_{'off' if dones_off else 'on'}"
    g, i, l = env.scalars()
    out[f"{key}/goal_s"], out[f"{key}/initial_s"], out[f"{key}/logged_progress"] = g, i, l
    out[f"{key}/accel"], out[f"{key}/steer"] = A, S
    st = env.init_state(42)
    states = {f: [getattr(st, f).copy()] for f in STATE_F}
    so_rec = {f: [] for f in STEPOUT_F}
    for t in range(A.shape[0]):
        ob = env.observe(st)
        if t in OBS_STEPS:
            for f in OBS_F:
                out[f"{key}/obs{t}/{f}"] = getattr(ob, f).copy()
        st, so = env.step(st, A[t], S[t])
        for f in STATE_F:
            states[f].append(getattr(st, f).copy())
        for f in STEPOUT_F:
            so_rec[f].append(getattr(so, f).copy())
    for f in STATE_F:
        out[f"{key}/state/{f}"] = np.stack(states[f])
    for f in STEPOUT_F:
        out[f"{key}/stepout/{f}"] = np.stack(so_rec[f])


def main() -> None:
    if not refpy.available():
        raise SystemExit("oracle/_ref not built: run oracle/build_oracle.py where /root/reference exists")
    gen8 = refpy.generate(8, seed=2, num_steps=92)
    stress4 = z.stress_scenarios(z.StressConfig(count=4, agents=8, road_points=256, lane_vertices=24), seed=3)
    for b in range(4):
        msg = refpy.validate(stress4, b)
        assert not msg, msg
    (OUT / "gen8.zsim").write_bytes(gen8)
    (OUT / "stress4.zsim").write_bytes(stress4)
    out: dict = {}
    for name, zsim in (("gen8", gen8), ("stress4", stress4)):
        for dones_off in (True, False):
            record(name, zsim, dones_off, out)
    np.savez_compressed(OUT / "golden.npz", **out)
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
