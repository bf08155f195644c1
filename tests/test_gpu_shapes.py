"""Shape coverage against the reference (oracle/_ref, else the C port):
paths the default C1 shapes never take.

* more than 4 route lanes (several lane blocks in the projection),
* long lane centrelines (more than 16 8-segment groups: groups always scanned),
* more than 32 agents per row in ego mode (chunked agent ordering, bound
  pruning; C3/C4), and so many agents that the per-warp shared memory forces
  the 4-warp CTA arrangement,
* large roadgraphs (8192 points, 256 chunks: C4; 10000 points: more chunks than
  the candidate capacity),
* fewer road / route points than k (partially filled top-k, zero padding),
* a single-scenario batch.

Each runs a rollout with random actions, dones on and off, and compares
every state, StepOut and observation like test_gpu_parity."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2312_15122_b200 as z
from oracle import portpy, refpy
from tests.parity import compare_obs, compare_state, compare_stepout

pytestmark = pytest.mark.gpu


def _oracle(zsim, cfg):
    return refpy.RefEnv(zsim, config=cfg) if refpy.available() else portpy.PortEnv(zsim, config=cfg)


def _rollout(zsim, dones_off, steps=40, seed=3):
    cfg = z.SimConfig(disable_dones=dones_off)
    genv, renv = z.Env(zsim, config=cfg), _oracle(zsim, cfg)
    B = genv.info.batch
    A, S = z.random_actions(steps, B, seed=seed)
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
    errs += compare_obs(genv.observe(sg), renv.observe(sr), "final ")
    return errs


SHAPES = {
    "six_lanes": dict(count=6, lanes=6, road_points=512),
    "long_lanes": dict(count=4, lane_vertices=200, road_points=512),
    "very_long_lanes": dict(count=2, lane_vertices=600, road_points=256),
    "agents_64": dict(count=6, agents=64, road_points=1024),
    "agents_128": dict(count=4, agents=128, road_points=1024),
    "agents_900": dict(count=2, agents=900, road_points=512),
    "roadgraph_8k": dict(count=4, agents=16, road_points=8192),
    # more than cap (256) chunks: the top-k chunk list outgrows the candidate buffers
    "roadgraph_10k": dict(count=2, agents=8, road_points=10000),
    "sparse_map": dict(count=6, agents=4, road_points=40, lanes=1, lane_vertices=12),
    "single": dict(count=1, agents=8, road_points=300),
}


@pytest.mark.parametrize("dones_off", [True, False])
@pytest.mark.parametrize("shape", sorted(SHAPES))
def test_shape_rollout_matches_reference(shape, dones_off):
    zsim = z.stress_scenarios(z.StressConfig(**SHAPES[shape]), 11)
    errs = _rollout(zsim, dones_off)
    assert not errs, "\n".join(errs[:20])


def test_sparse_map_pads_topk_with_zero_rows():
    zsim = z.stress_scenarios(z.StressConfig(**SHAPES["sparse_map"]), 11)
    env = z.Env(zsim, config=z.SimConfig())
    ob = env.observe(env.init_state(42))
    # valid flags: at most 40 road points and 2*1*12 route points exist
    assert (ob.road[:, :, 11].sum(1) <= 40).all() and (ob.road[:, 40:, :] == 0).all()
    assert (ob.route[:, 24:, :] == 0).all()
