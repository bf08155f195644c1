"""BatchStream (scenario_stream.hpp:12-40): the dataset
in file order as device Envs of `batch_size` scenarios (last batch short),
batch k+1 staged and uploaded while batch k runs.  Every delivered batch must
behave exactly like an Env created directly over the same scenarios, with or
without prefetch."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2312_15122_b200 as z

pytestmark = pytest.mark.gpu


def _run(env, steps=20):
    A, S = z.random_actions(steps, env.info.batch, seed=4)
    st = env.init_state(42)
    out = []
    for t in range(steps):
        ob = env.observe(st)
        st, so = env.step(st, A[t], S[t])
        out.append((ob.road.copy(), ob.agents.copy(), st.x.copy(), st.events.copy(), so.reward.copy()))
    return out


@pytest.mark.parametrize("prefetch", [True, False])
def test_stream_batches_equal_direct_envs(prefetch):
    zsim = z.stress_scenarios(z.StressConfig(count=11, road_points=512), 3)
    cfg = z.SimConfig(disable_dones=False)
    stream = z.BatchStream(zsim, batch_size=4, config=cfg, prefetch=prefetch)
    assert len(stream) == 3
    sizes = []
    for k, env in enumerate(stream):
        sizes.append(env.info.batch)
        idx = list(range(4 * k, min(4 * k + 4, 11)))
        want = _run(z.Env(zsim, indices=idx, config=cfg))
        got = _run(env)
        for a, b in zip(got, want):
            for x, y in zip(a, b):
                assert np.array_equal(x, y)
    assert sizes == [4, 4, 3]
    stream.close()


def test_stream_controlled_batches():
    zsim = z.stress_scenarios(z.StressConfig(count=4, agents=6, road_points=256, flags=z.STRESS_C2), 5)
    envs = [(e.info.batch, e.info.scenarios, e.info.controlled) for e in z.BatchStream(zsim, 2, controlled=True)]
    assert envs == [(12, 2, 1), (12, 2, 1)]
