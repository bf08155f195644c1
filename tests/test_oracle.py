"""CPU tests of the oracles (test infrastructure): the plain-C restatement
(oracle/zsim_oracle.c) against the golden fixtures produced by the reference,
against the reference compiled in place (when oracle/_ref is built here), and
the SPEC known-answer cases against both."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2312_15122_b200 as z
from oracle import portpy, refpy
from tests import golden_check, kat_cases
from tests.parity import compare_obs, compare_state, compare_stepout
from tests.zsim_py import read_zsim

needs_ref = pytest.mark.skipif(not refpy.available(), reason="oracle/_ref not built (needs /root/reference)")


def port_env(zsim, cfg):
    return portpy.PortEnv(zsim, config=cfg)


def ref_env(zsim, cfg):
    return refpy.RefEnv(zsim, config=cfg)


def test_golden_fixtures_decode():
    g8 = read_zsim((golden_check.GOLDEN / "gen8.zsim").read_bytes())
    s4 = read_zsim((golden_check.GOLDEN / "stress4.zsim").read_bytes())
    assert len(g8) == 8 and len(s4) == 4
    assert sum(len(s["stops"]) for s in g8) >= 2 and max(len(s["lanes"]) for s in g8) == 4  # junctions
    assert all(len(s["agents"]) == 7 and len(s["lights"]) == 1 and len(s["stops"]) == 1 for s in s4)


@pytest.mark.parametrize("name,mode", golden_check.CASES)
def test_port_matches_golden_bit_exact(name, mode):
    errs, frac = golden_check.replay(port_env, name, mode, exact=True)
    assert not errs, "\n".join(errs[:10])
    assert frac > 0.99


@needs_ref
@pytest.mark.parametrize("name,mode", golden_check.CASES)
def test_reference_reproduces_golden(name, mode):
    errs, frac = golden_check.replay(ref_env, name, mode, exact=True)
    assert not errs and frac == 1.0, "\n".join(errs[:10])


@needs_ref
@pytest.mark.parametrize("dones_off", [True, False])
def test_port_matches_reference_on_stress_rollout(dones_off):
    zsim = z.stress_scenarios(z.StressConfig(count=6, agents=32, road_points=2048), seed=21)
    cfg = z.SimConfig(disable_dones=dones_off)
    A, S = z.random_actions(91, 6, seed=77)
    r, p = refpy.RefEnv(zsim, config=cfg), portpy.PortEnv(zsim, config=cfg)
    assert all(np.array_equal(a, b) for a, b in zip(r.scalars(), p.scalars()))
    sr, sp = r.init_state(9), p.init_state(9)
    errs = compare_state(sp, sr)
    for t in range(91):
        errs += compare_obs(p.observe(sp), r.observe(sr), f"t{t} ")
        sr, sor = r.step(sr, A[t], S[t])
        sp, sop = p.step(sp, A[t], S[t])
        errs += compare_state(sp, sr, f"t{t} ") + compare_stepout(sop, sor, f"t{t} ")
        assert np.array_equal(sp.x, sr.x) and np.array_equal(sop.reward, sor.reward)
    assert not errs, "\n".join(errs[:10])


@needs_ref
def test_stress_scenarios_pass_reference_validate():
    zsim = z.stress_scenarios(z.StressConfig(count=8), seed=7)
    for b in range(8):
        assert refpy.validate(zsim, b) == ""


@pytest.mark.parametrize("case", kat_cases.ALL, ids=lambda f: f.__name__)
def test_port_known_answers(case):
    case(port_env)


@needs_ref
@pytest.mark.parametrize("case", kat_cases.ALL, ids=lambda f: f.__name__)
def test_reference_known_answers(case):
    case(ref_env)


def test_port_rejects_bad_action():
    zsim = (golden_check.GOLDEN / "stress4.zsim").read_bytes()
    env = portpy.PortEnv(zsim)
    st = env.init_state(1)
    with pytest.raises(portpy.PortError):
        env.step(st, np.array([0, 0, 9, 0], np.int32), np.zeros(4, np.int32))
