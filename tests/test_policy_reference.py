"""Pins the policy oracle to the reference's own code (CPU).

oracle/_ref/libzsim_ref.so carries the reference's core/nn/model.hpp and
core/train/policy.hpp compiled UNCHANGED (oracle/ref_policy_shim.cpp), with
oracle/eigen_mini standing in for Eigen, which this image does not have.
These tests check the float64 numpy restatement (oracle/policy_oracle.py,
the checker the device policy tests also use) against it:

* Model::init (model.hpp:199-212): bit-identical parameters;
* forward_row (model.hpp:464-585) in Model<double>: logits / value within
  1e-12 of the restatement (same arithmetic, different summation order);
* NNPolicy::act (policy.hpp:27-58) in the reference's Model<float>: the same
  actions (argmax and sampling), rng streams bit-identical, joint log-prob
  within 1e-5 of the float64 restatement.
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle import policy_oracle as po
from oracle import refpy
from tests.test_policy import random_obs

pytestmark = pytest.mark.skipif(not refpy.available(), reason="oracle/_ref not built")


def test_reference_init_matches_restatement():
    cfg = po.ModelConfig()
    for seed in (0, 11):
        assert np.array_equal(refpy.policy_init(None, seed), po.init_params(cfg, seed))
    assert refpy.policy_param_count() == po.init_params(cfg, 0).size


def test_reference_forward_matches_restatement_float64():
    cfg = po.ModelConfig()
    params = refpy.policy_init(None, 7)
    B = 12
    obs = random_obs(B, np.random.default_rng(21))
    logits, value = refpy.policy_forward(params, obs, B, double=True)
    m = po.Model(cfg, params)
    for b in range(B):
        la, ls, v = po.forward_row(m, obs, b)
        np.testing.assert_allclose(logits[b], np.concatenate([la, ls]), rtol=0, atol=1e-12)
        assert abs(value[b] - v) < 1e-12


def test_reference_float_forward_is_within_fp32_of_float64():
    params = refpy.policy_init(None, 3)
    B = 8
    obs = random_obs(B, np.random.default_rng(2))
    l32, v32 = refpy.policy_forward(params, obs, B, double=False)
    l64, v64 = refpy.policy_forward(params, obs, B, double=True)
    assert np.abs(l32 - l64).max() < 1e-5 and np.abs(v32 - v64).max() < 1e-5


@pytest.mark.parametrize("use_argmax", [True, False])
def test_reference_act_matches_restatement(use_argmax):
    cfg = po.ModelConfig()
    params = refpy.policy_init(None, 5)
    B = 16
    obs = random_obs(B, np.random.default_rng(9))
    rng0 = (np.arange(1, B + 1, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15)) ^ np.uint64(12345)
    ref = refpy.policy_act(params, obs, B, rng0, use_argmax)
    ora = po.act(po.Model(cfg, params), obs, rng0.copy(), use_argmax)
    assert np.array_equal(ref["accel"], ora["accel"]) and np.array_equal(ref["steer"], ora["steer"])
    assert np.abs(ref["logp"] - ora["logp"]).max() < 1e-5
    assert np.abs(ref["value"] - ora["value"]).max() < 1e-5
    if not use_argmax:
        assert np.array_equal(ref["rng"], ora["rng"])
