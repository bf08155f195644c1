"""The drop-in demonstration on the GPU: oracle/_ref/dropin_check runs the
same C++ caller code against zsim::sim::Env (reference) and zsim::gpu::Env
(include/zsim_gpu.hpp -> libzsim_gpu.so): the generator's log-replay
soundness check and a random-policy rollout compared field by field."""
from __future__ import annotations

import json
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
BIN = Path(__file__).resolve().parent.parent / "oracle" / "_ref" / "dropin_check"


@pytest.mark.skipif(not BIN.exists(), reason="oracle/_ref/dropin_check not built (needs /root/reference)")
def test_cpp_dropin_env_matches_reference():
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert r.returncode == 0 and line["ok"], r.stdout + r.stderr
    assert line["clean_gpu"] == line["replays"] and line["flag_mismatches"] == 0
