"""Flat key = value configs (paper_2312_15122_b200/config.py) against the
reference's own cfg::KeyValue (core/config.cpp compiled in place as
oracle/_ref/kv_check): identical dump and FNV-1a hash on the same text,
including comments, spacing, duplicate keys and doubles written by set()."""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

import paper_2312_15122_b200 as z
from paper_2312_15122_b200.config import KeyValue, fnv1a, sim_config_from_kv, sim_config_to_kv

KV = Path(__file__).resolve().parent.parent / "oracle" / "_ref" / "kv_check"
needs_ref = pytest.mark.skipif(not KV.exists(), reason="oracle/_ref/kv_check not built")

TEXTS = [
    "b = 2 # c\n a=  x y \n\n# only comment\nc=3.5\nb=4\n",
    "n_agents = 16\nfeature_radius = 100\ndisable_dones = true\n",
    "\tk\t=\tv\t\r\nz=1\nA=upper\n_u = 0\n",
    "",
]


def _ref(text: str, sets=()) -> tuple[str, int]:
    inp = text + ("\n---\n" + "".join(f"{k} {v!r}\n" for k, v in sets) if sets else "")
    out = subprocess.run([str(KV)], input=inp, capture_output=True, text=True, timeout=60).stdout
    body, h = out.rsplit("hash=", 1)
    return body, int(h)


@needs_ref
@pytest.mark.parametrize("text", TEXTS)
def test_dump_and_hash_match_reference(text):
    kv = KeyValue.parse_text(text)
    assert (kv.dump(), kv.hash()) == _ref(text)


@needs_ref
def test_set_double_matches_reference_formatting():
    sets = [("d", 0.1), ("e", 1.0), ("f", 1e20), ("g", -2.5e-7), ("h", 123456.789)]
    kv = KeyValue.parse_text("a = 1\n")
    for k, v in sets:
        kv.set(k, v)
    assert (kv.dump(), kv.hash()) == _ref("a = 1\n", sets)


def test_fnv1a_known_values():
    assert fnv1a(b"") == 0xCBF29CE484222325
    assert fnv1a(b"a") == 0xAF63DC4C8601EC8C


def test_sim_config_round_trip_and_strictness():
    cfg = z.SimConfig(disable_dones=True, feature_radius=75.5, n_road=96)
    kv = sim_config_to_kv(cfg)
    back = sim_config_from_kv(KeyValue.parse_text(kv.dump()))
    assert back == cfg
    assert sim_config_to_kv(back).hash() == kv.hash()
    with pytest.raises(z.ZsimError) as e:
        sim_config_from_kv(KeyValue.parse_text("n_road = 12\nbogus = 1\n"))
    assert e.value.kind == "config"
    with pytest.raises(z.ZsimError):
        sim_config_from_kv(KeyValue.parse_text("n_road = 1_2\n"))
    with pytest.raises(z.ZsimError):
        KeyValue.parse_text("novalue\n")
