"""bench.py's driver contract on CPU: `--gpus N` spawns N ranks itself
(torch.distributed.run, 127.0.0.1) and rank 0 prints one line with n_gpus == N;
the reference arm never imports the product package or maps libzsim_gpu.so;
both arms emit the same `config` block."""
from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import refpy  # noqa: E402

needs_ref = pytest.mark.skipif(not refpy.available(), reason="oracle/_ref not built")


def _json_lines(out: str) -> list[dict]:
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


@needs_ref
def test_gpus_flag_spawns_ranks_reference_arm():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--impl", "reference", "--config",
                        "C0", "--steps", "2", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"]["scenarios"] == 128 and line["config"]["scenarios_per_gpu"] == 64
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "reference"


@needs_ref
def test_reference_arm_does_not_load_the_product():
    code = (
        "import sys, json; sys.argv = ['bench.py', '--impl', 'reference', '--config', 'C0', '--steps', '1'];"
        "import bench; bench.main();"
        "maps = open('/proc/self/maps').read();"
        "print(json.dumps({'product_imported': 'paper_2312_15122_b200' in sys.modules,"
        " 'gpu_lib_mapped': 'libzsim_gpu.so' in maps, 'ref_mapped': 'libzsim_ref.so' in maps}))")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    res = _json_lines(r.stdout)[-1]
    assert res == {"product_imported": False, "gpu_lib_mapped": False, "ref_mapped": True}


def test_config_block_identical_in_both_arms():
    import bench
    for name in bench.CONFIGS:
        for world in (1, 2, 8):
            p = bench.plan(name, world)
            a, b = bench.config_block(p, world), bench.config_block(bench.plan(name, world), world)
            assert a == b
            if p["scaling"] == "strong":
                assert p["total"] == bench.CONFIGS[name]["global_"]
            else:
                assert p["total"] == bench.CONFIGS[name]["per_gpu"] * world


def test_c4_strong_split_matches_baseline():
    """BASELINE configs[4]: 131072 scenarios = 65536 / 32768 / 16384 per GPU at 2 / 4 / 8."""
    import bench
    from paper_2312_15122_b200.shard import shard_rows
    for world, per in ((2, 65536), (4, 32768), (8, 16384)):
        p = bench.plan("C4", world)
        assert {hi - lo for lo, hi in (shard_rows(p["total"], world, r) for r in range(world))} == {per}


def test_config_hash_is_the_key_value_hash():
    """bench.py's config_hash is KeyValue.hash() of the same keys
    (paper_2312_15122_b200.config, pinned to the reference's cfg::KeyValue)."""
    import bench
    from paper_2312_15122_b200.config import KeyValue
    p = bench.plan("C1", 1)
    kv = KeyValue()
    for k, v in bench.SIM_CONFIG.items():
        kv.set(f"sim.{k}", v)
    for k, v in (("bench.config", "C1"), ("bench.scenarios", 4096), ("bench.agents", 32),
                 ("bench.road_points", 2048), ("bench.controlled", 0), ("bench.lanes", 4),
                 ("bench.lane_vertices", 64), ("bench.steps_per_episode", 91), ("bench.seed.scenarios", 7),
                 ("bench.seed.actions", 123), ("bench.seed.reset", 42)):
        kv.set(k, v)
    assert bench.config_hash(p) == f"{kv.hash():016x}"
    assert bench.config_hash(bench.plan("C2", 1)) != bench.config_hash(p)
