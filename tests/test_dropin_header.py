"""CPU check that include/zsim_gpu.hpp compiles against the reference's own
headers (the drop-in boundary) -- only where /root/reference is present."""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF = Path("/root/reference/proj/src")


@pytest.mark.skipif(not (REF / "core" / "simcore.hpp").exists(), reason="reference sources absent")
def test_dropin_header_compiles_against_reference_headers(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text('#include "zsim_gpu.hpp"\n'
                   'using SimEnv = zsim::gpu::Env;\n'
                   'static_assert(sizeof(SimEnv) > 0);\n'
                   'int main() { return 0; }\n')
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", str(REF), "-I", str(ROOT / "include"), str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
