"""Build recipe for the parity oracles (TEST INFRASTRUCTURE).

* ``oracle/_ref/libzsim_ref.so`` -- the reference simulator compiled IN PLACE
  from ``/root/reference/proj/src/core/*.cpp`` (never copied) plus our
  ``ref_shim.cpp``.  Flags ``-std=c++20 -O2 -ffp-contract=off``: the
  reference's own default ``-march=native`` build contracts FMAs and changes
  output bits, so the oracle pins the uncontracted arithmetic
  that the device (``-fmad=false``) reproduces.  Only built where
  ``/root/reference`` exists; the built ``.so`` travels to the GPU box with the
  repo snapshot (``oracle/_ref/`` is git-ignored, not gpurun-ignored).
* ``oracle/_build/libzsim_oracle.so`` -- the plain-C restatement
  ``oracle/zsim_oracle.c`` (always buildable, needs only gcc).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_ROOT = Path(os.environ.get("ZSIM_REFERENCE_DIR", "/root/reference"))
REF_SRC = REF_ROOT / "proj" / "src"
REF_OUT = HERE / "_ref" / "libzsim_ref.so"
PORT_OUT = HERE / "_build" / "libzsim_oracle.so"
NLOHMANN = Path("/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann")

REF_UNITS = ["common", "config", "geometry", "dynamics", "roads", "scenario_io", "scenario_gen", "simcore",
             "metrics", "train/replay"]
CXX = os.environ.get("CXX", "g++")


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")


def reference_available() -> bool:
    return (REF_SRC / "core" / "simcore.cpp").exists()


def build_ref(force: bool = False) -> Path | None:
    """Compile the reference + shim into oracle/_ref (None if the reference is absent)."""
    if not reference_available():
        return REF_OUT if REF_OUT.exists() else None
    srcs = [REF_SRC / "core" / f"{u}.cpp" for u in REF_UNITS] + [HERE / "ref_shim.cpp", HERE / "ref_policy_shim.cpp"]
    if not force and REF_OUT.exists():
        t = REF_OUT.stat().st_mtime
        if all(s.stat().st_mtime <= t for s in srcs + [HERE / "eigen_mini" / "Eigen" / "Dense"]):
            return REF_OUT
    objdir = HERE / "_ref" / "obj"
    objdir.mkdir(parents=True, exist_ok=True)
    # oracle/eigen_mini stands in for Eigen (absent here) so core/nn/model.hpp
    # and core/train/policy.hpp compile unchanged (ref_policy_shim.cpp)
    flags = ["-std=c++20", "-O2", "-ffp-contract=off", "-fPIC", "-I", str(REF_SRC), "-I", str(NLOHMANN),
             "-I", str(HERE / "eigen_mini"),
             "-I", str(HERE.parent / "include")]
    jobs, objs = [], []
    for s in srcs:
        o = objdir / (s.stem + ".o")
        objs.append(str(o))
        jobs.append([CXX, *flags, "-c", str(s), "-o", str(o)])
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 2) as ex:
        list(ex.map(_run, jobs))
    tmp = REF_OUT.with_suffix(".tmp")
    _run([CXX, "-shared", "-o", str(tmp), *objs, "-lpthread"])
    os.replace(tmp, REF_OUT)
    return REF_OUT


def build_port(force: bool = False) -> Path | None:
    """Compile the plain-C restatement (None if its source is not present yet)."""
    src = HERE / "zsim_oracle.c"
    if not src.exists():
        return None
    if not force and PORT_OUT.exists() and src.stat().st_mtime <= PORT_OUT.stat().st_mtime and \
            (HERE / "zsim_oracle.h").stat().st_mtime <= PORT_OUT.stat().st_mtime:
        return PORT_OUT
    PORT_OUT.parent.mkdir(exist_ok=True)
    tmp = PORT_OUT.with_suffix(".tmp")
    _run(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-I", str(HERE.parent / "include"),
          "-o", str(tmp), str(src), "-lm"])
    os.replace(tmp, PORT_OUT)
    return PORT_OUT


STRESS_OUT = HERE / "_ref" / "libzsim_stress.so"
CSRC = HERE.parent / "paper_2312_15122_b200" / "csrc"


def build_stress(force: bool = False) -> Path:
    """The benchmark workload generator for the oracle side (stress_shim.cpp +
    the generator / ZSIM codec sources), so the reference arm never maps the
    product library."""
    srcs = [HERE / "stress_shim.cpp", CSRC / "zsim_stressgen.cpp", CSRC / "zsim_scenario.cpp"]
    deps = srcs + [CSRC / "zsim_scenario.hpp", CSRC / "zsim_geom.cuh", HERE.parent / "include" / "zsim_gpu.h"]
    if not force and STRESS_OUT.exists() and all(d.stat().st_mtime <= STRESS_OUT.stat().st_mtime for d in deps):
        return STRESS_OUT
    STRESS_OUT.parent.mkdir(exist_ok=True)
    tmp = STRESS_OUT.with_suffix(".tmp")
    _run([CXX, "-std=c++17", "-O2", "-ffp-contract=off", "-fPIC", "-shared",
          "-I", str(HERE.parent / "include"), "-I", str(CSRC), "-o", str(tmp), *map(str, srcs), "-lpthread"])
    os.replace(tmp, STRESS_OUT)
    return STRESS_OUT


DROPIN_OUT = HERE / "_ref" / "dropin_check"


def build_dropin(force: bool = False) -> Path | None:
    """The drop-in demonstration binary: dropin_check.cpp + the reference
    objects + libzsim_gpu.so (needs the reference and the built library)."""
    lib = HERE.parent / "paper_2312_15122_b200" / "libzsim_gpu.so"
    if not reference_available() or not lib.exists() or build_ref(force) is None:
        return DROPIN_OUT if DROPIN_OUT.exists() else None
    src = HERE / "dropin_check.cpp"
    deps = [src, lib, HERE.parent / "include" / "zsim_gpu.hpp", HERE.parent / "include" / "zsim_gpu.h"]
    if not force and DROPIN_OUT.exists() and all(d.stat().st_mtime <= DROPIN_OUT.stat().st_mtime for d in deps):
        return DROPIN_OUT
    objs = [str(HERE / "_ref" / "obj" / f"{Path(u).name}.o") for u in REF_UNITS]
    tmp = DROPIN_OUT.with_suffix(".tmp")
    _run([CXX, "-std=c++20", "-O2", "-ffp-contract=off", "-I", str(REF_SRC), "-I", str(NLOHMANN), "-I",
          str(HERE.parent / "include"), "-o", str(tmp), str(src), *objs, str(lib),
          "-Wl,-rpath,$ORIGIN/../../paper_2312_15122_b200", "-lpthread"])
    os.replace(tmp, DROPIN_OUT)
    return DROPIN_OUT


KV_OUT = HERE / "_ref" / "kv_check"


def build_kv_check(force: bool = False) -> Path | None:
    """The reference's cfg::KeyValue as a stdin/stdout program (kv_check.cpp)."""
    if not reference_available() or build_ref(force) is None:
        return KV_OUT if KV_OUT.exists() else None
    src = HERE / "kv_check.cpp"
    if not force and KV_OUT.exists() and src.stat().st_mtime <= KV_OUT.stat().st_mtime:
        return KV_OUT
    objs = [str(HERE / "_ref" / "obj" / f"{u}.o") for u in ("common", "config")]
    tmp = KV_OUT.with_suffix(".tmp")
    _run([CXX, "-std=c++20", "-O2", "-I", str(REF_SRC), "-o", str(tmp), str(src), *objs, "-lpthread"])
    os.replace(tmp, KV_OUT)
    return KV_OUT


def build(force: bool = False) -> None:
    build_port(force)
    build_stress(force)
    build_ref(force)
    build_kv_check(force)
    build_dropin(force)


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    print(REF_OUT if REF_OUT.exists() else "(no reference)", PORT_OUT if PORT_OUT.exists() else "(no port)")
