"""Build the native library ``libzsim_gpu.so`` in-tree for sm_100a.

Host C++ (ZSIM codec, staging, stress generator) is compiled with
``-ffp-contract=off`` and every CUDA translation unit with ``-fmad=false`` so
the fp64 arithmetic rounds exactly like the reference built without FMA
contraction.  The CUDA runtime is linked statically so the
library does not depend on which libcudart torch happens to ship.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "libzsim_gpu.so"
BUILD = PKG / "_build"

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUDA_FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-fmad=false", "--expt-relaxed-constexpr",
              "-Xcompiler", "-fPIC,-ffp-contract=off,-fvisibility=hidden", *ARCH]
CXX = os.environ.get("CXX", "g++")
CXX_FLAGS = ["-std=c++17", "-O2", "-fPIC", "-ffp-contract=off", "-fvisibility=hidden", "-Wall"]

CU_SOURCES = ["zsim_kernels.cu", "zsim_capi.cu", "zsim_policy.cu", "zsim_comm.cu"]
CXX_SOURCES = ["zsim_scenario.cpp", "zsim_stressgen.cpp"]


def _sources() -> list[Path]:
    return [CSRC / s for s in CU_SOURCES + CXX_SOURCES] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp")) + [
        PKG.parent / "include" / "zsim_gpu.h"]


def _stale() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    return any(p.stat().st_mtime > t for p in _sources())


def _run(cmd: list[str]) -> str:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stdout + r.stderr


# Diagnostic variant (tools/episode_profile.py): the same sources with
# per-path counters compiled in (ZS_PATHSTATS); never loaded by the product.
PATHSTATS_OUT = BUILD / "pathstats" / "libzsim_gpu_pathstats.so"


def build(force: bool = False, verbose: bool = False, pathstats: bool = False, variant: str | None = None,
          defines: list[str] | None = None, nvcc_flags: list[str] | None = None) -> Path:
    """Compile libzsim_gpu.so (no-op when up to date).  `variant` builds an
    experiment copy with extra -D flags (and nvcc flags) under
    _build/<variant>/ (tools only)."""
    out, bdir, defs = OUT, BUILD, []
    if pathstats:
        out, bdir, defs = PATHSTATS_OUT, PATHSTATS_OUT.parent, ["-DZS_PATHSTATS"]
    if variant:
        bdir = BUILD / variant
        out, defs = bdir / "libzsim_gpu.so", defs + [f"-D{d}" for d in (defines or [])] + list(nvcc_flags or [])
    if not force and not (_stale() if out == OUT else not out.exists() or any(
            p.stat().st_mtime > out.stat().st_mtime for p in _sources())):
        return out
    bdir.mkdir(parents=True, exist_ok=True)
    jobs = []
    for s in CU_SOURCES:
        o = bdir / (s + ".o")
        extra = ["-Xptxas", "-v"] if verbose else []
        jobs.append([NVCC, *CUDA_FLAGS, *defs, *extra, "-I", str(PKG.parent / "include"), "-c", str(CSRC / s), "-o",
                     str(o)])
    for s in CXX_SOURCES:
        o = bdir / (s + ".o")
        jobs.append([CXX, *CXX_FLAGS, "-I", str(PKG.parent / "include"), "-c", str(CSRC / s), "-o", str(o)])
    logs = []
    with cf.ThreadPoolExecutor(max_workers=min(4, os.cpu_count() or 1)) as ex:
        for log in ex.map(_run, jobs):
            logs.append(log)
    objs = [str(bdir / (s + ".o")) for s in CU_SOURCES + CXX_SOURCES]
    tmp = out.with_suffix(".so.tmp")
    _run([NVCC, "-shared", *ARCH, "-Xcompiler", "-fPIC", "-o", str(tmp), *objs, "-lpthread"])
    os.replace(tmp, out)
    if verbose:
        sys.stderr.write("\n".join(l for l in logs if l.strip()) + "\n")
    return out


MULTI_GPU_OUT = PKG / "zsim_multi_gpu"


def build_multi_gpu(force: bool = False) -> Path:
    """The single-process multi-GPU driver (csrc/zsim_multi_gpu.cpp, SURVEY
    8e): host C++ over the C-ABI, linked against libzsim_gpu.so in-tree."""
    lib = build()
    src = CSRC / "zsim_multi_gpu.cpp"
    deps = [src, lib, PKG.parent / "include" / "zsim_gpu.h"]
    if not force and MULTI_GPU_OUT.exists() and all(d.stat().st_mtime <= MULTI_GPU_OUT.stat().st_mtime for d in deps):
        return MULTI_GPU_OUT
    cuda = Path(NVCC).resolve().parent.parent
    tmp = MULTI_GPU_OUT.with_suffix(".tmp")
    _run([CXX, "-std=c++17", "-O2", "-Wall", "-I", str(PKG.parent / "include"), "-I", str(cuda / "include"),
          str(src), "-o", str(tmp), str(lib), "-Wl,-rpath,$ORIGIN", str(cuda / "lib64" / "libcudart_static.a"),
          "-ldl", "-lrt", "-lpthread"])
    os.replace(tmp, MULTI_GPU_OUT)
    return MULTI_GPU_OUT


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), None)
    defs = [a[2:] for a in sys.argv if a.startswith("-D")]
    flags = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--nvcc=")]  # e.g. --nvcc=-Xptxas=-O2
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, pathstats="--pathstats" in sys.argv,
                variant=var, defines=defs, nvcc_flags=flags))
