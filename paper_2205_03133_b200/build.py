"""Builds the in-tree shared libraries (no JIT cache: the .so files travel with
the repo snapshot to the GPU box).

  paper_2205_03133_b200/libpstereo_gpu.so   sm_100a kernels + C ABI + generator
  oracle/libbdis_oracle.so                  CPU checker (test infrastructure)
  oracle/_ref/libbdis_ref.so                the reference itself (only when
                                            /root/reference is present)
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libpstereo_gpu.so"
CLI = PKG / "pstereo_gpu_cli"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

CUDA_SOURCES = ["bdis_kernels.cu", "bdis_patches.cu", "bdis_metrics.cu", "bdis_capi.cu",
                "bdis_synth.cu", "bdis_render.cu"]
CXX_SOURCES = ["host_io.cpp", "bdis_multi.cpp", "host_expand.cpp"]
TOOLS = ["cli.cpp"]
C_SOURCES = ["synth.c"]
HEADERS = ["bdis_device.cuh", "bdis_kernels.h", "synth_core.h", "host_expand.h"]

# Bit-exact parity with the x86-64 SSE2 reference needs IEEE double with no
# FMA contraction anywhere (--fmad=false); the kernels also spell the critical
# operations with explicit _rn intrinsics.
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xptxas", "-v",
]


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd: list[str], verbose: bool) -> str:
    if verbose:
        print(" ".join(str(c) for c in cmd), flush=True)
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        sys.stderr.write(p.stdout + p.stderr)
        raise RuntimeError(f"command failed: {' '.join(str(c) for c in cmd)}")
    return p.stdout + p.stderr


def build_gpu_lib(verbose: bool = False, force: bool = False) -> Path:
    deps = [CSRC / s for s in CUDA_SOURCES + C_SOURCES + CXX_SOURCES + TOOLS + HEADERS]
    deps.append(ROOT / "include" / "pstereo_gpu.h")
    deps.append(ROOT / "include" / "pstereo_gpu.hpp")
    if not force and not _stale(LIB, deps) and not _stale(CLI, deps):
        return LIB
    objdir = ROOT / "build" / "obj"
    objdir.mkdir(parents=True, exist_ok=True)
    objs = []
    log = []
    hdrs = [CSRC / h for h in HEADERS] + [ROOT / "include" / "pstereo_gpu.h"]
    fresh = lambda obj, src: not force and not _stale(obj, [CSRC / src, *hdrs])  # noqa: E731
    for src in CUDA_SOURCES:
        obj = objdir / (src + ".o")
        objs.append(obj)
        plog = objdir / (src + ".ptxas")  # per-source ptxas -v output, joined below
        if not (fresh(obj, src) and plog.exists()):
            plog.write_text(_run([NVCC, *NVCC_FLAGS, "-c", str(CSRC / src), "-o", str(obj)],
                                 verbose))
        log.append(plog.read_text())
    for src in C_SOURCES:
        obj = objdir / (src + ".o")
        _run(["gcc", "-std=gnu11", "-O2", "-fPIC", "-ffp-contract=off", "-c",
              str(CSRC / src), "-o", str(obj)], verbose)
        objs.append(obj)
    for src in CXX_SOURCES:
        obj = objdir / (src + ".o")
        _run(["g++", "-std=c++17", "-O2", "-fPIC", "-Wall", "-Wextra", "-c",
              str(CSRC / src), "-o", str(obj)], verbose)
        objs.append(obj)
    _run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
          "-o", str(LIB), *map(str, objs), "-lpthread", "-lm", "-lz"], verbose)
    (ROOT / "build" / "ptxas.log").write_text("".join(log))
    # the reference's command line (src/runner.cpp) over the shim
    _run(["g++", "-std=c++17", "-O2", "-Wall", "-I", str(ROOT / "include"), str(CSRC / "cli.cpp"),
          "-L", str(PKG), "-lpstereo_gpu", "-Wl,-rpath,$ORIGIN", "-o", str(CLI)], verbose)
    return LIB


def build_oracle(verbose: bool = False) -> None:
    _run(["make", "-s", "-C", str(ROOT / "oracle")], verbose)
    if Path("/root/reference/proj/src").is_dir():
        _run(["make", "-s", "-j8", "-C", str(ROOT / "oracle"), "ref"], verbose)
        # the C++ drop-in check (reference + shim from one caller), test infra
        _run(["sh", str(ROOT / "tests" / "cpp" / "build.sh")], verbose)


def build_all(verbose: bool = False, force: bool = False) -> None:
    build_gpu_lib(verbose=verbose, force=force)
    build_oracle(verbose=verbose)


if __name__ == "__main__":
    build_all(verbose=True, force="--force" in sys.argv)
