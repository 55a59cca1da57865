"""Build the sm_100a kernel library in-tree (no JIT cache: the .so travels).

    python -m paper_1804_10112_b200.build [--verbose]

Produces paper_1804_10112_b200/_lib/libsl_b200.so from csrc/*.cu with
`nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo`, cudart linked
statically so the library does not depend on the CUDA runtime torch ships.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
LIBDIR = PKG / "_lib" / ("alt" if os.environ.get("SL_BUILD_ALT", "") not in ("", "0") else "")
LIB = LIBDIR / "libsl_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
         "-Xcompiler", "-fPIC,-O2", "-cudart", "static", "-I", str(INCLUDE), "-I", str(CSRC)]
if os.environ.get("SL_BUILD_ALT", "") not in ("", "0"):
    FLAGS += ["-DSL_WITH_ALT"]
# A/B experiments: extra -D definitions for an SL_BUILD_ALT build (e.g. SL_DEFS="-DSL_XGATHER=1")
FLAGS += os.environ.get("SL_DEFS", "").split()


# SL_BUILD_ALT=1: also the A/B alternatives kept for measurement (CSR variants
# 1 / 3 / 4, the persistent TMA pipelines of pipe.cu, the resident-range COO
# kernel of coo_resident.cu), into _lib/alt/ —
# load it with SL_LIB_PATH.  The default library carries only the kernels the
# dispatch chooses.
ALT = os.environ.get("SL_BUILD_ALT", "") not in ("", "0")
ALT_ONLY = {"pipe.cu", "coo_resident.cu"}


def sources():
    return sorted(p for p in CSRC.glob("*.cu") if ALT or p.name not in ALT_ONLY)


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    LIBDIR.mkdir(parents=True, exist_ok=True)
    objs, procs = [], []
    for src in sources():                     # one nvcc per translation unit, in parallel
        obj = LIBDIR / (src.stem + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)]
        if verbose:
            cmd += ["-Xptxas", "-v"]
            print(" ".join(cmd), flush=True)
        procs.append((cmd, subprocess.Popen(cmd)))
        objs.append(str(obj))
    for cmd, proc in procs:
        if proc.wait() != 0:
            raise subprocess.CalledProcessError(proc.returncode, cmd)
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(tmp), *objs]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    for o in objs:
        os.unlink(o)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose="--verbose" in sys.argv)
    print(LIB)
